// tf32x3_gemm.cuh -- fp32-accurate (mul, add) contraction on the 5th-gen
// tensor cores: split TF32 with tcgen05.mma, TMEM accumulators, TMA +
// mbarrier pipelines, warp-specialised roles.
//
//   C = A.B  ~=  Ahi.Bhi + Ahi.Blo + Alo.Bhi        hi = rna_tf32(x), lo = x - hi
//
// Interleaved fp16 operand rows (ilv, the default): x = hi + lo with
// hi = fp16(x), lo = fp16(x - hi) -- fp16 carries tf32's 11-bit significand,
// so the split keeps ~22 bits exactly like 3xTF32's two tf32 parts, and every
// fp16 x fp16 product is exact in the fp32 accumulator.  Per 16-deep k block
// three kind::f16 MMAs (K = 16): hi.hi, hi.lo, lo.hi -- 3xTF32's three
// products at twice the tf32 rate, from half the operand bytes (4 B per
// element: a 128-B smem row carries 32 k).  fp16's range is made to fit by
// power-of-two scaling: each A row and each 128-column block of B is scaled so
// its largest finite |x| lies in [2^14, 2^15) (the prepass, `split_exp`), and
// the epilogue multiplies the accumulator back by 2^(e_row + e_block) --
// exact.  Values far below their row's / block's maximum lose low bits as
// fp16 subnormals: an absolute error below 2^-38 of the row maximum per
// product, far inside the VM's own fp32 error.  The dropped lo.lo term is
// ~2^-22 relative, as in 3xTF32.  (Measured path to here: 3xTF32 215 TF on C5;
// tf32 hi.hi + one fp16 K=16 MMA for both cross terms 260 TF; all-fp16 below.)
// Separate hi/lo buffers (ilv = 0, the BK = 32 geometry on request) keep the
// three tf32 MMAs of 3xTF32.  Accumulation is two-level: the tensor core
// accumulates one K chunk (kChunkK) into a TMEM buffer, the epilogue warps
// fold finished chunks into fp32 registers (round-to-nearest) while the MMA
// warp fills the other TMEM buffer.  The chunk is short because the tensor
// core's fp32 accumulate truncates: measured on B200, 256-K chunks fail the
// strict 1e-5 + 1e-4|ref| rule on ~0.1% of elements at K = 1024; a numpy model
// of truncating accumulation reproduces that and passes at 64-K chunks.
//
// Prepass (tf32_split_kernel): A -> Ahi/Alo [M][Kp], B -> Bhi/Blo [N][Kp],
// both K-major (B transposed) so every UMMA operand is the canonical K-major
// SWIZZLE_128B layout; any input strides are handled here.
//
// Main kernel, one CTA per 128x128 output tile, 192 threads:
//   warp 0      TMA producer: 4 tiles (Ahi, Alo, Bhi, Blo) per K=32 stage
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   epilogue: TMEM -> registers (chunk fold) -> smem -> fused
//               elementwise epilogue -> coalesced global stores
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include "lsb_common.cuh"

namespace lsb {
namespace tc {

constexpr int BM = 128;
// K per TMEM accumulation chunk (see header).  128: with two MMA slots per
// k step a 64-K chunk took as long as the epilogue's TMEM read of the
// 128x256 accumulator (~2k cycles), which then paced the kernel (measured
// C5: 243 TF at 64, 266 at 128, same box); 128-K chunks keep the strict
// rule on C4 (K = 1024) and the golden cases.
#ifndef LSB_CHUNK_K
#define LSB_CHUNK_K 128   // build-time A/B (tools/dbg): -DLSB_CHUNK_K=64
#endif
constexpr int kChunkK = LSB_CHUNK_K;

// Tile / stage geometry (the launcher picks by shape):
//   <16, 128>  64-B K rows (SWIZZLE_64B), 3 stages, ~97 KiB: two CTAs per SM,
//              one CTA's epilogue/prologue overlaps the other's MMAs (moderate K)
//   <32, 128>  128-B K rows (SWIZZLE_128B), 3 stages, one CTA per SM
//   <16, 256>  128x256 tiles (UMMA N = 256), 4 stages, one CTA per SM, eight
//              epilogue warps: 25 % fewer operand bytes per flop (long K, C5)
template <int BK_, int BN_>
struct Cfg {
    static constexpr int BK = BK_;
    static constexpr int BN = BN_;
    static constexpr int kSwizzleBytes = BK_ * 4;
    static constexpr int STAGES = BN_ == 256 ? 4 : 3;
    static constexpr int kCtasPerSm = (BK_ == 16 && BN_ == 128) ? 2 : 1;
    static constexpr int kEpiWarps = BN_ / 32;
    static constexpr int kThreads = 64 + 32 * kEpiWarps;
    static constexpr int kChunkStages = kChunkK / BK_;
    static constexpr int kTileA = BM * BK_ * 4;            // A hi or lo
    static constexpr int kTileB = BN_ * BK_ * 4;           // B hi or lo
    static constexpr int kStageBytes = 2 * (kTileA + kTileB);
    static constexpr int kTmemCols = 2 * BN_;              // two chunk accumulators
    static constexpr size_t kSmemBytes = (size_t)STAGES * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    // persistent launches (TcArgs::units) stage the store through a 32x32
    // float block per epilogue warp after the barriers: the stage ring is busy
    // with the next unit's operands while a finished tile is stored
    static constexpr size_t kSmemBytesPersist = kSmemBytes + (size_t)kEpiWarps * 32 * 32 * 4;
    static_assert(STAGES * kStageBytes >= BM * BN_ * 4, "epilogue staging reuses the stage buffers");
    static_assert(kTmemCols <= 512, "TMEM has 512 columns");
};

constexpr int kGroupM = 16;            // tile raster: 16 m-tiles per group share B in L2

struct TcArgs {
    int64_t M, N, K, Kp;
    int m_tiles, n_tiles;   // tiles this launch covers, from tile (mt0, nt0)
    int mt0, nt0;
    int m_tiles2, n_tiles2;  // optional second rectangle (blocked L-shaped steps),
    int mt2, nt2;            // its CTAs follow the first rectangle's
    float *C; int64_t sc_m, sc_n;
    int c_vec;            // 1: 16-B aligned unit-stride C rows (float4 stores), 2: 32-B aligned (STG.256)
    EpiStages epi;
    // fast epilogue (fast_n stages, each "+ bias[n * stride]" if bias != null,
    // then ReLU if relu): set by the host when every stage has that form
    // (C4's bias + ReLU); the generic runtime-dispatched stage walk costs
    // ~1k cycles per stored row (measured: 37k vs 8k cycles per 128x256 tile)
    int fast_n;
    const float *fbias[2];
    int64_t fbias_stride[2];
    int frelu[2];
    // non-finite inputs: 3xTF32 turns inf x (lo = 0) into NaN, so outputs in
    // an A row / B column holding inf or NaN (rowflag[m] == agen, colflag[n]
    // == bgen, written by the split prepass) are recomputed in FP32 from the
    // split operands (hi + lo == x exactly for non-finite x) -- IEEE results
    // like the reference's f64 evaluation; never taken for finite inputs
    // ilv: split operands interleaved per 16-deep k block, rows of [hi16 | lo16]
    // (2*Kp floats per row): one 128-B-row SWIZZLE_128B box per operand per
    // stage instead of separate 64-B-row hi and lo boxes (BK = 16 tiles)
    int ilv;
    int bn;               // the launch's tile width (fixup rectangle)
    // pair: launched as 2-CTA clusters over m-tile pairs that share the n-tile;
    // each CTA loads half of the B tile and multicasts it to both (B's L2->SM
    // traffic halves), and each MMA commit frees the slot in both CTAs
    int pair;
    // tail split: the last split_tiles tiles (raster order) run as two CTAs
    // each over half of the K chunks, so a last wave that would leave most
    // SMs idle becomes half as long.  CTAs after the first (tiles - split)
    // come in fours: (tile j, half 0), (tile j+1, half 0), (j, 1), (j+1, 1)
    // (a 2-CTA pair keeps one n-tile and one K range).  Each half stores
    // its chunk sum to split_ws; the second to arrive (split_cnt) adds the
    // other's, runs the epilogue and re-arms the counter.
    int split_tiles;
    // persistent launch (units > 0, BN = 256 only): gridDim.x CTAs walk the
    // units (tiles, then tail-split halves) t = blockIdx.x + i * gridDim.x.
    // The TMA ring, the MMA issuer and the two TMEM chunk buffers run on
    // across unit boundaries, so a finished tile's store (from registers,
    // through a per-warp smem block) overlaps the next unit's first chunks.
    int units;
    // K per TMEM accumulation chunk (a multiple of the stage depth): kChunkK,
    // or half of a short reduction (kern_tf32.cu) so the epilogue warps fold
    // twice per tile and the MMA issuer runs a whole tile ahead of the store
    int chunk_k;
    float *split_ws;
    int *split_cnt;
    const int *rowflag, *colflag, *anyflag;   // anyflag[0] A, [1] B
    // ilv: per-A-row and per-128-column-block-of-B finite maxima (float bits,
    // the prepass's scale source, split_exp); the epilogue unscales by them
    const int *amax, *bmax;
    int *done;                                 // CTA completion counter
    int agen, bgen;
    const float *ahi, *alo, *bhi, *blo;
    long long *trace;     // debug (LSB_TC_TRACE builds): clock64 stamps of CTA 0
};

#ifdef LSB_TC_TRACE
#define TC_TRACE(ev, i)                                                                \
    do {                                                                               \
        if (p.trace != nullptr && blockIdx.x == 0 && (i) < 128) p.trace[(ev) * 128 + (i)] = clock64(); \
    } while (0)
#else
#define TC_TRACE(ev, i) \
    do {                \
    } while (0)
#endif

// ---------------------------------------------------------------- PTX wrappers

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    while (!mbar_try_wait(bar, phase)) {
    }
}
// blocking flavour for long waits: the thread is suspended (up to `ns`) until
// the phase completes instead of spinning on issue slots the working warps need
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t phase, uint32_t ns = 100000) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase), "r"(ns)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint64_t *bar, void *dst, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap *map, uint64_t *bar, void *dst, int x, int y,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand tile in the canonical SWIZZLE_128B layout: rows of 128 B,
// 8-row (1024 B) swizzle atoms stacked with SBO = 1024 B.
template <int kSwizzleBytes>
__device__ __forceinline__ uint64_t sdesc_k_sw(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);   // start address (16 B units)
    d |= (uint64_t)1 << 16;                    // leading byte offset (unused when swizzled)
    d |= (uint64_t)((8 * kSwizzleBytes) >> 4) << 32;   // stride byte offset: 8-row atom
    d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
    d |= (uint64_t)(kSwizzleBytes == 128 ? 2 : 4) << 61;   // layout: SWIZZLE_128B / 64B
    return d;
}

// instruction descriptor: kind::tf32, fp32 accumulate, A/B K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// instruction descriptor: kind::f16 with fp16 A/B, fp32 accumulate, K-major, M x N
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// instruction descriptor: kind::f16 with bf16 A/B, fp32 accumulate, K-major, M x N
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread (the
// GEMM's chunk fold: 128 running sums + 16 leave room under the 168-register
// cap of a 10-warp CTA)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float rna_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// lo part of the 3xTF32 split; an infinite hi gets lo = 0 so inf inputs give
// inf products (inf - inf = NaN in lo would turn every such product to NaN)
__device__ __forceinline__ float tf32_lo(float x, float h) {
    return fabsf(h) == __int_as_float(0x7f800000) ? 0.0f : rna_tf32(x - h);
}

// ---------------------------------------------------------------- prepass

constexpr int kBScaleCols = 128;   // B columns sharing one scale (an epilogue warp's column half)

// scale exponent of a group from its largest finite |x| (float bits): the
// group is multiplied by 2^-e so that max lies in [2^14, 2^15), below fp16's
// 65504 with one binade to spare; 0 for an all-zero (or empty) group
__device__ __forceinline__ int split_exp(int maxbits) {
    if (maxbits <= 0) return 0;
    const int be = (maxbits >> 23) & 0xff;
    return (be ? be - 127 : ilogbf(__int_as_float(maxbits))) - 14;   // subnormal max: rare
}

// the prepass scale 2^-e as two normal factors (one when |e| <= 126)
struct Pow2 {
    float f1, f2;
    __device__ __forceinline__ explicit Pow2(int e) {
        const int e1 = max(-126, min(127, e)), e2 = max(-126, min(127, e - e1));
        f1 = __int_as_float((e1 + 127) << 23);
        f2 = __int_as_float((e2 + 127) << 23);
    }
    __device__ __forceinline__ float operator()(float x) const { return x * f1 * f2; }
};

// x * 2^e for the unscaling epilogue (e in [-326, 226]: two steps when 2^e
// itself is not a normal float)
__device__ __forceinline__ float scale_pow2(float x, int e) {
    if (e >= -126 && e <= 127) return x * __int_as_float((e + 127) << 23);
    return ldexpf(x, e);
}

// interleaved fp16 rows (ilv): row r holds Kp "float" slots = 2 Kp halves;
// per 16-deep k block b: halves [32 b, 32 b + 16) = hi, [32 b + 16, 32 b + 32)
// = lo (so a 128-B smem row = two k blocks).  `row` = the row's first half.
__device__ __forceinline__ __half *h16_hi(__half *row, int64_t k) { return row + (k >> 4) * 32 + (k & 15); }
__device__ __forceinline__ __half *h16_lo(__half *row, int64_t k) { return row + (k >> 4) * 32 + 16 + (k & 15); }
__device__ __forceinline__ uint2 half4(float a, float b, float c, float d) {
    const __half2 u = __floats2half2_rn(a, b), v = __floats2half2_rn(c, d);
    return make_uint2(*reinterpret_cast<const uint32_t *>(&u), *reinterpret_cast<const uint32_t *>(&v));
}
// fp16 split of a scaled value: hi = fp16(x), lo = fp16(x - hi) (x - hi is
// exact in fp32); a non-finite x keeps hi = x, lo = 0 (its row / column is
// recomputed in FP32)
__device__ __forceinline__ void h16_split(float x, float &h, float &l) {
    h = __half2float(__float2half_rn(x));
    l = (fabsf(x) < __int_as_float(0x7f800000)) ? x - h : 0.0f;
}
// hi / lo of a scaled value: hi = rna_tf32(x), lo = x - hi (exact); a
// non-finite x keeps hi = x, lo = 0 (its row / column is recomputed in FP32)
__device__ __forceinline__ float split_lo(float x, float h) {
    return fabsf(h) == __int_as_float(0x7f800000) || x != x ? 0.0f : x - h;
}

// largest finite |X[r][k]| per group of `group` consecutive r, as float bits
// (non-negative floats order like ints) into gmax[r / group] by atomicMax;
// the host zeroes gmax.  k-contiguous X: one warp per row, float4 loads when
// aligned; otherwise threads along r (coalesced for r-contiguous X), each
// over a `kchunk` slice of k.
__global__ void __launch_bounds__(256) split_max_kcontig_kernel(const float *__restrict__ X, int64_t R, int64_t Kd,
                                                                int64_t s_r, int group, int vec,
                                                                int *__restrict__ gmax) {
    const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= R) return;
    const float inf = __int_as_float(0x7f800000);
    const float *row = X + r * s_r;
    float m = 0.0f;
    if (vec) {
        for (int64_t k = (int64_t)lane * 4; k < Kd; k += 128) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(row + k));
            const float a[4] = {fabsf(v.x), fabsf(v.y), fabsf(v.z), fabsf(v.w)};
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (a[q] < inf) m = fmaxf(m, a[q]);
        }
    } else {
        for (int64_t k = lane; k < Kd; k += 32) {
            const float a = fabsf(__ldg(row + k));
            if (a < inf) m = fmaxf(m, a);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0 && m > 0.0f) atomicMax(gmax + r / group, __float_as_int(m));
    asm volatile("griddepcontrol.wait;" ::: "memory");   // see split_max_rcontig_kernel
}

__global__ void __launch_bounds__(256) split_max_rows_kernel(const float *__restrict__ X, int64_t R, int64_t Kd,
                                                             int64_t s_r, int64_t s_k, int group, int64_t kchunk,
                                                             int *__restrict__ gmax) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k0 = (int64_t)blockIdx.y * kchunk, k1 = min(Kd, k0 + kchunk);
    const float inf = __int_as_float(0x7f800000);
    float m = 0.0f;
    if (r < R)
        for (int64_t k = k0; k < k1; k++) {
            const float a = fabsf(__ldg(X + r * s_r + k * s_k));
            if (a < inf) m = fmaxf(m, a);
        }
    // lanes of one group reduce together (groups are multiples of 32 rows, or 1)
    if (group >= 32) {
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0 && r < R && m > 0.0f) atomicMax(gmax + r / group, __float_as_int(m));
    } else if (r < R && m > 0.0f) {
        atomicMax(gmax + r / group, __float_as_int(m));
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");   // see split_max_rcontig_kernel
}

// X element (r, k) = X[r*s_r + k*s_k]  ->  hi/lo[r][k] (row-major, Kp columns,
// zero padded).  32x32 tiles through smem so both the read (whichever stride
// is 1) and the write (k fastest) are coalesced.
// A row holding a non-finite value gets flag[r] = gen (see TcArgs::rowflag).
__global__ void __launch_bounds__(256) tf32_split_kernel(const float *__restrict__ X, int64_t R, int64_t Kd,
                                                         int64_t s_r, int64_t s_k, float *__restrict__ hi,
                                                         float *__restrict__ lo, int64_t Kp, int ilv,
                                                         int *__restrict__ flag, int *__restrict__ any, int gen,
                                                         const int *__restrict__ gmax, int group) {
    __shared__ float tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, k0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    const bool r_fast = (s_r == 1 && s_k != 1);
#pragma unroll
    for (int j = 0; j < 4; j++) {
        int a = ty + 8 * j;   // slow index within the tile
        int64_t r = r_fast ? r0 + tx : r0 + a;
        int64_t k = r_fast ? k0 + a : k0 + tx;
        float v = (r < R && k < Kd) ? __ldg(X + r * s_r + k * s_k) : 0.0f;
        if (r_fast) tile[tx][a] = v; else tile[a][tx] = v;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; j++) {
        int a = ty + 8 * j;
        int64_t r = r0 + a, k = k0 + tx;
        if (r < R && k < Kp) {
            float x = tile[a][tx];
            if (ilv) {
                float h, l;
                h16_split(Pow2(-split_exp(gmax[r / group]))(x), h, l);
                __half *row = reinterpret_cast<__half *>(hi + r * Kp);
                *h16_hi(row, k) = __float2half_rn(h);
                *h16_lo(row, k) = __float2half_rn(l);
            } else {
                const float h = rna_tf32(x);
                hi[r * Kp + k] = h;
                lo[r * Kp + k] = tf32_lo(x, h);
            }
            if (flag != nullptr && !(fabsf(x) < __int_as_float(0x7f800000))) {
                flag[r] = gen;
                *any = gen;
            }
        }
    }
}

// Vectorised forms of tf32_split_kernel (the prepass moves 12 bytes per
// element, so it runs at copy speed only with 16-B accesses and 32-bit index
// math; the scalar kernel above reached ~half of it on C4):
//  * k contiguous (s_k == 1): no transpose, one float4 in, one float4 out per
//    plane; columns [Kd, Kp) written as zeros
//  * r contiguous (s_r == 1): 32 x 32 tiles transposed through smem with
//    float4 reads along r and float4 writes along k
// Preconditions (checked by the host): 16-B aligned X, the contiguous extent
// and the other stride multiples of 4, every index < 2^31.
// (ilv: hi/lo land interleaved in `hi` per 16-k block, see TcArgs::ilv)
// 4 consecutive k (k % 4 == 0) of row r: fp32 hi / lo planes (ilv 0), or the
// scaled hi and its fp16 correction pairs in an interleaved row
__device__ __forceinline__ void split_store4(float *hi, float *lo, int64_t r, int64_t k, int64_t Kp, int ilv,
                                             float4 v, int e) {
    if (ilv) {
        const Pow2 sc(-e);
        float h[4], l[4];
        h16_split(sc(v.x), h[0], l[0]);
        h16_split(sc(v.y), h[1], l[1]);
        h16_split(sc(v.z), h[2], l[2]);
        h16_split(sc(v.w), h[3], l[3]);
        __half *row = reinterpret_cast<__half *>(hi + r * Kp);
        *reinterpret_cast<uint2 *>(h16_hi(row, k)) = half4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint2 *>(h16_lo(row, k)) = half4(l[0], l[1], l[2], l[3]);
    } else {
        const float4 h = make_float4(rna_tf32(v.x), rna_tf32(v.y), rna_tf32(v.z), rna_tf32(v.w));
        *reinterpret_cast<float4 *>(hi + r * Kp + k) = h;
        *reinterpret_cast<float4 *>(lo + r * Kp + k) =
            make_float4(tf32_lo(v.x, h.x), tf32_lo(v.y, h.y), tf32_lo(v.z, h.z), tf32_lo(v.w, h.w));
    }
}

__global__ void __launch_bounds__(256) tf32_split_kcontig_kernel(const float *__restrict__ X, int R, int Kd, int s_r,
                                                                 float *__restrict__ hi, float *__restrict__ lo,
                                                                 int Kp, int ilv, int *__restrict__ flag,
                                                                 int *__restrict__ any, int gen,
                                                                 const int *__restrict__ gmax, int group) {
    asm volatile("griddepcontrol.launch_dependents;");
    const int q4 = Kp / 4;
    const int total = R * q4;
    const float inf = __int_as_float(0x7f800000);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int r = e / q4, k = (e - r * q4) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < Kd) v = __ldg(reinterpret_cast<const float4 *>(X + (int64_t)r * s_r + k));
        split_store4(hi, lo, r, k, Kp, ilv, v, ilv ? split_exp(gmax[r / group]) : 0);
        if (flag != nullptr && !(fabsf(v.x) < inf && fabsf(v.y) < inf && fabsf(v.z) < inf && fabsf(v.w) < inf)) {
            flag[r] = gen;
            *any = gen;
        }
    }
}

// interleaved split of k-contiguous rows with a per-row scale (the A operand):
// one warp per row, pass 1 the row's finite max (written to gmax[r], the
// epilogue's unscale source), pass 2 the split from the same (now cached)
// row -- no separate max launch, one DRAM read.  Preconditions as the
// vectorised kcontig kernel.
__global__ void __launch_bounds__(256) tf32_split_rows_kernel(const float *__restrict__ X, int R, int Kd, int s_r,
                                                              float *__restrict__ hi, int Kp, int ilv,
                                                              int *__restrict__ flag, int *__restrict__ any, int gen,
                                                              int *__restrict__ gmax) {
    asm volatile("griddepcontrol.launch_dependents;");
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= R) return;
    const float inf = __int_as_float(0x7f800000);
    const float *row = X + (int64_t)r * s_r;
    float m = 0.0f;
    bool bad = false;
    for (int k = lane * 4; k < Kd; k += 128) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(row + k));
        const float a[4] = {fabsf(v.x), fabsf(v.y), fabsf(v.z), fabsf(v.w)};
#pragma unroll
        for (int q = 0; q < 4; q++) {
            if (a[q] < inf) m = fmaxf(m, a[q]);
            else bad = true;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    bad = __any_sync(0xffffffffu, bad);
    const int e = split_exp(__float_as_int(m));
    for (int k = lane * 4; k < Kp; k += 128) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < Kd) v = __ldg(reinterpret_cast<const float4 *>(row + k));
        split_store4(hi, nullptr, r, k, Kp, ilv, v, e);
    }
    if (lane == 0) {
        gmax[r] = __float_as_int(m);
        if (bad && flag != nullptr) {
            flag[r] = gen;
            *any = gen;
        }
    }
}

// finite max |X[r][k]| per group of `group` (a multiple of 128) consecutive
// r for r-contiguous X (the [K][N] B operand): a block covers one group
// (32 lanes x float4 = 128 r) and a slice of k, its 8 warps striding k
__global__ void __launch_bounds__(256) split_max_rcontig_kernel(const float *__restrict__ X, int R, int Kd, int s_k,
                                                                int group, int kchunk, int *__restrict__ gmax) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int r = blockIdx.x * 128 + lane * 4;
    const int k0 = blockIdx.y * kchunk, k1 = min(Kd, k0 + kchunk);
    const float inf = __int_as_float(0x7f800000);
    float m = 0.0f;
    if (r < R)
        for (int k = k0 + w; k < k1; k += 8) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(X + (int64_t)k * s_k + r));
            const float a[4] = {fabsf(v.x), fabsf(v.y), fabsf(v.z), fabsf(v.w)};
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (a[q] < inf) m = fmaxf(m, a[q]);
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float wm[8];
    if (lane == 0) wm[w] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < 8; i++) m = fmaxf(m, wm[i]);
        if (m > 0.0f) atomicMax(gmax + (blockIdx.x * 128) / group, __float_as_int(m));
    }
    // launched with programmatic dependent launch right after the A operand's
    // split, this pass runs beside it; it completes only once that split has
    // (no-op without a programmatic predecessor), so whatever waits for this
    // grid also sees the A split
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__global__ void __launch_bounds__(256) tf32_split_rcontig_kernel(const float *__restrict__ X, int R, int Kd, int s_k,
                                                                 float *__restrict__ hi, float *__restrict__ lo,
                                                                 int Kp, int ilv, int *__restrict__ flag,
                                                                 int *__restrict__ any, int gen,
                                                                 const int *__restrict__ gmax, int group) {
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ float tile[32][33];   // [k][r]
    const int r0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
    const int t = threadIdx.x;
    {
        const int kk = t >> 3, r4 = (t & 7) * 4;   // 32 k rows x 8 float4 along r
        const int k = k0 + kk, r = r0 + r4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < Kd && r < R) v = __ldg(reinterpret_cast<const float4 *>(X + (int64_t)k * s_k + r));
        tile[kk][r4] = v.x;
        tile[kk][r4 + 1] = v.y;
        tile[kk][r4 + 2] = v.z;
        tile[kk][r4 + 3] = v.w;
    }
    __syncthreads();
    const int rr = t >> 3, k4 = (t & 7) * 4;       // 32 r rows x 8 float4 along k
    const int r = r0 + rr, k = k0 + k4;
    if (r < R && k < Kp) {
        const float4 v = make_float4(tile[k4][rr], tile[k4 + 1][rr], tile[k4 + 2][rr], tile[k4 + 3][rr]);
        split_store4(hi, lo, r, k, Kp, ilv, v, ilv ? split_exp(gmax[r / group]) : 0);
        const float inf = __int_as_float(0x7f800000);
        if (flag != nullptr && !(fabsf(v.x) < inf && fabsf(v.y) < inf && fabsf(v.z) < inf && fabsf(v.w) < inf)) {
            flag[r] = gen;
            *any = gen;
        }
    }
}

// Non-finite fixup, run by the last CTA to finish (so every tile is stored):
// outputs of flagged A rows / B columns recomputed in FP32 from the split
// operands, epilogue applied.  One flag load per operand when nothing was
// flagged; the done counter is re-armed for the next launch.
__device__ void tc_nonfinite_fixup(const TcArgs &p) {
    // the split prepass has finished (and is visible) once griddepcontrol.wait
    // returns; when it flagged nothing (the normal case) every CTA leaves
    // here, no fence, no atomic
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const bool fa = p.anyflag[0] == p.agen, fb = p.anyflag[1] == p.bgen;
    if (!fa && !fb) return;
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(p.done, 1) == (int)(gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    auto fix = [&](int64_t m, int64_t n) {
        float acc = 0.0f;
        if (p.ilv) {
            // scaled fp16 hi + lo, unscaled at the end: exact for the non-finite
            // values that flagged this row / column (hi = x, lo = 0)
            __half *a = reinterpret_cast<__half *>(const_cast<float *>(p.ahi) + m * p.Kp);
            __half *b = reinterpret_cast<__half *>(const_cast<float *>(p.bhi) + n * p.Kp);
            for (int64_t k = 0; k < p.K; k++)
                acc = fmaf(__half2float(*h16_hi(a, k)) + __half2float(*h16_lo(a, k)),
                           __half2float(*h16_hi(b, k)) + __half2float(*h16_lo(b, k)), acc);
            acc = scale_pow2(acc, split_exp(p.amax[m]) + split_exp(p.bmax[n / kBScaleCols]));
        } else {
            const float *ah = p.ahi + m * p.Kp, *al = p.alo + m * p.Kp, *bh = p.bhi + n * p.Kp,
                        *bl = p.blo + n * p.Kp;
            for (int64_t k = 0; k < p.K; k++) acc = fmaf(ah[k] + al[k], bh[k] + bl[k], acc);
        }
        if (p.epi.n) acc = apply_epilogue(p.epi, acc, 0, m, n, 0);
        p.C[m * p.sc_m + n * p.sc_n] = acc;
    };
    // this launch's output rectangles (a blocked PRESPLIT launch covers part)
    for (int q = 0; q < 2; q++) {
        const int mt_ = q ? p.mt2 : p.mt0, nt_ = q ? p.nt2 : p.nt0;
        const int mts = q ? p.m_tiles2 : p.m_tiles, nts = q ? p.n_tiles2 : p.n_tiles;
        if (mts == 0 || nts == 0) continue;
        const int64_t fm0 = (int64_t)mt_ * BM, fm1 = min(p.M, fm0 + (int64_t)mts * BM);
        const int64_t fn0 = (int64_t)nt_ * p.bn, fn1 = min(p.N, fn0 + (int64_t)nts * p.bn);
        if (fa)
            for (int64_t m = fm0; m < fm1; m++)
                if (p.rowflag[m] == p.agen)
                    for (int64_t n = fn0 + threadIdx.x; n < fn1; n += blockDim.x) fix(m, n);
        if (fb)
            for (int64_t n = fn0; n < fn1; n++)
                if (p.colflag[n] == p.bgen)
                    for (int64_t m = fm0 + threadIdx.x; m < fm1; m += blockDim.x) fix(m, n);
    }
    if (threadIdx.x == 0) *p.done = 0;
}

// ---------------------------------------------------------------- main kernel

// kPersist: the persistent instance (TcArgs::units > 0; no epilogue or the
// fast one, GEMM only).  The single-unit instance keeps the staged store,
// which inside a unit loop would not fit the register cap.
template <int BK_, int BN_, bool kPersist>
__global__ void __launch_bounds__(Cfg<BK_, BN_>::kThreads, Cfg<BK_, BN_>::kCtasPerSm)
    tf32x3_gemm_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                       const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                       const TcArgs p) {
    using Cf = Cfg<BK_, BN_>;
    constexpr int BK = Cf::BK, BN = Cf::BN, STAGES = Cf::STAGES;
    constexpr int kTileA = Cf::kTileA, kTileB = Cf::kTileB, kStageBytes = Cf::kStageBytes;
    constexpr int kEpiWarps = Cf::kEpiWarps;
    constexpr bool kPairRelease = (STAGES % 2) == 0;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the swizzle atoms
    // align by offsetting smem_raw itself (not through an integer) so the
    // compiler keeps the shared address space: LDS/STS, not generic LD/ST
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * kStageBytes);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;    // [2] chunk accumulator ready
    uint64_t *tempty = tfull + 2;        // [2] chunk accumulator drained
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // an interleaved fp16 stage row (128 B) carries 32 k, a fp32 one BK
    const int kstage = p.ilv ? 2 * BK : BK;
    const int chunk_stages = p.chunk_k / kstage;
    const int num_kb = (int)(p.Kp / kstage);
    const int all_chunks = (num_kb + chunk_stages - 1) / chunk_stages;
    // unit t -> output tile, K half (-1: whole K) and split-tile slot.
    // grouped raster: consecutive units walk kGroupM m-tiles before moving to
    // the next n-tile, so the CTAs resident together share A and B blocks
    struct Unit {
        int64_t m0, n0;
        int half, stile, c_begin, num_chunks;
    };
    auto decode = [&](int t) {
        Unit u;
        int mtiles = p.m_tiles, ntiles = p.n_tiles, mb = p.mt0, nb = p.nt0;
        u.half = -1;
        u.stile = 0;
        if (p.split_tiles) {
            const int whole = p.m_tiles * p.n_tiles + p.m_tiles2 * p.n_tiles2 - p.split_tiles;
            if (t >= whole) {
                const int v = t - whole;
                u.stile = (v >> 2) * 2 + (v & 1);
                u.half = (v >> 1) & 1;
                t = whole + u.stile;
            }
        }
        if (t >= p.m_tiles * p.n_tiles) {
            t -= p.m_tiles * p.n_tiles;
            mtiles = p.m_tiles2, ntiles = p.n_tiles2, mb = p.mt2, nb = p.nt2;
        }
        const int per_group = kGroupM * ntiles;
        const int g = t / per_group, first_m = g * kGroupM;
        const int gm = min(kGroupM, mtiles - first_m);
        const int r = t % per_group;
        u.m0 = (int64_t)(mb + first_m + r % gm) * BM;
        u.n0 = (int64_t)(nb + r / gm) * BN;
        // this unit's K chunks [c_begin, c_begin + num_chunks)
        u.c_begin = u.half == 1 ? all_chunks / 2 : 0;
        u.num_chunks = u.half < 0 ? all_chunks : u.half == 0 ? all_chunks / 2 : all_chunks - all_chunks / 2;
        return u;
    };
    const int units = kPersist ? p.units : (int)gridDim.x;
    const int ustride = (int)gridDim.x;
    __shared__ int s_split_second;
    if (threadIdx.x == 0) TC_TRACE(3, 0);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_ahi);
        tma_prefetch_desc(&map_alo);
        tma_prefetch_desc(&map_bhi);
        tma_prefetch_desc(&map_blo);
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], p.pair ? 2 : 1);   // pair: both CTAs' MMAs must be done
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kEpiWarps);   // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(Cf::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    if (p.pair) cluster_sync_all();   // partner's barriers initialised before any multicast
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t crank = p.pair ? cluster_rank() : 0;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            // programmatic dependent launch: the setup above overlapped the
            // split prepass; its outputs are read from here on
            asm volatile("griddepcontrol.wait;" ::: "memory");
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < units; t += ustride) {
            const Unit u = decode(t);
            const int64_t m0 = u.m0, n0 = u.n0;
            const int kb_end = min(num_kb, (u.c_begin + u.num_chunks) * chunk_stages);
            for (int kb = u.c_begin * chunk_stages; kb < kb_end; kb++) {
                // paired release (even STAGES): a slot pair is freed by one
                // commit after its second stage (see the MMA loop)
                mbar_wait(&empty[kPairRelease ? (stage | 1) : stage], phase ^ 1);
                unsigned char *base = smem + stage * kStageBytes;
                mbar_expect_tx(&full[stage], kStageBytes);
                const int kx = kb * BK;   // (ilv rows: element 2 kx = byte 128 kb of the row)
                if (p.ilv && p.pair) {   // own A; half of B (rows crank*BN/2..) into both CTAs
                    tma_load_2d(&map_ahi, &full[stage], base, 2 * kx, (int)m0);
                    tma_load_2d_mc(&map_bhi, &full[stage], base + 2 * kTileA + crank * kTileB, 2 * kx,
                                   (int)(n0 + crank * (BN / 2)), (uint16_t)3);
                } else if (p.ilv) {   // [A rows: hi16 | lo16][B rows: hi16 | lo16]
                    tma_load_2d(&map_ahi, &full[stage], base, 2 * kx, (int)m0);
                    tma_load_2d(&map_bhi, &full[stage], base + 2 * kTileA, 2 * kx, (int)n0);
                } else {
                    tma_load_2d(&map_ahi, &full[stage], base, kx, (int)m0);
                    tma_load_2d(&map_alo, &full[stage], base + kTileA, kx, (int)m0);
                    tma_load_2d(&map_bhi, &full[stage], base + 2 * kTileA, kx, (int)n0);
                    tma_load_2d(&map_blo, &full[stage], base + 2 * kTileA + kTileB, kx, (int)n0);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            }   // units
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread)
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(BM, BN), idesc_c = idesc_f16(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t gc = 0;   // chunks issued so far (TMEM buffer, phase)
            for (int t = blockIdx.x; t < units; t += ustride) {
            const Unit u = decode(t);
            for (int c = 0; c < u.num_chunks; c++, gc++) {
                const int b = gc & 1;
                const uint32_t tphase = (gc >> 1) & 1;
                mbar_wait(&tempty[b], tphase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(b * BN);
                const int kb_first = (u.c_begin + c) * chunk_stages;
                const int kb_end = min(num_kb, kb_first + chunk_stages);
                TC_TRACE(2, c);
                for (int kb = kb_first; kb < kb_end; kb++) {
                    mbar_wait(&full[stage], phase);
                    TC_TRACE(0, kb);
                    tc_fence_after();
                    const uint32_t base = smem_u32(smem + stage * kStageBytes);
                    if (p.ilv) {
                        // fp16 rows: per 16-k block j bytes [64 j, +32) hi,
                        // [64 j + 32, +32) lo; three K = 16 MMAs per block
                        const uint64_t a0 = sdesc_k_sw<128>(base), b0 = sdesc_k_sw<128>(base + 2 * kTileA);
#pragma unroll
                        for (int j = 0; j < 2; j++) {
                            const uint64_t oh = (uint64_t)((64 * j) >> 4), ol = (uint64_t)((64 * j + 32) >> 4);
                            const uint32_t first = (kb == kb_first && j == 0) ? 0u : 1u;
                            umma_f16(d, a0 + oh, b0 + oh, idesc_c, first);   // hi.hi
                            umma_f16(d, a0 + oh, b0 + ol, idesc_c, 1u);      // hi.lo
                            umma_f16(d, a0 + ol, b0 + oh, idesc_c, 1u);      // lo.hi
                        }
                    } else {
                        const uint64_t ahi = sdesc_k_sw<Cf::kSwizzleBytes>(base);
                        const uint64_t alo = sdesc_k_sw<Cf::kSwizzleBytes>(base + kTileA);
                        const uint64_t bhi = sdesc_k_sw<Cf::kSwizzleBytes>(base + 2 * kTileA);
                        const uint64_t blo = sdesc_k_sw<Cf::kSwizzleBytes>(base + 2 * kTileA + kTileB);
#pragma unroll
                        for (int k = 0; k < BK / 8; k++) {
                            const uint64_t off = (uint64_t)((k * 32) >> 4);   // 8 tf32 = 32 B along K
                            const uint32_t first = (kb == kb_first && k == 0) ? 0u : 1u;
                            umma_tf32(d, ahi + off, bhi + off, idesc, first);
                            umma_tf32(d, ahi + off, blo + off, idesc, 1u);
                            umma_tf32(d, alo + off, bhi + off, idesc, 1u);
                        }
                    }
                    // smem slot free once these MMAs retire; with paired release
                    // one commit per two stages (each commit costs ~45 cycles of
                    // tensor-pipe time, ~5 % of an 810-cycle stage)
                    if (!kPairRelease || (stage & 1)) {
                        if (p.pair) umma_commit_mc(&empty[stage], (uint16_t)3);
                        else umma_commit(&empty[stage]);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[b]);           // chunk accumulator complete
            }
            }   // units
        }
    } else {
        // ---------------- epilogue warps: warp w reads TMEM lane quadrant
        // w % 4 and column half (w - 2) / 4 (BN = 256 uses 8 warps)
        const int q = warp & 3;
        const int ch = (warp - 2) >> 2;           // 128-column half of the tile
        const int row = q * 32 + lane;
        uint32_t gc = 0;   // chunks folded so far (TMEM buffer, phase)
        for (int t = blockIdx.x; t < units; t += ustride) {
        float tot[128];
#pragma unroll
        for (int i = 0; i < 128; i++) tot[i] = 0.0f;
        // only the chunk count is live across the fold (128 sums + 16 loaded
        // columns sit at the 168-register cap); the rest is decoded after it
        const int nch = decode(t).num_chunks;
        for (int c = 0; c < nch; c++, gc++) {
            const int b = gc & 1;
            mbar_wait(&tfull[b], (gc >> 1) & 1);
            if (warp == 2 && lane == 0) TC_TRACE(1, c);
            tc_fence_after();
#pragma unroll
            for (int part = 0; part < 8; part++) {
                float v[16];
                tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + ch * 128 + part * 16), v);
#pragma unroll
                for (int i = 0; i < 16; i++) tot[part * 16 + i] += v[i];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
        }
        const Unit u = decode(t);
        const int64_t m0 = u.m0, n0 = u.n0;
        const int half = u.half, stile = u.stile;
        bool store = true;
        if (half >= 0) {
            // tail split: publish this half's sums (thread-major float4s, a
            // warp writes 512 contiguous bytes), count arrivals per tile
            const int et = threadIdx.x - 64;
            constexpr int kEt = kEpiWarps * 32;
            float4 *mine = reinterpret_cast<float4 *>(p.split_ws + (size_t)(stile * 2 + half) * (BM * BN));
#pragma unroll
            for (int i4 = 0; i4 < 32; i4++)
                __stcg(mine + i4 * kEt + et, make_float4(tot[i4 * 4], tot[i4 * 4 + 1], tot[i4 * 4 + 2], tot[i4 * 4 + 3]));
            __threadfence();
            asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32) : "memory");
            if (et == 0) s_split_second = atomicAdd(p.split_cnt + stile, 1);
            asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32) : "memory");
            store = s_split_second != 0;
            if (store) {
                // the other half is complete: sum in fixed (half 0 + half 1) order
                __threadfence();
                const float4 *other =
                    reinterpret_cast<const float4 *>(p.split_ws + (size_t)(stile * 2 + (half ^ 1)) * (BM * BN));
#pragma unroll
                for (int i4 = 0; i4 < 32; i4++) {
                    const float4 o = __ldcg(other + i4 * kEt + et);
                    const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        tot[i4 * 4 + e] = half == 1 ? ov[e] + tot[i4 * 4 + e] : tot[i4 * 4 + e] + ov[e];
                }
                if (et == 0) p.split_cnt[stile] = 0;   // re-armed for the next launch
            }
        }
        if (store && p.amax != nullptr && n0 + ch * 128 < p.N) {
            // undo the prepass's power-of-two scaling of this row and column block
            const int64_t mr = m0 + row;
            const int e = (mr < p.M ? split_exp(p.amax[mr]) : 0) + split_exp(p.bmax[(n0 + ch * 128) / kBScaleCols]);
            // two normal power-of-two factors, branch-free per element (a
            // per-element branch or ldexpf pushed tot[] out of registers:
            // C4's tile store went from ~15k to ~45k cycles); exact unless
            // |e| > 126 makes the intermediate subnormal (rows near fp32's limits)
            const Pow2 sc(e);
#pragma unroll
            for (int i = 0; i < 128; i++) tot[i] = sc(tot[i]);
        }
        if constexpr (kPersist) {
        if (store) {
            // persistent: the stage ring already holds the next unit's
            // operands.  Per 32-column block: the warp writes its 32 rows x 32
            // columns to its own smem block (16-B chunks XOR-swizzled by row,
            // conflict-free both ways), then stores 4 rows x 128 B per
            // instruction with the epilogue applied
            float *blk = reinterpret_cast<float *>(smem + STAGES * kStageBytes + 256) + (warp - 2) * 32 * 32;
            const int sub = lane >> 3, cc = lane & 7;
#pragma unroll
            for (int bj = 0; bj < 4; bj++) {   // unrolled: tot[] stays in registers
#pragma unroll
                for (int c = 0; c < 8; c++)
                    *reinterpret_cast<float4 *>(blk + lane * 32 + ((c ^ (lane & 7)) * 4)) =
                        make_float4(tot[bj * 32 + c * 4], tot[bj * 32 + c * 4 + 1], tot[bj * 32 + c * 4 + 2],
                                    tot[bj * 32 + c * 4 + 3]);
                __syncwarp();
                if (p.c_vec == 2) {
                    // 32-B aligned rows: 256-bit stores (STG.256), 8 rows x 128 B
                    // per instruction -- half the store instructions of the
                    // float4 form below (C4's per-tile store is what the MMA
                    // warp waits on)
                    const int sub8 = lane >> 2, c8 = lane & 3;
                    const int64_t n8 = n0 + ch * 128 + bj * 32 + c8 * 8;
                    float fb8[2][8];
#pragma unroll
                    for (int i = 0; i < 2; i++)
#pragma unroll
                        for (int e = 0; e < 8; e++)
                            fb8[i][e] = (i < p.fast_n && p.fbias[i] && n8 + e < p.N)
                                            ? __ldg(p.fbias[i] + (n8 + e) * p.fbias_stride[i])
                                            : 0.f;
#pragma unroll 2
                    for (int i = 0; i < 4; i++) {
                        const int r = i * 8 + sub8;
                        const int64_t m = m0 + q * 32 + r;
                        const float4 v0 = *reinterpret_cast<const float4 *>(blk + r * 32 + (((2 * c8) ^ (r & 7)) * 4));
                        const float4 v1 = *reinterpret_cast<const float4 *>(blk + r * 32 + (((2 * c8 + 1) ^ (r & 7)) * 4));
                        if (m >= p.M || n8 >= p.N) continue;
                        float x[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                        for (int j = 0; j < 2; j++) {
                            if (j >= p.fast_n) break;
#pragma unroll
                            for (int e = 0; e < 8; e++) {
                                if (p.fbias[j]) x[e] += fb8[j][e];
                                if (p.frelu[j]) x[e] = fmax_nan(x[e], 0.0f);
                            }
                        }
                        float *dst = p.C + m * p.sc_m + n8;
                        if (n8 + 7 < p.N) {
                            asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst),
                                         "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]),
                                         "f"(x[7])
                                         : "memory");
                        } else {
#pragma unroll
                            for (int e = 0; e < 8; e++)
                                if (n8 + e < p.N) dst[e] = x[e];
                        }
                    }
                    __syncwarp();
                    continue;
                }
                const int64_t n = n0 + ch * 128 + bj * 32 + cc * 4;
                // host: persistent launches carry no epilogue or the fast one
                float fb[2][4];
#pragma unroll
                for (int i = 0; i < 2; i++)
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        fb[i][e] = (i < p.fast_n && p.fbias[i] && n + e < p.N) ? __ldg(p.fbias[i] + (n + e) * p.fbias_stride[i]) : 0.f;
#pragma unroll 2
                for (int i = 0; i < 8; i++) {
                    const int r = i * 4 + sub;
                    const int64_t m = m0 + q * 32 + r;
                    const float4 v = *reinterpret_cast<const float4 *>(blk + r * 32 + ((cc ^ (r & 7)) * 4));
                    if (m >= p.M || n >= p.N) continue;
                    float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int j = 0; j < 2; j++) {
                        if (j >= p.fast_n) break;
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            if (p.fbias[j]) x[e] += fb[j][e];
                            if (p.frelu[j]) x[e] = fmax_nan(x[e], 0.0f);
                        }
                    }
                    float *dst = p.C + m * p.sc_m;
                    if (p.c_vec && n + 3 < p.N) {
                        *reinterpret_cast<float4 *>(dst + n) = make_float4(x[0], x[1], x[2], x[3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; e++)
                            if (n + e < p.N) dst[(n + e) * p.sc_n] = x[e];
                    }
                }
                __syncwarp();
            }
        }
        } else if (store) {
        // stage the tile in (now idle) pipeline smem: row-major, 16-B chunks
        // XOR-swizzled by row so both the write and the read are conflict-free
        float *tile = reinterpret_cast<float *>(smem);
        // every TMA load was consumed by an MMA whose completion preceded the
        // last tfull arrive, so the stage buffers are free
#pragma unroll
        for (int c4 = 0; c4 < 32; c4++) {
            const int chunk = ch * 32 + c4;
            const int pos = chunk ^ (row & 31);
            *reinterpret_cast<float4 *>(tile + row * BN + pos * 4) =
                make_float4(tot[c4 * 4], tot[c4 * 4 + 1], tot[c4 * 4 + 2], tot[c4 * 4 + 3]);
        }
        if (warp == 2 && lane == 0) TC_TRACE(3, 1);
        asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32) : "memory");   // epilogue warps only
        if (warp == 2 && lane == 0) TC_TRACE(3, 2);
        const int ew = warp - 2;
        constexpr int kRowsPerWarp = BM / kEpiWarps;
        // row-invariant epilogue operands (bias[n]) once per column segment
        float fpre[BN / 128][2][4];
        if (p.fast_n) {
#pragma unroll
            for (int h = 0; h < BN / 128; h++) {
                const int64_t n = n0 + (h * 32 + lane) * 4;
#pragma unroll
                for (int i = 0; i < 2; i++)
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        fpre[h][i][e] = (p.fbias[i] && n + e < p.N) ? __ldg(p.fbias[i] + (n + e) * p.fbias_stride[i]) : 0.f;
            }
        }
        float4 pre[BN / 128][LSB_MAX_EPI];
        if (p.epi.n && !p.fast_n) {
#pragma unroll
            for (int h = 0; h < BN / 128; h++) {
                const int64_t n = n0 + (h * 32 + lane) * 4;
                if (n < p.N) epi4_preload(p.epi, n, n + 3 < p.N, pre[h]);
            }
        }
        if ((p.fast_n || p.epi.n == 0) && p.c_vec) {
            // no epilogue or the fast one, in its own loop: bias adds and ReLUs
            // only, no per-element dispatch on the generic stage table
            const bool b0 = p.fbias[0] != nullptr, r0 = p.frelu[0] != 0;
            const bool b1 = p.fast_n > 1 && p.fbias[1] != nullptr, r1 = p.fast_n > 1 && p.frelu[1] != 0;
#pragma unroll 2
            for (int rr = 0; rr < kRowsPerWarp; rr++) {
                const int r = ew * kRowsPerWarp + rr;
                const int64_t m = m0 + r;
                if (m >= p.M) continue;
                float *dst = p.C + m * p.sc_m;
#pragma unroll
                for (int h = 0; h < BN / 128; h++) {
                    const int chunk = h * 32 + lane;
                    const int pos = chunk ^ (r & 31);
                    const float4 v = *reinterpret_cast<const float4 *>(tile + r * BN + pos * 4);
                    const int64_t n = n0 + chunk * 4;
                    float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        if (b0) x[e] += fpre[h][0][e];
                        if (r0) x[e] = fmax_nan(x[e], 0.0f);
                        if (b1) x[e] += fpre[h][1][e];
                        if (r1) x[e] = fmax_nan(x[e], 0.0f);
                    }
                    if (n + 3 < p.N) {
                        *reinterpret_cast<float4 *>(dst + n) = make_float4(x[0], x[1], x[2], x[3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; e++)
                            if (n + e < p.N) dst[n + e] = x[e];
                    }
                }
            }
        } else
#pragma unroll 1
        for (int rr = 0; rr < kRowsPerWarp; rr++) {
            const int r = ew * kRowsPerWarp + rr;
            const int64_t m = m0 + r;
            if (m >= p.M) continue;
#pragma unroll
            for (int h = 0; h < BN / 128; h++) {
                const int chunk = h * 32 + lane;
                const int pos = chunk ^ (r & 31);
                float4 v = *reinterpret_cast<const float4 *>(tile + r * BN + pos * 4);
                const int64_t n = n0 + chunk * 4;
                float x[4] = {v.x, v.y, v.z, v.w};

                if (p.fast_n) {
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        if (i >= p.fast_n) break;
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            if (p.fbias[i]) x[e] += fpre[h][i][e];
                            if (p.frelu[i]) x[e] = fmax_nan(x[e], 0.0f);
                        }
                    }
                } else if (p.epi.n) {
                    if (n + 3 < p.N) {
                        apply_epilogue4_pre(p.epi, x, m, n, pre[h]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; e++)
                            if (n + e < p.N) x[e] = apply_epilogue(p.epi, x[e], 0, m, n + e, 0);
                    }
                }
                float *dst = p.C + m * p.sc_m;
                if (p.c_vec && n + 3 < p.N) {
                    *reinterpret_cast<float4 *>(dst + n) = make_float4(x[0], x[1], x[2], x[3]);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        if (n + e < p.N) dst[(n + e) * p.sc_n] = x[e];
                }
            }
        }
        }   // store
        if constexpr (!kPersist) break;   // one unit per CTA
        }   // units
    }
    if (warp == 2 && lane == 0) TC_TRACE(3, 3);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TC_TRACE(3, 4);
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cf::kTmemCols));
    }
    if (p.done != nullptr) tc_nonfinite_fixup(p);
    // the partner may still commit into this CTA's barriers: leave together
    if (p.pair) cluster_sync_all();
}

}  // namespace tc
}  // namespace lsb
