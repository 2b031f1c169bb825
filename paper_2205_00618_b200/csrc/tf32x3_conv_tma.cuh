// tf32x3_conv_tma.cuh -- NCHW direct convolution on the tensor cores, fed by
// TMA: implicit GEMM D[pixel][co] = Σ_(r,s,c) X[pixel, tap] W[co, tap] in
// split-TF32 (Xhi.Whi + Xhi.Wlo + Xlo.Whi).
//
// The gather variant (tf32x3_conv.cuh) loads X with per-thread LDGs; its
// per-stage fence.proxy.async drains every load still in flight, so each stage
// paid a full L2 round trip.  Here no thread ever waits on global memory:
//   warp 0      TMA of raw X boxes {36 w, 4 c, 4 h, 1 n} (SWIZZLE_NONE, zero
//               fill = the conv's zero padding) into a 3-slot raw ring; the
//               taps are ordered (r, s, c) so 4 consecutive taps are 4
//               channels of one (r, s) and one box holds a 128-pixel x 4-tap
//               operand group (the box starts at the 16-B aligned column
//               below the tap's first input column; TMA rejects unaligned
//               innermost coordinates)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warp 2      one 8 KiB bulk copy per stage of the pre-split filter tiles,
//               stored by filter_image_kernel as the stage's smem image
//   warps 3-10  converters: raw box -> shift by the tap's column offset (0..3,
//               warp-uniform) -> tf32 hi/lo -> MN-major SW128_32B operand
//               (16-B stores), fence.proxy.async (cheap: nothing in flight)
//               + mbarrier arrive; afterwards all eight drain TMEM (two
//               warps per lane quadrant) and store the tile with the fused
//               epilogue
// Output tile: 4 output rows x 32 output columns of one image (128 pixels);
// operand row m = 32 * row + column.  Accumulation in CT_CHUNKS TMEM buffers
// as in the GEMM path (tensor-core accumulate truncates).
#pragma once

#include "tf32x3_conv.cuh"

namespace lsb {
namespace tc {

constexpr int CT_BN = 64;                 // output channels per tile (UMMA N)
constexpr int CT_BK = 16;                 // taps per stage = 4 groups of 4 channels
constexpr int CT_MSTAGES = 3;             // A operand stages (hi/lo)
constexpr int CT_BSTAGES = 4;             // B (filter) stages: own ring, loads run ahead of the MMA
constexpr int CT_RSTAGES = 3;             // raw X stages
constexpr int CT_CONV_WARPS = 8;          // epilogue warps (2 per TMEM lane quadrant)
#ifndef CT_SPLIT_WARPS
#define CT_SPLIT_WARPS 4                  // of which split the operands in the mainloop
#endif
constexpr int CT_THREADS = 96 + 32 * CT_CONV_WARPS;   // 352
constexpr int CT_CHUNKS = 2;              // TMEM accumulators of 128 columns (2 x 128: 2 CTAs / SM)
constexpr int CT_ACC_COLS = 2 * CT_BN;    // [Xhi.Whi + Xlo.Whi | Xhi.Wlo]
constexpr int CT_RAW_W = 36;              // box width: 32 columns + up to 3 of alignment shift
constexpr int CT_RAW_GROUP = 4 * 4 * CT_RAW_W * 4;    // [h 4][c 4][w 36] fp32 = 2304 B
constexpr int CT_RAW_STAGE = 4 * CT_RAW_GROUP;        // 9216 B
constexpr int CT_TILE_A = 128 * CT_BK * 4;            // 8 KiB
constexpr int CT_TILE_B = CT_BN * CT_BK * 4;          // 4 KiB
constexpr int CT_MSTAGE = 2 * CT_TILE_A;                // 16 KiB
constexpr int CT_BSTAGE = 2 * CT_TILE_B;                // 8 KiB
constexpr int CT_MAX_GROUPS = 256;        // Kp <= 1024
__host__ __device__ constexpr size_t ct_smem_bytes(int64_t groups) {
    return (size_t)CT_MSTAGES * CT_MSTAGE + (size_t)CT_BSTAGES * CT_BSTAGE + (size_t)CT_RSTAGES * CT_RAW_STAGE + 256 +
           (size_t)groups * 16 + 1024;
}
static_assert(CT_MSTAGES * CT_MSTAGE >= CT_BN * 128 * 4, "epilogue staging reuses the A stages");

struct ConvTmaArgs {
    int64_t C, K, Kp, R, S, HO, WO, ph, pw, dh, dw, sh;
    int64_t n_img, tiles_h, tiles_w, CO;
    const float *wimg;    // filter_image_kernel output
    float *o;
    int64_t so[4];
    int stages_per_chunk;
    int dbg;              // debug: 1 = no raw TMA, 2 = no split stores, 4 = no MMAs (timing experiments)
    EpiStages epi;
    long long *trace;     // debug: per-stage clock64 stamps of CTA 0 (null = off)
};

#ifdef LSB_CT_TRACE
#define CT_TRACE(ev, kb)                                                                                 \
    do {                                                                                                 \
        if (p.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && (kb) < 64)                      \
            p.trace[(ev) * 64 + (kb)] = clock64();                                                       \
    } while (0)
#else
#define CT_TRACE(ev, kb) \
    do {                 \
    } while (0)
#endif
#define CT_TRACE_LANE(ev, kb)                   \
    do {                                        \
        if (lane == 0 && cw == 0) CT_TRACE(ev, kb); \
    } while (0)

__device__ __forceinline__ void tma_load_4d(const CUtensorMap *map, uint64_t *bar, void *dst, int x, int y, int z,
                                            int w) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w)
        : "memory");
}

// 1-D bulk copy global -> shared, completion on an mbarrier (tx bytes)
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// filters W[co][c][r][s] -> the exact shared-memory image of every stage's B
// operand: [co tile][stage][hi | lo][64 co rows x 16 taps, K-major SWIZZLE_64B],
// taps in (r, s, c) order, so one 8 KiB bulk copy feeds a stage (a 2-D TMA
// box of 64-B rows costs one request per row)
// (tap k -> (r, s) = k / Cp, channel c = k % Cp; zero for c >= C or k >= K)
// One thread per element with 32-bit index decomposition (the int64 div/mod
// chain per element made this tiny prepass take 4.9 us on C3).  The body is
// shared with the NHWC conv's fused prepass (extra blocks of its X split).
struct FilterImgArgs {
    const float *w;
    int64_t CO, K, Kp, C, Cp, S;
    int64_t sw[4];
    float *img;
    // 0: rows 0-63 hi, 64-127 lo; 1: channel c's hi / lo rows at
    // 32 (c / 16) + 2 (c % 16) and +1 (tf32x3_conv_nhwc_t_kernel)
    int ilv_rows;
};

__device__ __forceinline__ void filter_image_body(const FilterImgArgs &f, int *any, int gen, int first, int step) {
    const int nkb = (int)(f.Kp / CT_BK);
    const int co_tiles = (int)((f.CO + CT_BN - 1) / CT_BN);
    const int total = co_tiles * nkb * CT_BN * CT_BK;
    const int cp = (int)f.Cp, sS = (int)f.S, kK = (int)f.K, cC = (int)f.C;
    for (int e = first; e < total; e += step) {
        const int kk = e & (CT_BK - 1), n = (e >> 4) & (CT_BN - 1);
        const int t = e >> 10;   // / (CT_BK * CT_BN)
        const int kb = t % nkb, ct = t / nkb;
        const int64_t co = (int64_t)ct * CT_BN + n;
        const int k = kb * CT_BK + kk;
        const int rs = k / cp, c = k - rs * cp;
        float v = 0.0f;
        if (co < f.CO && k < kK && c < cC) {
            const int r = rs / sS, sx = rs - r * sS;
            v = __ldg(f.w + co * f.sw[0] + c * f.sw[1] + r * f.sw[2] + sx * f.sw[3]);
        }
        const float h = rna_tf32(v);
        const float l = tf32_lo(v, h);
        if (any != nullptr && !(fabsf(v) < __int_as_float(0x7f800000))) *any = gen;
        float *base = f.img + ((int64_t)(ct * nkb + kb) * 2) * (CT_BN * CT_BK);
        // row R of the 128-row K-major SW64 image: 16 floats, 16-B chunks XOR (R >> 1) & 3
        const int rh = f.ilv_rows ? 32 * (n >> 4) + 2 * (n & 15) : n;
        const int rl = f.ilv_rows ? rh + 1 : CT_BN + n;
        base[rh * 16 + (((kk >> 2) ^ ((rh >> 1) & 3)) << 2) + (kk & 3)] = h;
        base[rl * 16 + (((kk >> 2) ^ ((rl >> 1) & 3)) << 2) + (kk & 3)] = l;
    }
}

__global__ void __launch_bounds__(256) filter_image_kernel(const FilterImgArgs f, int *__restrict__ any, int gen) {
    asm volatile("griddepcontrol.launch_dependents;");
    filter_image_body(f, any, gen, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

__device__ __forceinline__ void split4_store(uint32_t dst_hi, uint32_t dst_lo, float a, float b, float c, float d) {
    const float ha = split_hi(a), hb = split_hi(b), hc = split_hi(c), hd = split_hi(d);
    const float la = split_lo(a, ha), lb = split_lo(b, hb), lc = split_lo(c, hc), ld = split_lo(d, hd);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst_hi), "f"(ha), "f"(hb), "f"(hc), "f"(hd)
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst_lo), "f"(la), "f"(lb), "f"(lc), "f"(ld)
                 : "memory");
}

// 32 lanes x 16 columns, no wait (pair with tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
                 : "memory");
    return v;
}

// grid: x = image * tiles_h * tiles_w output tiles, y = channel tiles
__global__ void __launch_bounds__(CT_THREADS, 2)
    tf32x3_conv_tma_kernel(const __grid_constant__ CUtensorMap map_x, const ConvTmaArgs p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char *bring = smem + CT_MSTAGES * CT_MSTAGE;
    unsigned char *raw = bring + CT_BSTAGES * CT_BSTAGE;
    uint64_t *full = reinterpret_cast<uint64_t *>(raw + CT_RSTAGES * CT_RAW_STAGE);
    uint64_t *empty = full + CT_MSTAGES;
    uint64_t *bfull = empty + CT_MSTAGES;
    uint64_t *bempty = bfull + CT_BSTAGES;
    uint64_t *rfull = bempty + CT_BSTAGES;
    uint64_t *rempty = rfull + CT_RSTAGES;
    uint64_t *tdone = rempty + CT_RSTAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tdone + 1);
    int4 *gtab = reinterpret_cast<int4 *>(raw + CT_RSTAGES * CT_RAW_STAGE + 256);   // per 4-tap group

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t t = blockIdx.x;
    const int tw = (int)(t % p.tiles_w);
    t /= p.tiles_w;
    const int th = (int)(t % p.tiles_h);
    const int n = (int)(t / p.tiles_h);
    const int h0 = th * 4, w0 = tw * 32;
    const int64_t c0 = (int64_t)blockIdx.y * CT_BN;
    const int num_kb = (int)(p.Kp / CT_BK);
    const int groups = (int)(p.Kp / 4);
    if (threadIdx.x == 0) CT_TRACE(5, 2);

    // group table: {aligned input column of the box, channel, input row, shift}
    for (int g = threadIdx.x; g < groups; g += CT_THREADS) {
        const int64_t k0 = 4 * (int64_t)g;
        if (k0 < p.K) {
            const int64_t rs = k0 / p.C, c = k0 % p.C, r = rs / p.S, s = rs % p.S;
            const int win = (int)(w0 - p.pw + s * p.dw);
            const int wal = win & ~3;
            gtab[g] = make_int4(wal, (int)c, (int)(h0 * p.sh - p.ph + r * p.dh), win - wal);
        } else {
            gtab[g] = make_int4(0, (int)p.C, 0, 0);   // padded taps: channel out of range -> zero box
        }
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_x);
        for (int s = 0; s < CT_MSTAGES; s++) {
            mbar_init(&full[s], CT_SPLIT_WARPS);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < CT_BSTAGES; s++) {
            mbar_init(&bfull[s], 1);
            mbar_init(&bempty[s], 1);
        }
        for (int s = 0; s < CT_RSTAGES; s++) {
            mbar_init(&rfull[s], 1);
            mbar_init(&rempty[s], CT_SPLIT_WARPS);
        }
        mbar_init(tdone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(CT_CHUNKS * CT_ACC_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA: raw X boxes
        if (lane == 0) {
            for (int kb = 0; kb < num_kb; kb++) {
                const int slot = kb % CT_RSTAGES;
                mbar_wait(&rempty[slot], (uint32_t)(((kb / CT_RSTAGES) & 1) ^ 1));
                CT_TRACE(0, kb);
                if (p.dbg & 1) {
                    mbar_arrive(&rfull[slot]);
                    continue;
                }
                mbar_expect_tx(&rfull[slot], CT_RAW_STAGE);
                unsigned char *dst = raw + slot * CT_RAW_STAGE;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int4 e = gtab[kb * 4 + j];
                    tma_load_4d(&map_x, &rfull[slot], dst + j * CT_RAW_GROUP, e.x, e.y, e.z, n);
                }
            }
        }
    } else if (warp == 2) {
        // ---------------- TMA: filter hi/lo tiles [CT_BN co][CT_BK taps]
        if (lane == 0) {
            for (int kb = 0; kb < num_kb; kb++) {
                const int slot = kb % CT_BSTAGES;
                mbar_wait(&bempty[slot], (uint32_t)(((kb / CT_BSTAGES) & 1) ^ 1));
                mbar_expect_tx(&bfull[slot], CT_BSTAGE);
                bulk_load(bring + slot * CT_BSTAGE, p.wimg + ((int64_t)blockIdx.y * num_kb + kb) * (2 * CT_BN * CT_BK),
                          CT_BSTAGE, &bfull[slot]);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (A: MN-major SW128_32B, B: K-major SW64)
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(128, CT_BN) | (1u << 15);
            constexpr uint32_t idesc_n128 = idesc_tf32(128, 2 * CT_BN) | (1u << 15);
            for (int kb = 0; kb < num_kb; kb++) {
                const int slot = kb % CT_MSTAGES, bslot = kb % CT_BSTAGES;
                mbar_wait(&bfull[bslot], (uint32_t)((kb / CT_BSTAGES) & 1));
                mbar_wait(&full[slot], (uint32_t)((kb / CT_MSTAGES) & 1));
                CT_TRACE(1, kb);
                tc_fence_after();
                const int chunk = kb / p.stages_per_chunk;
                const uint32_t d = tmem + (uint32_t)(chunk * CT_ACC_COLS);
                const uint32_t base = smem_u32(smem + slot * CT_MSTAGE);
                const uint64_t ahi = sdesc_mn_sw128_32b(base), alo = sdesc_mn_sw128_32b(base + CT_TILE_A);
                const uint64_t bhi = sdesc_k_sw<64>(smem_u32(bring + bslot * CT_BSTAGE));
                // B rows 0-63 = Whi, 64-127 = Wlo (contiguous K-major tiles):
                // one N=128 MMA gives Xhi.Whi | Xhi.Wlo, an N=64 one adds
                // Xlo.Whi onto the first half -- 2 tensor instructions per
                // 8 taps instead of 3 (N <= 128 costs the same per instruction)
#pragma unroll
                for (int k = 0; k < CT_BK / 8; k++) {
                    if (p.dbg & 4) break;
                    const uint64_t aoff = (uint64_t)((k * 4096) >> 4);
                    const uint64_t boff = (uint64_t)((k * 32) >> 4);
                    const uint32_t first = (kb % p.stages_per_chunk == 0 && k == 0) ? 0u : 1u;
                    umma_tf32(d, ahi + aoff, bhi + boff, idesc_n128, first);
                    umma_tf32(d, alo + aoff, bhi + boff, idesc, 1u);
                }
                umma_commit(&empty[slot]);
                umma_commit(&bempty[bslot]);
            }
            umma_commit(tdone);
        }
    } else {
        // ---------------- converters (warps 3..10; the first CT_SPLIT_WARPS split)
        const int cw = warp - 3;
        const uint32_t sbase = smem_u32(smem), rbase = smem_u32(raw);
        // chunk q = cw*32 + lane + 32*CT_SPLIT_WARPS*i: group j = q>>7, row
        // h = (q>>5)&3, channel c = (q>>3)&3 (= lane>>3), 4-column block
        // wq = q&7 (= lane&7)
        const int c = lane >> 3, wq = lane & 7;
        constexpr int kPer = 512 / (32 * CT_SPLIT_WARPS);   // 16-B chunks per thread per stage
        if (cw < CT_SPLIT_WARPS) {
            int rslot = 0, mslot = 0;
            uint32_t rph = 0, mph = 0;
            for (int kb = 0; kb < num_kb; kb++) {
                mbar_wait(&rfull[rslot], rph);
                CT_TRACE_LANE(2, kb);
                float4 v[kPer];
#pragma unroll
                for (int i = 0; i < kPer; i++) {
                    const int q = cw * 32 + 32 * CT_SPLIT_WARPS * i;   // + lane
                    const int j = q >> 7, h = (q >> 5) & 3;
                    const int shift = gtab[kb * 4 + j].w;              // warp-uniform
                    const uint32_t ra = rbase + (uint32_t)(rslot * CT_RAW_STAGE + j * CT_RAW_GROUP +
                                                           ((h * 4 + c) * CT_RAW_W + 4 * wq) * 4);
                    const float4 a = lds4(ra);
                    if (shift == 0) {
                        v[i] = a;
                    } else {
                        const float4 b = lds4(ra + 16);
                        v[i] = shift == 1   ? make_float4(a.y, a.z, a.w, b.x)
                               : shift == 2 ? make_float4(a.z, a.w, b.x, b.y)
                                            : make_float4(a.w, b.x, b.y, b.z);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&rempty[rslot]);   // raw slot free once read
                mbar_wait(&empty[mslot], mph ^ 1);
                CT_TRACE_LANE(3, kb);
                const uint32_t mb = sbase + (uint32_t)(mslot * CT_MSTAGE);
#pragma unroll
                for (int i = 0; i < kPer; i++) {
                    if (p.dbg & 2) break;
                    const int q = cw * 32 + 32 * CT_SPLIT_WARPS * i;
                    const int j = q >> 7, h = (q >> 5) & 3;
                    const uint32_t off =
                        (uint32_t)(j * 2048 + h * 512 + c * 128 + (((wq >> 1) ^ c) << 5) + (wq & 1) * 16);
                    split4_store(mb + off, mb + CT_TILE_A + off, v[i].x, v[i].y, v[i].z, v[i].w);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[mslot]);
                CT_TRACE_LANE(4, kb);
                if (++rslot == CT_RSTAGES) {
                    rslot = 0;
                    rph ^= 1;
                }
                if (++mslot == CT_MSTAGES) {
                    mslot = 0;
                    mph ^= 1;
                }
            }
        }

        // ---------------- epilogue: TMEM (chunk accumulators) -> fp32 sum
        mbar_wait(tdone, 0);
        CT_TRACE_LANE(5, 0);
        tc_fence_after();
        float *tile = reinterpret_cast<float *>(smem);   // [CT_BN][128], operand stages retired
        {
            // all eight warps drain: quadrant = warp % 4 (the TMEM lanes this
            // warp may read), half = which 32 of the 64 channel columns; per
            // 16 columns the loads of every chunk are issued before one wait
            const int qd = warp & 3, half = cw >> 2;
            const int row = qd * 32 + lane;
            const int nch = (num_kb + p.stages_per_chunk - 1) / p.stages_per_chunk;
#pragma unroll
            for (int part = 0; part < 2; part++) {
                const int col = half * 32 + part * 16;
                uint32_t r[CT_CHUNKS][2][16];
#pragma unroll
                for (int ch = 0; ch < CT_CHUNKS; ch++)
                    if (ch < nch) {
                        const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ch * CT_ACC_COLS + col);
                        tmem_ld16_issue(ta, r[ch][0]);
                        tmem_ld16_issue(ta + CT_BN, r[ch][1]);
                    }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    float acc = __uint_as_float(r[0][0][i]) + __uint_as_float(r[0][1][i]);
#pragma unroll
                    for (int ch = 1; ch < CT_CHUNKS; ch++)
                        if (ch < nch) acc += __uint_as_float(r[ch][0][i]) + __uint_as_float(r[ch][1][i]);
                    tile[(col + i) * 128 + row] = acc;
                }
            }
        }
        CT_TRACE_LANE(5, 3);
        tc_fence_before();
        asm volatile("bar.sync 1, %0;" ::"r"(CT_CONV_WARPS * 32) : "memory");
        CT_TRACE_LANE(5, 4);
        // store: warp cw writes channels cw, cw+8, ...; lanes run along the 32 columns
        const int wo = w0 + lane;
        for (int co_l = cw; co_l < CT_BN; co_l += CT_CONV_WARPS) {
            const int64_t co = c0 + co_l;
            if (co >= p.CO) break;
            float *orow = p.o + n * p.so[0] + co * p.so[1] + wo * p.so[3];
#pragma unroll
            for (int h = 0; h < 4; h++) {
                const int ho = h0 + h;
                if (ho >= p.HO || wo >= p.WO) continue;
                float v = tile[co_l * 128 + h * 32 + lane];
                if (p.epi.n) v = apply_epilogue(p.epi, v, n, co, ho, wo);
                orow[(int64_t)ho * p.so[2]] = v;
            }
        }
    }
    if (warp == 3 && lane == 0) CT_TRACE(5, 5);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) CT_TRACE(5, 1);
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CT_CHUNKS * CT_ACC_COLS));
    }
}

}  // namespace tc
}  // namespace lsb
