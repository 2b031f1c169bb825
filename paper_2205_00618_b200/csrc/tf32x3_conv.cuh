// tf32x3_conv.cuh -- NCHW direct convolution on the 5th-gen tensor cores with
// an in-kernel im2col: implicit GEMM  D[pixel][co] = Σ_(c,r,s) X[pixel, tap] W[co, tap]
// in split-TF32 (Xhi.Whi + Xhi.Wlo + Xlo.Whi), fp32-accurate like the GEMM path.
//
// The materialised-im2col variant (tf32x3_conv in kern_tf32.cu) wrote 8*P*K
// bytes and lost to the SIMT kernel; here the im2col tile never leaves the SM:
//   warp 0      TMA of the pre-split filter tiles (Whi, Wlo: [CO][Kp], tiny)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (128 x CO_TILE x 8)
//   warps 2-9   converters: gather 128 pixels x 16 taps of X straight from HBM/L2
//               (per-CTA smem tap table, guards -> zero), split into tf32 hi/lo
//               and store them as an MN-major (pixel-contiguous) SW128_32B
//               operand -- each lane owns 4 consecutive output pixels, so one
//               tap costs one guard/address computation, 4 scalar loads and
//               one 16-B store per half -- then fence.proxy.async + mbarrier
//               arrive; after the mainloop warps 2-5 drain TMEM and all eight
//               store the tile (smem-transposed, pixel-contiguous NCHW writes,
//               fused epilogue)
// Accumulation: the K range is cut into CV_CHUNKS TMEM buffers (fresh
// accumulators, summed in fp32 by the epilogue) so the tensor core's truncating
// accumulate never runs over more than K/4 taps (see tf32x3_gemm.cuh).
#pragma once

#include "tf32x3_gemm.cuh"

namespace lsb {
namespace tc {

constexpr int CV_BM = 128;          // output pixels per tile (UMMA M)
constexpr int CV_BN = 64;           // output channels per tile (UMMA N)
constexpr int CV_BK = 16;           // taps per stage (two 8-tap UMMA K groups)
constexpr int CV_STAGES = 4;
constexpr int CV_CONV_WARPS = 8;    // 2 taps of the stage each
constexpr int CV_THREADS = 64 + 32 * CV_CONV_WARPS;
constexpr int CV_CHUNKS = 4;        // TMEM accumulators (4 x 64 = 256 columns: 2 CTAs / SM)
constexpr int CV_TILE_A = CV_BM * CV_BK * 4;            // 8 KiB: [4-tap group 4][m atom 4][4 taps][32 px]
constexpr int CV_TILE_B = CV_BN * CV_BK * 4;            // 4 KiB: K-major SWIZZLE_64B (TMA)
constexpr int CV_STAGE_BYTES = 2 * (CV_TILE_A + CV_TILE_B);
constexpr int CV_MAX_K = 1024;      // longer reductions stay on the SIMT kernel
// stages | barriers (256 B) | tap table (16 B per tap), plus 1 KiB for the
// 1024-B alignment of the swizzled tiles.  Kp <= 960 keeps two CTAs per SM.
__host__ __device__ constexpr size_t cv_smem_bytes(int64_t Kp) {
    return (size_t)CV_STAGES * CV_STAGE_BYTES + 256 + (size_t)Kp * 16 + 1024;
}
static_assert(CV_STAGES * CV_STAGE_BYTES >= CV_BN * CV_BM * 4, "epilogue staging reuses the stages");

struct ConvTcArgs {
    ConvGeom g;           // input geometry (P = images * HO * WO, K = C*R*S, Kp padded to 32)
    int64_t CO;
    float *o;
    int64_t so[4];        // n, co, h, w
    int stages_per_chunk;
    EpiStages epi;
    long long *trace;     // debug: per-stage clock64 stamps of CTA 0 (null = off)
};

#define CV_TRACE(ev, kb)                                                              \
    do {                                                                              \
        if (p.trace != nullptr && blockIdx.x == 0 && (kb) < 64) p.trace[(ev) * 64 + (kb)] = clock64(); \
    } while (0)

// MN-major tf32 operand in the SWIZZLE_128B_BASE32B canonical layout (the
// only MN-major layout the tensor core takes for 32-bit types): atoms of
// 4 taps x 32 pixels (128-B rows, 32-B granules XORed with the row), the
// 32-pixel atoms 512 B apart (LBO), the 4-tap groups 2 KiB apart (SBO); one
// 8-tap UMMA K step spans two groups.  Layout of the 8 KiB A tile:
//   byte(m, k) = (k/4)*2048 + (m/32)*512 + (k%4)*128 + ((((m%32)/8) ^ (k%4)) * 32) + (m%8)*4
__device__ __forceinline__ uint64_t sdesc_mn_sw128_32b(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)(512 >> 4) << 16;           // leading byte offset: next 32-pixel atom
    d |= (uint64_t)(2048 >> 4) << 32;          // stride byte offset: next 4-tap group
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;                    // SWIZZLE_128B_BASE32B
    return d;
}

// 3xTF32 split for the gather: hi = x rounded to nearest (ties away) on the
// 10-bit tf32 mantissa (the integer form of cvt.rna.tf32.f32, 2 instructions
// instead of the 5 the cvt lowers to on sm_100; a NaN whose payload sits in
// the dropped bits becomes inf in hi, but lo stays NaN so products do too),
// lo = x - hi exactly; the tensor core drops lo's low 13 bits (a 2^-22
// relative effect on lo, i.e. below fp32 resolution of x).  Infinite hi gets
// lo = 0 so inf inputs give inf, not inf - inf = NaN.
__device__ __forceinline__ float split_hi(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ float split_lo(float x, float hi) {
    return fabsf(hi) == __int_as_float(0x7f800000) ? 0.0f : x - hi;
}

// predicated read-only load, 0 when !ok (plain PTX predication: the C++
// ternary on __ldg made ptxas rebuild the memory descriptor per load)
__device__ __forceinline__ float ldg_or_zero(const float *p, uint32_t ok) {
    float v;
    // volatile: keeps the load where the software pipeline issues it (a
    // plain asm/__ldg gets sunk next to its first use under register pressure)
    asm volatile("{\n\t.reg .pred q;\n\t"
        "setp.ne.u32 q, %2, 0;\n\t"
        "mov.f32 %0, 0f00000000;\n\t"
        "@q ld.global.nc.f32 %0, [%1];\n\t}"
        : "=f"(v)
        : "l"(p), "r"(ok));
    return v;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// tmem_ld16: tf32x3_gemm.cuh

// grid: x = pixel tiles, y = channel tiles.  kRow4: every aligned group of 4
// output pixels lies in one output row (WO % 4 == 0) and steps 1 element
// along W (stride_w * sx3 == 1), so a lane's 4 taps share one row guard and
// one address; otherwise each pixel is guarded and addressed on its own.
template <bool kRow4>
__global__ void __launch_bounds__(CV_THREADS, 2)
    tf32x3_conv_kernel(const __grid_constant__ CUtensorMap map_whi, const __grid_constant__ CUtensorMap map_wlo,
                       const ConvTcArgs p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // align by offsetting smem_raw itself (not through an integer) so the
    // compiler keeps the shared address space: LDS/STS, not generic LD/ST
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + CV_STAGES * CV_STAGE_BYTES);
    uint64_t *empty = full + CV_STAGES;
    uint64_t *tdone = empty + CV_STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tdone + 1);
    int4 *taps = reinterpret_cast<int4 *>(smem + CV_STAGES * CV_STAGE_BYTES + 256);   // [Kp]

    const ConvGeom &g = p.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p0 = (int64_t)blockIdx.x * CV_BM;
    const int64_t c0 = (int64_t)blockIdx.y * CV_BN;
    const int num_kb = (int)(g.Kp / CV_BK);

    // tap table: k -> {input offset of (c, r*dil, s*dil), r*dil, s*dil}; the
    // host guarantees every in-range element offset fits in 31 bits
    const int64_t rs = g.R * g.S;
    for (int64_t k = threadIdx.x; k < g.Kp; k += CV_THREADS) {
        if (k < g.K) {
            const int64_t c = k / rs, r = (k % rs) / g.S, s = k % g.S;
            const int rr = (int)(r * g.dh), ss = (int)(s * g.dw);
            taps[k] = make_int4((int)(c * g.sx1 + (int64_t)rr * g.sx2 + (int64_t)ss * g.sx3), rr, ss, 0);
        } else {
            taps[k] = make_int4(0, 1 << 28, 1 << 28, 0);   // padded taps: always out of range -> 0
        }
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_whi);
        tma_prefetch_desc(&map_wlo);
        for (int s = 0; s < CV_STAGES; s++) {
            mbar_init(&full[s], 1 + CV_CONV_WARPS);   // TMA arrive_expect_tx + one per converter warp
            mbar_init(&empty[s], 1);
        }
        mbar_init(tdone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(CV_CHUNKS * CV_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA: filter hi/lo tiles [CV_BN co][CV_BK taps]
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = 0; kb < num_kb; kb++) {
                mbar_wait_sleep(&empty[stage], phase ^ 1);
                CV_TRACE(0, kb);
                unsigned char *base = smem + stage * CV_STAGE_BYTES;
                mbar_expect_tx(&full[stage], 2 * CV_TILE_B);
                tma_load_2d(&map_whi, &full[stage], base + 2 * CV_TILE_A, kb * CV_BK, (int)c0);
                tma_load_2d(&map_wlo, &full[stage], base + 2 * CV_TILE_A + CV_TILE_B, kb * CV_BK, (int)c0);
                if (++stage == CV_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (A: MN-major SW128, B: K-major SW64)
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(CV_BM, CV_BN) | (1u << 15);   // A MN-major
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = 0; kb < num_kb; kb++) {
                mbar_wait_sleep(&full[stage], phase);
                CV_TRACE(1, kb);
                tc_fence_after();
                const int chunk = kb / p.stages_per_chunk;
                const uint32_t d = tmem + (uint32_t)(chunk * CV_BN);
                const uint32_t base = smem_u32(smem + stage * CV_STAGE_BYTES);
                const uint64_t ahi = sdesc_mn_sw128_32b(base), alo = sdesc_mn_sw128_32b(base + CV_TILE_A);
                const uint64_t bhi = sdesc_k_sw<64>(base + 2 * CV_TILE_A);
                const uint64_t blo = sdesc_k_sw<64>(base + 2 * CV_TILE_A + CV_TILE_B);
#pragma unroll
                for (int k = 0; k < CV_BK / 8; k++) {
                    const uint64_t aoff = (uint64_t)((k * 4096) >> 4);   // next two 4-tap groups
                    const uint64_t boff = (uint64_t)((k * 32) >> 4);     // 8 taps along the 64-B row
                    const uint32_t first = (kb % p.stages_per_chunk == 0 && k == 0) ? 0u : 1u;
                    umma_tf32(d, ahi + aoff, bhi + boff, idesc, first);
                    umma_tf32(d, ahi + aoff, blo + boff, idesc, 1u);
                    umma_tf32(d, alo + aoff, bhi + boff, idesc, 1u);
                }
                umma_commit(&empty[stage]);
                if (++stage == CV_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            umma_commit(tdone);
        }
    } else {
        // ---------------- converters (warps 2..9): im2col gather + tf32 split
        // warp cw handles taps 2cw, 2cw+1 of every stage; lane l owns output
        // pixels 4l .. 4l+3 of the tile (one 16-B chunk of an MN atom row)
        const int cw = warp - 2;
        const int64_t hw = g.HO * g.WO;
        const unsigned H = (unsigned)g.H, W = (unsigned)g.W;
        const float *x = g.x;
        int hb[4], wb[4], pb[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int64_t pix = p0 + 4 * lane + i;
            hb[i] = -(1 << 29);
            wb[i] = -(1 << 29);
            pb[i] = 0;
            if (pix < g.P) {
                const int64_t img = pix / hw, ho = (pix % hw) / g.WO, wo = pix % g.WO;
                hb[i] = (int)(ho * g.sh - g.ph);
                wb[i] = (int)(wo * g.sw - g.pw);
                pb[i] = (int)(img * g.sx0 + (int64_t)hb[i] * g.sx2 + (int64_t)wb[i] * g.sx3);
            }
        }
        // kRow4: bit d of wmask = column wb[0] + d is inside [0, W)
        uint32_t wmask = 0;
        if (kRow4) {
#pragma unroll 1
            for (int d = 0; d < 32; d++)
                if ((unsigned)(wb[0] + d) < W) wmask |= 1u << d;
        }
        // this lane's 16-B half-granule inside an atom row (tap row r = kk % 4)
        const uint32_t sbase = smem_u32(smem);
        const uint32_t lane_off = (uint32_t)((lane >> 3) * 512 + (lane & 1) * 16);
        auto chunk_off = [&](int kk) -> uint32_t {
            const int r = kk & 3;
            return (uint32_t)((kk >> 2) * 2048 + r * 128 + ((((lane & 7) >> 1) ^ r) << 5)) + lane_off;
        };
        const uint32_t off0 = chunk_off(2 * cw), off1 = chunk_off(2 * cw + 1);

        auto load = [&](int kb, float (&v)[8]) {
            if (lane == 0 && (cw == 0 || cw == 7)) CV_TRACE(2 + (cw ? 4 : 0), kb);
#pragma unroll
            for (int t2 = 0; t2 < 2; t2++) {
                const int4 t = taps[kb * CV_BK + 2 * cw + t2];
                if (kRow4) {
                    const uint32_t m = ((unsigned)(hb[0] + t.y) < H) ? (wmask >> t.z) : 0u;
                    const float *src = x + (pb[0] + t.x);
#pragma unroll
                    for (int i = 0; i < 4; i++) v[t2 * 4 + i] = ldg_or_zero(src + i, (m >> i) & 1u);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const bool ok = ((unsigned)(hb[i] + t.y) < H) & ((unsigned)(wb[i] + t.z) < W);
                        v[t2 * 4 + i] = ldg_or_zero(x + (pb[i] + t.x), ok);
                    }
                }
            }
        };
        auto store = [&](int kb, const float (&v)[8]) {
            const int slot = kb % CV_STAGES;
            float h[8], l[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                h[i] = split_hi(v[i]);
                l[i] = split_lo(v[i], h[i]);
            }
            if (lane == 0 && (cw == 0 || cw == 7)) CV_TRACE(3 + (cw ? 4 : 0), kb);
            mbar_wait_sleep(&empty[slot], (uint32_t)(((kb / CV_STAGES) & 1) ^ 1));
            if (lane == 0 && (cw == 0 || cw == 7)) CV_TRACE(4 + (cw ? 4 : 0), kb);
            const uint32_t sb = sbase + (uint32_t)(slot * CV_STAGE_BYTES);
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sb + off0), "f"(h[0]), "f"(h[1]),
                         "f"(h[2]), "f"(h[3]) : "memory");
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sb + off1), "f"(h[4]), "f"(h[5]),
                         "f"(h[6]), "f"(h[7]) : "memory");
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sb + CV_TILE_A + off0), "f"(l[0]),
                         "f"(l[1]), "f"(l[2]), "f"(l[3]) : "memory");
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sb + CV_TILE_A + off1), "f"(l[4]),
                         "f"(l[5]), "f"(l[6]), "f"(l[7]) : "memory");
            fence_proxy_async_smem();   // generic-proxy stores -> visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[slot]);
            if (lane == 0 && (cw == 0 || cw == 7)) CV_TRACE(5 + (cw ? 4 : 0), kb);
        };
        // software pipeline: the loads of stages kb+1 and kb+2 are in flight
        // while stage kb is split and stored
        float va[8], vb[8], vc[8];
        load(0, va);
        if (num_kb > 1) load(1, vb);
        for (int kb = 0; kb < num_kb; kb += 3) {
            if (kb + 2 < num_kb) load(kb + 2, vc);
            store(kb, va);
            if (kb + 1 < num_kb) {
                if (kb + 3 < num_kb) load(kb + 3, va);
                store(kb + 1, vb);
            }
            if (kb + 2 < num_kb) {
                if (kb + 4 < num_kb) load(kb + 4, vb);
                store(kb + 2, vc);
            }
        }

        // ---------------- epilogue: TMEM (4 chunk accumulators) -> fp32 sum
        mbar_wait_sleep(tdone, 0);
        if (lane == 0 && cw == 0) CV_TRACE(10, 0);
        tc_fence_after();
        float *tile = reinterpret_cast<float *>(smem);   // [CV_BN][CV_BM], all stages retired
        if (warp < 6) {
            const int q = warp & 3;                      // TMEM lane quadrant = pixel rows
            const int row = q * 32 + lane;
            float acc[CV_BN];
#pragma unroll
            for (int i = 0; i < CV_BN; i++) acc[i] = 0.0f;
#pragma unroll
            for (int c = 0; c < CV_CHUNKS; c++) {
                if (c * p.stages_per_chunk >= num_kb) break;
#pragma unroll
                for (int part = 0; part < CV_BN / 16; part++) {
                    float t[16];
                    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * CV_BN + part * 16), t);
#pragma unroll
                    for (int i = 0; i < 16; i++) acc[part * 16 + i] += t[i];
                }
            }
#pragma unroll
            for (int i = 0; i < CV_BN; i++) tile[i * CV_BM + row] = acc[i];
        }
        tc_fence_before();
        asm volatile("bar.sync 1, %0;" ::"r"(CV_CONV_WARPS * 32) : "memory");
        // store: warp w writes channels w, w+8, ...; lanes run along pixels
        int64_t obase[CV_BM / 32];
        int pimg[CV_BM / 32], pho[CV_BM / 32], pwo[CV_BM / 32];
#pragma unroll
        for (int e = 0; e < CV_BM / 32; e++) {
            const int64_t px = p0 + e * 32 + lane;
            const int64_t img = px / hw, ho = (px % hw) / g.WO, wo = px % g.WO;
            pimg[e] = (int)img;
            pho[e] = (int)ho;
            pwo[e] = (int)wo;
            obase[e] = px < g.P ? img * p.so[0] + ho * p.so[2] + wo * p.so[3] : -1;
        }
        for (int co_l = cw; co_l < CV_BN; co_l += CV_CONV_WARPS) {
            const int64_t co = c0 + co_l;
            if (co >= p.CO) break;
            float *orow = p.o + co * p.so[1];
#pragma unroll
            for (int e = 0; e < CV_BM / 32; e++) {
                if (obase[e] < 0) continue;
                float v = tile[co_l * CV_BM + e * 32 + lane];
                if (p.epi.n) v = apply_epilogue(p.epi, v, pimg[e], co, pho[e], pwo[e]);
                orow[obase[e]] = v;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CV_CHUNKS * CV_BN));
    }
}

}  // namespace tc
}  // namespace lsb
