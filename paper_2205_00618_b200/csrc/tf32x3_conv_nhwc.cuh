// tf32x3_conv_nhwc.cuh -- NCHW direct convolution on the tensor cores through
// an NHWC hi/lo copy of the input: implicit GEMM D[pixel][co] = Σ_(r,s,c)
// X[pixel, tap] W[co, tap] in split-TF32 (Xhi.Whi + Xhi.Wlo + Xlo.Whi).
//
// Prepass (nchw_split_nhwc_kernel): X (any strides) -> Xs[N][H][W][Cp/16][32]:
// per pixel and 16-channel block the 16 tf32 hi values then the 16 lo values
// (channels zero padded to Cp = 16k).  With channels innermost a {32, 1 block,
// 32 columns, 4 rows} box is exactly a K-major SWIZZLE_128B UMMA operand
// (128 pixel rows of 128 B: hi at bytes 0-63, lo at 64-127; one TMA request
// stream per stage instead of two 64-B-row boxes), and the tap's (r, s) shift lands on
// non-innermost TMA coordinates, which may be any integer (out of range ->
// zero fill = the conv padding; stride via TMA element strides).  So the
// mainloop is the GEMM kernel's: no converter warps, no proxy fence, every
// operand byte moved by TMA.
//   warp 0      TMA: Xhi box, Xlo box, one 8 KiB bulk copy of the stage's
//               filter image (hi | lo, tf32x3_conv_tma.cuh:filter_image_kernel)
//   warp 1      TMEM allocator + tcgen05.mma issuer: N=128 (Xhi x [Whi|Wlo])
//               + N=64 (Xlo x Whi) per 8 taps
//   warps 2-9   epilogue: TMEM -> fp32 sum of the two accumulators of both
//               K halves -> smem [co][pixel] -> NCHW stores (fused stages)
// Tile: 4 output rows x 32 output columns of one image (M = 128), 64 channels.
#pragma once

#include "conv_common.cuh"

namespace lsb {
namespace tc {

constexpr int CN_BN = 64;
constexpr int CN_BK = 16;                 // channels per stage (one (r, s) tap)
constexpr int CN_STAGES = 4;   // even: slots are released in pairs
constexpr int CN_EPI_WARPS = 8;
constexpr int CN_THREADS = 64 + 32 * CN_EPI_WARPS;   // 320
constexpr int CN_CHUNKS = 2;
constexpr int CN_ACC_COLS = 2 * CN_BN;
constexpr int CN_TILE_A = 128 * CN_BK * 4;           // 8 KiB (one of hi / lo)
constexpr int CN_TILE_B = 2 * CN_BN * CN_BK * 4;     // 8 KiB (hi | lo)
constexpr int CN_STAGE = 2 * CN_TILE_A + CN_TILE_B;  // 24 KiB
constexpr size_t CN_SMEM = (size_t)CN_STAGES * CN_STAGE + 256 + 1024;
static_assert(CN_STAGES * CN_STAGE >= CN_BN * 128 * 4, "epilogue staging reuses the stages");

struct ConvNhwcArgs {
    int64_t Cp, R, S, HO, WO, ph, pw, dh, dw, sh, sw;
    int64_t tiles_h, tiles_w, CO;
    const float *wimg;
    float *o;
    int64_t so[4];
    int stages_per_chunk;
    int vec4;             // float4 output stores (see the epilogue)
    // non-finite inputs (flagged by the prepasses: *anyflag == gen): the
    // tile is recomputed in FP32 from the original X and W in the epilogue
    // (3xTF32 would turn inf x (lo = 0) into NaN)
    const int *anyflag;
    int gen;
    const float *x, *w;
    int64_t C, H, W, sx[4], swt[4];
    EpiStages epi;
    long long *trace;     // debug (LSB_CN_TRACE builds): per-stage clock64 stamps of CTA 0
};

#ifdef LSB_CN_TRACE
#define CN_TRACE(ev, kb)                                                                          \
    do {                                                                                          \
        if (p.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && (kb) < 64)               \
            p.trace[(ev) * 64 + (kb)] = clock64();                                                \
    } while (0)
#else
#define CN_TRACE(ev, kb) \
    do {                 \
    } while (0)
#endif

__device__ __forceinline__ void tma_load_5d(const CUtensorMap *map, uint64_t *bar, void *dst, int c0, int c1, int c2,
                                            int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}

// X[n][c][h][w] (element strides sx*) -> hi/lo [n][h][w][Cp], channels >= C
// zero; 32 x 32 (w, c) tiles through smem so both sides are coalesced
__global__ void __launch_bounds__(256) nchw_split_nhwc_kernel(const float *__restrict__ x, int64_t C, int64_t H,
                                                              int64_t W, int64_t Cp, int64_t sx0, int64_t sx1,
                                                              int64_t sx2, int64_t sx3, float *__restrict__ hi,
                                                              float *__restrict__ lo, int *__restrict__ any,
                                                              int gen) {
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ float tile[32][33];
    const int64_t nh = blockIdx.z;   // n * H + h
    const int64_t n = nh / H, h = nh % H;
    const int64_t w0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int cc = ty + 8 * j;
        const int64_t c = c0 + cc, w = w0 + tx;
        tile[cc][tx] = (c < C && w < W) ? __ldg(x + n * sx0 + c * sx1 + h * sx2 + w * sx3) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int ww = ty + 8 * j;
        const int64_t w = w0 + ww, c = c0 + tx;
        if (w < W && c < Cp) {
            const float v = tile[tx][ww];
            const float vh = rna_tf32(v);
            const int64_t o = (((nh * W) + w) * (Cp / 16) + (c >> 4)) * 32 + (c & 15);
            hi[o] = vh;
            hi[o + 16] = tf32_lo(v, vh);
            if (!(fabsf(v) < __int_as_float(0x7f800000))) *any = gen;
        }
    }
}

// Vectorised form (W % 4 == 0, unit w stride, sx1/sx2/sx0 multiples of 4,
// 16-B aligned x, 32-bit indices): float4 reads along w, float4 writes along c
// kRows input rows per block: their kRows float4 loads are in flight
// together (one row per block left the transpose latency-bound at ~2x the
// copy time)
constexpr int kSplitRows = 4;
// Blocks with blockIdx.z >= zsplit build the filter stage images instead
// (one launch for both prepasses; they run side by side).
__global__ void __launch_bounds__(256) nchw_split_nhwc_vec_kernel(const float *__restrict__ x, int C, int H, int W,
                                                                  int Cp, int sx0, int sx1, int sx2,
                                                                  float *__restrict__ hi, float *__restrict__ lo,
                                                                  int *__restrict__ any, int gen,
                                                                  const FilterImgArgs f, int zsplit) {
    asm volatile("griddepcontrol.launch_dependents;");
    if ((int)blockIdx.z >= zsplit) {
        const int b = ((blockIdx.z - zsplit) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        const int nb = (gridDim.z - zsplit) * gridDim.y * gridDim.x;
        filter_image_body(f, any, gen, b * blockDim.x + threadIdx.x, nb * blockDim.x);
        return;
    }
    __shared__ float tile[kSplitRows][32][33];   // [row][c][w]
    const int hblocks = (H + kSplitRows - 1) / kSplitRows;
    const int n = blockIdx.z / hblocks, hb = (blockIdx.z - n * hblocks) * kSplitRows;
    const int w0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    const int t = threadIdx.x;
    {
        const int cc = t >> 3, w4 = (t & 7) * 4;
        const int c = c0 + cc, w = w0 + w4;
        float4 v[kSplitRows];
#pragma unroll
        for (int q = 0; q < kSplitRows; q++) {
            v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < C && w < W && hb + q < H)
                v[q] = __ldg(reinterpret_cast<const float4 *>(x + n * sx0 + c * sx1 + (hb + q) * sx2 + w));
        }
#pragma unroll
        for (int q = 0; q < kSplitRows; q++) {
            tile[q][cc][w4] = v[q].x;
            tile[q][cc][w4 + 1] = v[q].y;
            tile[q][cc][w4 + 2] = v[q].z;
            tile[q][cc][w4 + 3] = v[q].w;
        }
    }
    __syncthreads();
    const int ww = t >> 3, c4 = (t & 7) * 4;
    const int w = w0 + ww, c = c0 + c4;
    const float inf = __int_as_float(0x7f800000);
    bool bad = false;
#pragma unroll
    for (int q = 0; q < kSplitRows; q++) {
        if (w < W && c < Cp && hb + q < H) {
            const float4 v =
                make_float4(tile[q][c4][ww], tile[q][c4 + 1][ww], tile[q][c4 + 2][ww], tile[q][c4 + 3][ww]);
            const float4 vh = make_float4(rna_tf32(v.x), rna_tf32(v.y), rna_tf32(v.z), rna_tf32(v.w));
            const int64_t nh = (int64_t)n * H + hb + q;
            const int64_t o = ((nh * W + w) * (Cp / 16) + (c >> 4)) * 32 + (c & 15);
            *reinterpret_cast<float4 *>(hi + o) = vh;
            *reinterpret_cast<float4 *>(hi + o + 16) =
                make_float4(tf32_lo(v.x, vh.x), tf32_lo(v.y, vh.y), tf32_lo(v.z, vh.z), tf32_lo(v.w, vh.w));
            bad |= !(fabsf(v.x) < inf && fabsf(v.y) < inf && fabsf(v.z) < inf && fabsf(v.w) < inf);
        }
    }
    if (bad) *any = gen;
}

// grid: x = image * tiles_h * tiles_w output tiles, y = channel tiles
__global__ void __launch_bounds__(CN_THREADS, 2)
    tf32x3_conv_nhwc_kernel(const __grid_constant__ CUtensorMap map_xs, const ConvNhwcArgs p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + CN_STAGES * CN_STAGE);
    uint64_t *empty = full + CN_STAGES;
    uint64_t *tdone = empty + CN_STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tdone + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t t = blockIdx.x;
    const int tw = (int)(t % p.tiles_w);
    t /= p.tiles_w;
    const int th = (int)(t % p.tiles_h);
    const int n = (int)(t / p.tiles_h);
    const int h0 = th * 4, w0 = tw * 32;
    const int64_t c0 = (int64_t)blockIdx.y * CN_BN;
    const int cblocks = (int)(p.Cp / CN_BK);
    const int num_kb = (int)(p.R * p.S) * cblocks;
    if (threadIdx.x == 0) CN_TRACE(2, 2);
#ifdef LSB_CN_TRACE
    long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map_xs);
        for (int s = 0; s < CN_STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tdone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(CN_CHUNKS * CN_ACC_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            // launched with programmatic stream serialization: everything above
            // overlapped the prepasses; their outputs are read from here on
            asm volatile("griddepcontrol.wait;" ::: "memory");
            const int hin0 = (int)(h0 * p.sh - p.ph), win0 = (int)(w0 * p.sw - p.pw);
            int stage = 0;
            uint32_t phase = 0;
            int cb = 0, s = 0, r = 0;
            for (int kb = 0; kb < num_kb; kb++) {
                mbar_wait(&empty[stage | 1], phase ^ 1);   // slot pairs released together
                CN_TRACE(0, kb);
                unsigned char *base = smem + stage * CN_STAGE;
                mbar_expect_tx(&full[stage], CN_STAGE);
                const int hi_ = hin0 + r * (int)p.dh, wi = win0 + s * (int)p.dw;
                tma_load_5d(&map_xs, &full[stage], base, 0, cb, wi, hi_, n);   // [pixel][hi16 | lo16]
                bulk_load(base + 2 * CN_TILE_A, p.wimg + ((int64_t)blockIdx.y * num_kb + kb) * (2 * CN_BN * CN_BK),
                          CN_TILE_B, &full[stage]);
                if (++cb == cblocks) {
                    cb = 0;
                    if (++s == p.S) {
                        s = 0;
                        ++r;
                    }
                }
                if (++stage == CN_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (A and B K-major SWIZZLE_64B)
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(128, CN_BN);
            constexpr uint32_t idesc_n128 = idesc_tf32(128, 2 * CN_BN);
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = 0; kb < num_kb; kb++) {
                mbar_wait(&full[stage], phase);
                CN_TRACE(1, kb);
                tc_fence_after();
                const int chunk = kb / p.stages_per_chunk;
                const uint32_t d = tmem + (uint32_t)(chunk * CN_ACC_COLS);
                const uint32_t base = smem_u32(smem + stage * CN_STAGE);
                const uint64_t ahi = sdesc_k_sw<128>(base), alo = ahi + (uint64_t)(64 >> 4);   // lo: bytes 64-127
                const uint64_t bhi = sdesc_k_sw<64>(base + 2 * CN_TILE_A);
#pragma unroll
                for (int k = 0; k < CN_BK / 8; k++) {
                    const uint64_t off = (uint64_t)((k * 32) >> 4);
                    const uint32_t first = (kb % p.stages_per_chunk == 0 && k == 0) ? 0u : 1u;
                    umma_tf32(d, ahi + off, bhi + off, idesc_n128, first);
                    umma_tf32(d, alo + off, bhi + off, idesc, 1u);
                }
                // one commit per two stages frees a slot pair (a commit costs
                // ~45 cycles of tensor-pipe time against ~264 of MMAs per stage)
                if (stage & 1) umma_commit(&empty[stage]);
                if (++stage == CN_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            umma_commit(tdone);
        }
    } else {
        // ---------------- epilogue (warps 2..9)
        const int ew = warp - 2;
        asm volatile("griddepcontrol.wait;" ::: "memory");   // anyflag below is a prepass output
        mbar_wait(tdone, 0);
        if (ew == 0 && lane == 0) CN_TRACE(2, 0);
        tc_fence_after();
        float *tile = reinterpret_cast<float *>(smem);   // [CN_BN][128]
        {
            const int qd = warp & 3, half = ew >> 2;
            const int row = qd * 32 + lane;
            const int nch = (num_kb + p.stages_per_chunk - 1) / p.stages_per_chunk;
#pragma unroll
            for (int part = 0; part < 2; part++) {
                const int col = half * 32 + part * 16;
                uint32_t rr[CN_CHUNKS][2][16];
#pragma unroll
                for (int ch = 0; ch < CN_CHUNKS; ch++)
                    if (ch < nch) {
                        const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ch * CN_ACC_COLS + col);
                        tmem_ld16_issue(ta, rr[ch][0]);
                        tmem_ld16_issue(ta + CN_BN, rr[ch][1]);
                    }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    float acc = __uint_as_float(rr[0][0][i]) + __uint_as_float(rr[0][1][i]);
#pragma unroll
                    for (int ch = 1; ch < CN_CHUNKS; ch++)
                        if (ch < nch) acc += __uint_as_float(rr[ch][0][i]) + __uint_as_float(rr[ch][1][i]);
                    tile[(col + i) * 128 + row] = acc;
                }
            }
        }
        if (ew == 0 && lane == 0) CN_TRACE(2, 3);
        tc_fence_before();
        asm volatile("bar.sync 1, %0;" ::"r"(CN_EPI_WARPS * 32) : "memory");
        if (ew == 0 && lane == 0) CN_TRACE(2, 4);
        if (*p.anyflag == p.gen) {
            // non-finite input somewhere: FP32 recompute of this tile's outputs
            asm volatile("bar.sync 1, %0;" ::"r"(CN_EPI_WARPS * 32) : "memory");
            for (int i = threadIdx.x - 64; i < CN_BN * 128; i += CN_EPI_WARPS * 32) {
                const int co_l = i / 128, pix = i % 128, ho = h0 + pix / 32, wo = w0 + pix % 32;
                const int64_t co = c0 + co_l;
                if (co >= p.CO || ho >= p.HO || wo >= p.WO) continue;
                float acc = 0.0f;
                // out-of-range taps contribute fill (0) x w, as the reference's
                // guarded view does: inf x 0 = NaN must appear there too
                for (int64_t c = 0; c < p.C; c++)
                    for (int64_t r = 0; r < p.R; r++) {
                        const int64_t hi_ = ho * p.sh - p.ph + r * p.dh;
                        for (int64_t s2 = 0; s2 < p.S; s2++) {
                            const int64_t wi = wo * p.sw - p.pw + s2 * p.dw;
                            const bool in = hi_ >= 0 && hi_ < p.H && wi >= 0 && wi < p.W;
                            const float xv = in ? p.x[n * p.sx[0] + c * p.sx[1] + hi_ * p.sx[2] + wi * p.sx[3]] : 0.0f;
                            acc = fmaf(xv, p.w[co * p.swt[0] + c * p.swt[1] + r * p.swt[2] + s2 * p.swt[3]], acc);
                        }
                    }
                tile[co_l * 128 + pix] = acc;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(CN_EPI_WARPS * 32) : "memory");
        }
        if (p.vec4) {
            // one float4 per lane: lane -> output row h = lane / 8, columns
            // w0 + 4 (lane % 8) .. +3; a warp stores one channel's 4 x 32 tile
            // (WO % 4 == 0, unit column stride, 16-B aligned rows)
            const int h = lane >> 3, w4 = (lane & 7) * 4;
            const int ho = h0 + h, wo = w0 + w4;
            const bool ok = ho < p.HO && wo < p.WO;
            for (int co_l = ew; co_l < CN_BN; co_l += CN_EPI_WARPS) {
                const int64_t co = c0 + co_l;
                if (co >= p.CO) break;
                float4 v = *reinterpret_cast<const float4 *>(&tile[co_l * 128 + h * 32 + w4]);
                if (p.epi.n) {
                    v.x = apply_epilogue(p.epi, v.x, n, co, ho, wo);
                    v.y = apply_epilogue(p.epi, v.y, n, co, ho, wo + 1);
                    v.z = apply_epilogue(p.epi, v.z, n, co, ho, wo + 2);
                    v.w = apply_epilogue(p.epi, v.w, n, co, ho, wo + 3);
                }
                if (ok)
                    *reinterpret_cast<float4 *>(p.o + n * p.so[0] + co * p.so[1] + (int64_t)ho * p.so[2] + wo) = v;
            }
        } else {
            const int wo = w0 + lane;
            for (int co_l = ew; co_l < CN_BN; co_l += CN_EPI_WARPS) {
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
        if (ew == 0 && lane == 0) CN_TRACE(2, 5);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) CN_TRACE(2, 1);
#ifdef LSB_CN_TRACE
    if (threadIdx.x == 0 && p.trace != nullptr) {
        long long t_end;
        unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long *c = p.trace + 3 * 64 + 3 * (blockIdx.x + gridDim.x * blockIdx.y);
        c[0] = t_start; c[1] = t_end; c[2] = smid;
    }
#endif
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CN_CHUNKS * CN_ACC_COLS));
    }
}

}  // namespace tc
}  // namespace lsb
