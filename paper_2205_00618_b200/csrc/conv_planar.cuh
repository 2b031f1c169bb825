// conv_planar.cuh -- single-pass NCHW direct convolution on the tensor cores
// (split TF32), stride 1, any padding / dilation, zero fill.
//
// Per-image flat padded pixel space.  With Hp = HO + (R-1) dh, Wp = WO + (S-1)
// dw (the padded extent the taps reach; padded (hp, wp) = raw (hp - ph,
// wp - pw)), the output pixel (ho, wo) of an image is computed at the flat
// position F = ho Wp + wo of its padded grid, and its tap (r, s) reads the
// padded input at F + r dh Wp + s dw.  Over a tile of NT consecutive F every
// tap is therefore one contiguous run of NT rows of a "halo" of NT + (R-1) dh
// Wp + (S-1) dw rows: the implicit GEMM's B operand for tap (r, s) is the halo
// shifted by a row offset.  Tiles never cross images (tiles per image =
// ceil(HO Wp / NT)); positions with wo >= WO are computed and dropped.
//
// Raw X by TMA.  A job's halo (16 channels) spans at most `rb` padded rows of
// one image: one 4-D TMA box {wb columns from w = -(pw + wsh), rb rows from
// h = hp0 - ph, 16 channels, 1 image} of the ORIGINAL NCHW tensor lands in a
// raw smem slot as [c][row][wb]; everything outside the image (the padding,
// channels >= C) is the TMA's zero fill.  (The innermost start coordinate of a
// box must be 16-B aligned -- a start of -1 float faults with "illegal
// instruction", tools/tma_box_probe.cu -- hence the wsh extra columns.)  Two raw slots: the box of job k + 2 is
// issued as soon as job k is converted, so the HBM latency sits under the
// MMAs of the jobs in between.
//
// Planar operands.  Converter warps turn a raw slot into the halo as K-major
// SWIZZLE_NONE "planes": fp32 plane g (0-3) holds channels 4g..4g+3 of every
// halo row, bf16 plane 4 + g (g = 0, 1) the lo parts of channels 8g..8g+7,
// rows 16 B apart ([plane][row][16 B]), so core matrices (8 rows x 16 B) are
// contiguous for ANY start row: descriptor LBO = plane stride, SBO = 128 B,
// and the tap shift is just start + off * 16 B (verified on B200:
// tools/umma_planar_probe.cu; 128 cycles per 128x256x8 MMA, the same as the
// swizzled layouts).
//
// Split TF32 + a bf16 correction.  The tensor core truncates fp32 operands to
// tf32 (probe mode 1), so the raw value IS the hi part; lo = x - trunc(x) is
// exact in fp32.  Per 16-channel tap: two kind::tf32 MMAs (K = 8 each) with A
// = 128 rows, row 2c = W[c] (hi after truncation), row 2c+1 = W[c] - trunc(W[c])
// (lo), against raw X: row 2c accumulates Whi.Xhi, row 2c+1 Wlo.Xhi; and one
// kind::f16 MMA (K = 16) with A rows 2c = bf16(W[c]), 2c+1 = 0 against the
// halo's bf16(lo) planes: row 2c += W.Xlo.  The epilogue adds the row pair.
// The correction term is ~2^-11 of the product, so bf16's 8-bit mantissa
// leaves ~2^-19 relative error per product (3xTF32: ~2^-21; both far inside
// the 1e-4 relative rule).  Three MMAs per tap instead of 3xTF32's four
// (the 4th, lo.lo, was the price of the 2-row-per-channel stacking): 25 %
// fewer tensor cycles and shared-memory operand reads, which bound this kernel.
// The filter stage images come from a small prepass (cp_filter_kernel)
// launched just before this kernel with programmatic dependent launch: only
// the filter producer waits for it (griddepcontrol.wait), the raw X boxes and
// their conversion start at once.
//
// Stream-K.  Work units are (co tile, pixel tile, stage), stage = (16-channel
// block cb, tap); a persistent grid of at most one CTA per SM takes equal unit
// ranges.  A CTA's range is a sequence of segments (runs within one tile); a
// segment that does not hold the whole tile publishes fp32 partials to a
// per-CTA slot, counts in, and the LAST segment to count in sums all partials
// in segment order (deterministic) before the fused epilogue and the NCHW
// stores.  No CTA ever waits for another.
//
// Two-level accumulation.  TMEM holds two NT-column accumulators; each job
// (one halo = one cb of one segment, <= R*S taps = 144-channel K for 3x3)
// accumulates into one while the epilogue warps fold the other into fp32
// registers (round to nearest; the tensor core's accumulate truncates).
//
// Warp roles (448 threads, 1 CTA / SM):
//   warp 0      filter stages: cp.async.bulk of 8 KiB planar stage images
//               into a 3-slot ring of tap pairs; thread 0 also issues the
//               first two raw X boxes
//   warp 1      TMEM allocator + tcgen05.mma issuer
//   warps 2-5   halo converters: raw slot -> hi / lo planes, non-finite
//               flags; converter 0 issues the later raw X boxes
//   warps 6-13  epilogue: fold, hi/lo row-pair sum (shfl), per 32-column
//               part: smem transpose, publish / fixup, coalesced NCHW stores
#pragma once

#include <cuda_bf16.h>

#include "conv_common.cuh"

namespace lsb {
namespace tc {

constexpr int CP_HALO = 384;                       // halo rows per buffer
constexpr int CP_PLANE = CP_HALO * 16;             // bytes per 4-channel plane
constexpr int CP_HALO_BYTES = 6 * CP_PLANE;        // fp32 planes 0-3, bf16 lo planes 4-5: 36 KiB
constexpr int CP_RAW_BYTES = 28 * 1024;            // raw X slot: 16 channels x rb rows x wb floats
constexpr int CP_RAW_SLOTS = 2;
constexpr int CP_FSLOTS = 3;                       // filter ring slots, each a tap pair
constexpr int CP_FSTAGE = 6 * 128 * 16;            // 12 KiB per tap: 4 fp32 + 2 bf16 planes x 128 rows x 16 B
constexpr int CP_CONV_WARPS = 4;
constexpr int CP_EPI_WARPS = 8;
constexpr int CP_THREADS = 64 + 32 * (CP_CONV_WARPS + CP_EPI_WARPS);   // 448
constexpr int CP_STG_ROW = 36;                     // staged floats per channel row of a 32-column part
constexpr int CP_STG_WARP = 16 * CP_STG_ROW * 4;   // 2304 B per epilogue warp
constexpr int CP_OFF_RAW = 2 * CP_HALO_BYTES;
constexpr int CP_OFF_FRING = CP_OFF_RAW + CP_RAW_SLOTS * CP_RAW_BYTES;
constexpr int CP_OFF_STG = CP_OFF_FRING + 2 * CP_FSLOTS * CP_FSTAGE;
constexpr int CP_OFF_BAR = CP_OFF_STG + CP_EPI_WARPS * CP_STG_WARP;
constexpr size_t CP_SMEM = (size_t)CP_OFF_BAR + 256 + 1024;
static_assert(CP_SMEM <= 232448, "conv_planar shared memory");
static_assert(CP_RAW_BYTES % 1024 == 0 && CP_OFF_FRING % 1024 == 0, "TMA / bulk destinations stay aligned");

struct ConvPlanarArgs {
    const float *x;
    int64_t sx[4];                 // NCHW element strides
    int N, C, H, W, CO, R, S, HO, WO, ph, pw, dh, dw;
    int Hp, Wp, halo;              // padded grid, halo rows used (<= CP_HALO)
    int tpi;                       // pixel tiles per image: ceil(HO * Wp / NT)
    int rb, wb, wsh;               // raw X box: rows, columns (a multiple of 4) from w = -(pw + wsh)
                                   // (the TMA's innermost start must be 16-B aligned: pw + wsh = 4k)
    int tiles, co_tiles, cbs, stages;   // tiles = N * tpi; stages per tile = cbs * R * S
    int64_t units;                 // co_tiles * tiles * stages
    const float *wimg;             // [co_tile][stage][4 planes][128][4] (cp_filter_kernel)
    float *o;
    int64_t so[4];
    float *part;                   // [2 * cta][64][NT] published partial sums
    int *tilecnt;                  // [co_tile * tiles + tile] segments arrived (reset by the last)
    int *tileflag;                 // [co_tile * tiles + tile] == gen: non-finite X in the tile's halo
    int *wflag;                    // == gen: non-finite filter (set by cp_filter_kernel)
    int gen;
    const float *w;
    int64_t swt[4];
    EpiStages epi;
    long long *trace;              // debug (LSB_CONV_TRACE): [cta][64] clock64 / globaltimer stamps
    int dbg;                       // experiments (LSB_CP_DBG): 1 skip output stores, 4 skip MMAs
};

__device__ __forceinline__ void cp_stamp(const ConvPlanarArgs &p, int slot) {
    if (p.trace != nullptr && slot < 64) p.trace[blockIdx.x * 64 + slot] = clock64();
}
// finer stamps: [148 * 64 + cta * 128 + slot]
__device__ __forceinline__ void cp_stamp2(const ConvPlanarArgs &p, int slot) {
    if (p.trace != nullptr && slot < 128) p.trace[148 * 64 + blockIdx.x * 128 + slot] = clock64();
}

// planar filter stage images: stage (cb, tap) of co tile ct holds, for the 16
// channels cb*16.., fp32 rows 2c = W[ct*64 + c] (the hi part: the tensor core
// truncates) and 2c+1 = W - trunc(W), then bf16 rows 2c = bf16(W), 2c+1 = 0;
// channels >= C and filters >= CO are zero.  One thread per (stage, 4-channel
// group, filter) -- e = ((ct * stages + stage) * 4 + g) * 64 + co -- writing
// 16-B hi / lo rows and an 8-B bf16 row piece.
struct CpFilterArgs {
    const float *w;
    int64_t swt[4];
    int CO, C, R, S, stages, total;
    float *img;
    int *wflag;
    int gen;
};

__global__ void __launch_bounds__(256) cp_filter_kernel(const CpFilterArgs f) {
    asm volatile("griddepcontrol.launch_dependents;");
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= f.total) return;
    const float inf = __int_as_float(0x7f800000);
    const int co_l = e & 63, g = (e >> 6) & 3, ts = e >> 8;
    const int stage = ts % f.stages, ct = ts / f.stages;
    const int RS = f.R * f.S;
    const int cb = stage / RS, tap = stage - cb * RS;
    const int r = tap / f.S, s = tap - r * f.S;
    const int co = ct * 64 + co_l, c0 = cb * 16 + 4 * g;
    float v[4], lo[4];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        v[q] = (co < f.CO && c0 + q < f.C)
                   ? __ldg(f.w + co * f.swt[0] + (c0 + q) * f.swt[1] + r * f.swt[2] + s * f.swt[3])
                   : 0.0f;
        const bool fin = fabsf(v[q]) < inf;
        bad |= !fin;
        lo[q] = fin ? v[q] - __uint_as_float(__float_as_uint(v[q]) & 0xffffe000u) : 0.0f;
    }
    float *st = f.img + (int64_t)ts * (CP_FSTAGE / 4);
    *reinterpret_cast<float4 *>(st + g * 512 + (2 * co_l) * 4) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4 *>(st + g * 512 + (2 * co_l + 1) * 4) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    // bf16 planes (after the 4 fp32 planes): [8-channel plane][128 rows][8]
    __nv_bfloat16 *sb = reinterpret_cast<__nv_bfloat16 *>(st + 4 * 512) + (g >> 1) * 1024 + (g & 1) * 4;
    // (a non-finite filter value keeps hi = the value for the flag path; its
    // bf16 copy is 0 -- tiles are recomputed in FP32 when wflag is set)
    const __nv_bfloat162 b01 = __floats2bfloat162_rn(fabsf(v[0]) < inf ? v[0] : 0.0f, fabsf(v[1]) < inf ? v[1] : 0.0f);
    const __nv_bfloat162 b23 = __floats2bfloat162_rn(fabsf(v[2]) < inf ? v[2] : 0.0f, fabsf(v[3]) < inf ? v[3] : 0.0f);
    *reinterpret_cast<uint2 *>(sb + (2 * co_l) * 8) =
        make_uint2(*reinterpret_cast<const uint32_t *>(&b01), *reinterpret_cast<const uint32_t *>(&b23));
    *reinterpret_cast<uint2 *>(sb + (2 * co_l + 1) * 8) = make_uint2(0u, 0u);
    if (bad) *f.wflag = f.gen;
}

// output position of per-image flat column F (false: a dropped position)
__device__ __forceinline__ bool cp_pixel(const ConvPlanarArgs &p, int F, int &ho, int &wo) {
    ho = F / p.Wp;
    wo = F - ho * p.Wp;
    return ho < p.HO && wo < p.WO;
}

// one output point recomputed in FP32 (non-finite inputs: 3xTF32 would turn
// inf x 0 in a cross term into NaN); out-of-range taps contribute 0 x w like
// the guarded view
__device__ __noinline__ float cp_fp32_point(const ConvPlanarArgs &p, int n, int co, int ho, int wo) {
    float a = 0.0f;
    for (int c = 0; c < p.C; c++)
        for (int r = 0; r < p.R; r++) {
            const int hi_ = ho - p.ph + r * p.dh;
            for (int s = 0; s < p.S; s++) {
                const int wi = wo - p.pw + s * p.dw;
                const bool in = hi_ >= 0 && hi_ < p.H && wi >= 0 && wi < p.W;
                const float xv = in ? p.x[n * p.sx[0] + c * p.sx[1] + hi_ * p.sx[2] + wi * p.sx[3]] : 0.0f;
                a = fmaf(xv, p.w[co * p.swt[0] + c * p.swt[1] + r * p.swt[2] + s * p.swt[3]], a);
            }
        }
    return a;
}

// cold path: the lane's column of the warp's staged 16 x 32 block recomputed in FP32
__device__ __noinline__ void cp_recompute(const ConvPlanarArgs &p, float *stg, int n, int F0, int co0, int lane) {
    int ho, wo;
    if (!cp_pixel(p, F0 + lane, ho, wo)) return;
    for (int cr = 0; cr < 16 && co0 + cr < p.CO; cr++) stg[cr * CP_STG_ROW + lane] = cp_fp32_point(p, n, co0 + cr, ho, wo);
}

// fused epilogue stages applied in place to a lane's staged column (out of
// line: most convs have none)
__device__ __noinline__ void cp_epilogue_col(const ConvPlanarArgs &p, float *stg, int n, int F0, int co0, int lane) {
    int ho, wo;
    if (!cp_pixel(p, F0 + lane, ho, wo)) return;
    for (int cr = 0; cr < 16 && co0 + cr < p.CO; cr++)
        stg[cr * CP_STG_ROW + lane] = apply_epilogue(p.epi, stg[cr * CP_STG_ROW + lane], n, co0 + cr, ho, wo);
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ uint64_t desc_planar(uint32_t saddr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;   // K direction: plane stride
    d |= (uint64_t)(128u >> 4) << 32;              // M/N direction: 8 rows x 16 B
    d |= (uint64_t)1 << 46;                        // sm_100 descriptor; SWIZZLE_NONE
    return d;
}

__device__ __forceinline__ void tma_load_4d(const CUtensorMap *map, uint64_t *bar, void *dst, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// one job = the stages of one (co tile, tile, cb) inside this CTA's range
struct CpJob {
    int ct, tile, cb, t0, t1;      // taps [t0, t1)
    bool seg_last;                 // the job ends its segment
    bool head;                     // the segment starts at stage 0 of the tile
    bool complete;                 // the segment ends at the tile's last stage
    bool last;                     // the CTA's last job
    int tile_end;                  // first unit after the tile
};

// the jobs of a unit range in order.  Divisions only in init(): next()
// steps (co tile, tile, cb) incrementally (the per-job division chain cost
// ~0.5k cycles at every job boundary of every role)
struct CpIter {
    int u, ub, ue;                 // next unit; the range (units < 2^31, checked by the host)
    int ct, tile, cb, tap;         // position of unit u
    __device__ __forceinline__ void init(const ConvPlanarArgs &p, int64_t b, int64_t e) {
        ub = (int)b;
        ue = (int)e;
        u = ub;
        const int RS = p.R * p.S;
        const int tl = u / p.stages, st = u - tl * p.stages;
        cb = st / RS;
        tap = st - cb * RS;
        ct = tl / p.tiles;
        tile = tl - ct * p.tiles;
    }
    __device__ __forceinline__ bool next(const ConvPlanarArgs &p, CpJob &j) {
        if (u >= ue) return false;
        const int RS = p.R * p.S;
        const int tile_begin = (ct * p.tiles + tile) * p.stages;
        const int job_end = min(ue, tile_begin + (cb + 1) * RS);
        j.ct = ct;
        j.tile = tile;
        j.cb = cb;
        j.t0 = tap;
        j.t1 = tap + (job_end - u);
        j.tile_end = tile_begin + p.stages;
        j.seg_last = job_end == ue || job_end == j.tile_end;
        j.head = tile_begin >= ub;
        j.complete = j.tile_end <= ue;
        j.last = job_end == ue;
        u = job_end;
        tap = 0;
        if (++cb == p.cbs) {
            cb = 0;
            if (++tile == p.tiles) {
                tile = 0;
                ++ct;
            }
        }
        return true;
    }
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);   // .x = lo (lower address)
    return *reinterpret_cast<const uint32_t *>(&v);
}

// a share of a job's halo conversion: rows first, first + step, ... of the
// raw slot [c][row][wb] -> fp32 planes + bf16 lo planes; returns true on a
// non-finite value
__device__ __forceinline__ bool cp_convert(const ConvPlanarArgs &p, const float *raw, float *hb, int F0, int first,
                                           int step) {
    const float inf = __int_as_float(0x7f800000);
    const int cstride = p.rb * p.wb;   // raw floats per channel
    const int hp0 = F0 / p.Wp;
    bool bad = false;
    for (int row = first; row < p.halo; row += step) {
        const int F = F0 + row;
        const int hp = F / p.Wp, wp = F - hp * p.Wp;
        const float *src = raw + (hp - hp0) * p.wb + wp + p.wsh;
        uint32_t lo2[8];
#pragma unroll
        for (int g = 0; g < 4; g++) {
            float4 hv = make_float4(src[(4 * g) * cstride], src[(4 * g + 1) * cstride], src[(4 * g + 2) * cstride],
                                    src[(4 * g + 3) * cstride]);
            float4 lv;
            float *h4 = &hv.x, *l4 = &lv.x;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float x = h4[q];
                const bool fin = fabsf(x) < inf;
                bad |= !fin;
                l4[q] = fin ? x - __uint_as_float(__float_as_uint(x) & 0xffffe000u) : 0.0f;
            }
            *reinterpret_cast<float4 *>(hb + g * (CP_PLANE / 4) + row * 4) = hv;
            lo2[2 * g] = pack_bf16x2(lv.x, lv.y);
            lo2[2 * g + 1] = pack_bf16x2(lv.z, lv.w);
        }
        *reinterpret_cast<uint4 *>(hb + 4 * (CP_PLANE / 4) + row * 4) = make_uint4(lo2[0], lo2[1], lo2[2], lo2[3]);
        *reinterpret_cast<uint4 *>(hb + 5 * (CP_PLANE / 4) + row * 4) = make_uint4(lo2[4], lo2[5], lo2[6], lo2[7]);
    }
    return bad;
}

// the raw X box of a job: image n, rows from hp0 - ph (hp0 = the padded row
// of the tile's first flat position), channels cb*16.., columns from -(pw + wsh)
template <int NT>
__device__ __forceinline__ void cp_issue_raw(const ConvPlanarArgs &p, const CUtensorMap *map, const CpJob &j,
                                             uint64_t *bar, void *dst) {
    const int n = j.tile / p.tpi, F0 = (j.tile - n * p.tpi) * NT;
    const int hp0 = F0 / p.Wp;
    mbar_expect_tx(bar, (uint32_t)(16 * p.rb * p.wb * 4));
    tma_load_4d(map, bar, dst, -(p.pw + p.wsh), hp0 - p.ph, j.cb * 16, n);
}

__device__ __forceinline__ int64_t cp_range(int64_t units, int ctas, int k) { return units * k / ctas; }

// the CTA whose range [cp_range(k), cp_range(k + 1)) holds unit u
__device__ __forceinline__ int cp_cta_of(int64_t units, int ctas, int64_t u) {
    int k = (int)(((u + 1) * ctas - 1) / units);   // first guess, then fix up
    while (k > 0 && cp_range(units, ctas, k) > u) k--;
    while (k + 1 < ctas && cp_range(units, ctas, k + 1) <= u) k++;
    return k;
}

__device__ __forceinline__ int ld_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// FP32 recompute / fused epilogue stages over a staged tile T[co][TS] (cold path)
__device__ __noinline__ void cp_fix_tile(const ConvPlanarArgs &p, float *T, int TS, int NT, int n, int Ft, int co0,
                                         int nco, int te, bool nf) {
    for (int e = te; e < nco * NT; e += 32 * CP_EPI_WARPS) {
        const int co_l = e / NT, col = e - co_l * NT;
        int ho, wo;
        if (!cp_pixel(p, Ft + col, ho, wo)) continue;
        float v = nf ? cp_fp32_point(p, n, co0 + co_l, ho, wo) : T[co_l * TS + col];
        if (p.epi.n) v = apply_epilogue(p.epi, v, n, co0 + co_l, ho, wo);
        T[co_l * TS + col] = v;
    }
}

// the epilogue warps' accumulators of a whole tile (64 channels x NT flat
// columns) -> T[co][NT + 4] in the free halo buffers -> NCHW rows: warps take
// channels, lanes consecutive flat columns
template <int NT>
__device__ __forceinline__ void cp_store_tile(const ConvPlanarArgs &p, float *T, const float (&acc)[NT / 64][16],
                                              int q, int h, int lane, int ew, int n, int Ft, int ct, bool nf) {
    constexpr int TS = NT + 4, kCols = NT / 2;
    static_assert(64 * TS * 4 <= 2 * CP_HALO_BYTES, "tile staging fits the halo buffers");
    const bool odd = lane & 1;
    const int rowc = 16 * q + (lane >> 1);
#pragma unroll
    for (int pp = 0; pp < NT / 64; pp++)
#pragma unroll
        for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4 *>(T + rowc * TS + h * kCols + pp * 32 + (odd ? 16 : 0) + i) =
                make_float4(acc[pp][i], acc[pp][i + 1], acc[pp][i + 2], acc[pp][i + 3]);
    asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
    const int co0 = ct * 64, nco = min(64, p.CO - co0);
    if (nf || p.epi.n) {
        cp_fix_tile(p, T, TS, NT, n, Ft, co0, nco, ew * 32 + lane, nf);
        asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
    }
    if (ew == 0 && lane == 0) cp_stamp2(p, 124);
    if (p.dbg & 1) return;
    // lanes take consecutive flat columns (32 per instruction), warps take
    // channels; the columns' output offsets are computed once.  (Measured on
    // C3, store phase per CTA: 4.5k cycles; float4 stores of 4-column quads,
    // two output rows per instruction: 7.3k; one output row per instruction:
    // 15.6k.)
    constexpr int kCpl = NT / 32;   // columns per lane
    int64_t off[kCpl];
    bool ok[kCpl];
    {
        int ho = (Ft + lane) / p.Wp, wo = Ft + lane - ho * p.Wp;
#pragma unroll
        for (int k = 0; k < kCpl; k++) {
            ok[k] = ho < p.HO && wo < p.WO;
            off[k] = (int64_t)n * p.so[0] + (int64_t)ho * p.so[2] + (int64_t)wo * p.so[3];
            wo += 32;
            while (wo >= p.Wp) {
                wo -= p.Wp;
                ho++;
            }
        }
    }
    const int64_t so1 = p.so[1];
    for (int co_l = ew; co_l < nco; co_l += CP_EPI_WARPS) {
        float *dst = p.o + (int64_t)(co0 + co_l) * so1;
        const float *src = T + co_l * TS + lane;
#pragma unroll
        for (int k = 0; k < kCpl; k++)
            if (ok[k]) dst[off[k]] = src[32 * k];
    }
}

template <int NT>
__global__ void __launch_bounds__(CP_THREADS, 1)
    conv_planar_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ ConvPlanarArgs p) {
    static_assert(NT % 64 == 0 && NT <= 256, "pixel tile: a multiple of 64 up to 256");
    constexpr uint32_t kTmemCols = 2 * NT <= 256 ? 256 : 512;   // power of two
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *halo_full = reinterpret_cast<uint64_t *>(smem + CP_OFF_BAR);
    uint64_t *halo_empty = halo_full + 2;
    uint64_t *f_full = halo_empty + 2;
    uint64_t *f_empty = f_full + CP_FSLOTS;
    uint64_t *c_full = f_empty + CP_FSLOTS;
    uint64_t *c_empty = c_full + 2;
    uint64_t *raw_full = c_empty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(raw_full + CP_RAW_SLOTS);
    volatile int *last_flag = reinterpret_cast<volatile int *>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cta = blockIdx.x, ctas = gridDim.x;
    const int64_t u_begin = cp_range(p.units, ctas, cta), u_end = cp_range(p.units, ctas, cta + 1);
    CpIter it;
    it.init(p, u_begin, u_end);
    if (p.trace && threadIdx.x == 0) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[cta * 64 + 62] = t;
        p.trace[cta * 64 + 60] = clock64();
    }

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&map_x);
        for (int i = 0; i < 2; i++) {
            mbar_init(&halo_full[i], 32 * CP_CONV_WARPS);
            mbar_init(&halo_empty[i], 1);
            mbar_init(&c_full[i], 1);
            mbar_init(&c_empty[i], CP_EPI_WARPS);
        }
        for (int i = 0; i < CP_FSLOTS; i++) {
            mbar_init(&f_full[i], 1);
            mbar_init(&f_empty[i], 1);
        }
        for (int i = 0; i < CP_RAW_SLOTS; i++) mbar_init(&raw_full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the first raw X boxes go out before anything else
        CpIter is = it;
        CpJob j;
        for (int i = 0; i < CP_RAW_SLOTS && is.next(p, j); i++)
            cp_issue_raw<NT>(p, &map_x, j, &raw_full[i], smem + CP_OFF_RAW + i * CP_RAW_BYTES);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int RS = p.R * p.S;
    if (threadIdx.x == 0) cp_stamp(p, 0);

    if (warp == 0) {
        // ---------------- filter stages: 8 KiB bulk copies of the planar stage
        // images the prepass built (programmatic dependent launch: wait for it)
        if (lane == 0) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            int slot = 0;
            uint32_t ph = 0;
            CpJob j;
            while (it.next(p, j)) {
                for (int tap = j.t0; tap < j.t1; tap += 2) {   // slots hold tap pairs
                    const int n = min(2, j.t1 - tap);
                    mbar_wait_sleep(&f_empty[slot], ph ^ 1);
                    mbar_expect_tx(&f_full[slot], n * CP_FSTAGE);
                    const int64_t ts = (int64_t)j.ct * p.stages + j.cb * RS + tap;
                    for (int i = 0; i < n; i++)
                        bulk_load(smem + CP_OFF_FRING + (2 * slot + i) * CP_FSTAGE, p.wimg + (ts + i) * (CP_FSTAGE / 4),
                                  CP_FSTAGE, &f_full[slot]);
                    if (++slot == CP_FSLOTS) {
                        slot = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: the whole warp runs the loop, so the
        // descriptor arithmetic is warp-uniform (uniform registers, no
        // per-MMA broadcasts) and one elected lane issues each tcgen05 op
        constexpr uint32_t idesc = idesc_tf32(128, NT), idesc_lo = idesc_bf16(128, NT);
        constexpr uint64_t kPlane = CP_PLANE >> 4, kAPlane = 2048 >> 4;
        int slot = 0, b = 0, njob = 0;
        uint32_t fph = 0, hph[2] = {0, 0}, cph[2] = {0, 0};
        const uint64_t adesc0 = desc_planar(smem_u32(smem + CP_OFF_FRING), 2048);
        const uint32_t rowoff = (uint32_t)(p.dh * p.Wp);
        CpJob j;
        while (it.next(p, j)) {
            if (lane == 0 && njob < 4) cp_stamp2(p, 32 * njob + 4);
            mbar_wait_sleep(&halo_full[b], hph[b]);
            hph[b] ^= 1;
            if (lane == 0 && njob < 4) cp_stamp2(p, 32 * njob + 5);
            mbar_wait_sleep(&c_empty[b], cph[b] ^ 1);
            cph[b] ^= 1;
            if (lane == 0 && njob < 4) cp_stamp2(p, 32 * njob + 6);
            tc_fence_after();
            if (lane == 0 && njob < 4) cp_stamp(p, 56 + njob);
            const uint32_t d = tmem + (uint32_t)(b * NT);
            const uint64_t bdesc0 = desc_planar(smem_u32(smem + b * CP_HALO_BYTES), CP_PLANE);
            int r = j.t0 / p.S, s = j.t0 - r * p.S;
            for (int tap = j.t0; tap < j.t1; tap += 2) {
                // one filter slot = a tap pair: one barrier wait per 6 MMAs
                const int n = min(2, j.t1 - tap);
                mbar_wait_sleep(&f_full[slot], fph);
                tc_fence_after();
                const uint64_t a0 = adesc0 + (uint64_t)slot * (2 * CP_FSTAGE >> 4);
                const uint64_t b0 = bdesc0 + (uint64_t)(r * rowoff + s * (uint32_t)p.dw);
                if (++s == p.S) {
                    s = 0;
                    ++r;
                }
                const uint64_t a1 = a0 + (CP_FSTAGE >> 4);
                const uint64_t b1 = bdesc0 + (uint64_t)(r * rowoff + s * (uint32_t)p.dw);
                if (n == 2 && ++s == p.S) {
                    s = 0;
                    ++r;
                }
                if (elect_one()) {
                    if (!(p.dbg & 4)) {
                        umma_tf32(d, a0, b0, idesc, tap == j.t0 ? 0u : 1u);
                        umma_tf32(d, a0 + 2 * kAPlane, b0 + 2 * kPlane, idesc, 1u);
                        umma_f16(d, a0 + 4 * kAPlane, b0 + 4 * kPlane, idesc_lo, 1u);
                        if (n == 2) {
                            umma_tf32(d, a1, b1, idesc, 1u);
                            umma_tf32(d, a1 + 2 * kAPlane, b1 + 2 * kPlane, idesc, 1u);
                            umma_f16(d, a1 + 4 * kAPlane, b1 + 4 * kPlane, idesc_lo, 1u);
                        }
                    }
                    umma_commit(&f_empty[slot]);
                }
                __syncwarp();
                if (++slot == CP_FSLOTS) {
                    slot = 0;
                    fph ^= 1;
                }
            }
            if (elect_one()) {
                umma_commit(&halo_empty[b]);
                umma_commit(&c_full[b]);
            }
            __syncwarp();
            if (lane == 0) cp_stamp(p, 1 + min(njob, 14));
            njob++;
            b ^= 1;
        }
    } else if (warp < 2 + CP_CONV_WARPS) {
        // ---------------- halo converters: raw slot [c][row][wb] -> planar hi / lo
        const int t = threadIdx.x - 64;
        int b = 0, rs = 0, njob = 0;
        uint32_t eph = 0, rph = 0;   // barrier parities, one bit per buffer
        CpIter ia = it;              // runs CP_RAW_SLOTS jobs ahead: the box refilling the slot just converted
        CpJob j, ja;
        for (int i = 0; i < CP_RAW_SLOTS; i++) ia.next(p, ja);
        while (it.next(p, j)) {
            const int n = j.tile / p.tpi, F0 = (j.tile - n * p.tpi) * NT;
            mbar_wait_sleep(&raw_full[rs], (rph >> rs) & 1);
            rph ^= 1u << rs;
            mbar_wait_sleep(&halo_empty[b], ((eph >> b) & 1) ^ 1);
            eph ^= 1u << b;
            const float *raw = reinterpret_cast<const float *>(smem + CP_OFF_RAW + rs * CP_RAW_BYTES);
            float *hb = reinterpret_cast<float *>(smem + b * CP_HALO_BYTES);
            // the first halo is converted with the epilogue warps' help (idle until the first fold)
            const bool first = njob == 0;
            const bool bad = cp_convert(p, raw, hb, F0, t, first ? 32 * (CP_CONV_WARPS + CP_EPI_WARPS) : 32 * CP_CONV_WARPS);
            if (bad) {
                p.tileflag[(int64_t)j.ct * p.tiles + j.tile] = p.gen;
                __threadfence();
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (first) asm volatile("bar.sync 3, %0;" ::"r"(32 * (CP_CONV_WARPS + CP_EPI_WARPS)) : "memory");
            mbar_arrive(&halo_full[b]);
            if (t == 0) cp_stamp(p, 16 + min(njob, 14));
            // every converter is done reading raw slot rs: refill it
            asm volatile("bar.sync 2, %0;" ::"r"(32 * CP_CONV_WARPS) : "memory");
            if (ia.next(p, ja) && t == 0)
                cp_issue_raw<NT>(p, &map_x, ja, &raw_full[rs], smem + CP_OFF_RAW + rs * CP_RAW_BYTES);
            njob++;
            b ^= 1;
            if (++rs == CP_RAW_SLOTS) rs = 0;
        }
    } else {
        // ---------------- epilogue
        const int ew = warp - 2 - CP_CONV_WARPS;   // 0..7
        const int q = warp & 3;                    // TMEM lane quadrant (warp id % 4)
        const int h = ew >> 2;                     // column half
        const bool odd = lane & 1;
        constexpr int kParts = NT / 64;            // 32-column parts per warp (NT / 2 columns)
        constexpr int kCols = NT / 2;
        {
            // help the converters with the first halo (raw slot 0 -> halo buffer 0)
            CpIter i1 = it;
            CpJob j1;
            i1.next(p, j1);
            const int n = j1.tile / p.tpi, F0 = (j1.tile - n * p.tpi) * NT;
            mbar_wait_sleep(&raw_full[0], 0);
            const bool bad = cp_convert(p, reinterpret_cast<const float *>(smem + CP_OFF_RAW),
                                        reinterpret_cast<float *>(smem), F0, 32 * CP_CONV_WARPS + ew * 32 + lane,
                                        32 * (CP_CONV_WARPS + CP_EPI_WARPS));
            if (bad) {
                p.tileflag[(int64_t)j1.ct * p.tiles + j1.tile] = p.gen;
                __threadfence();
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.arrive 3, %0;" ::"r"(32 * (CP_CONV_WARPS + CP_EPI_WARPS)) : "memory");
        }
        float acc[kParts][16];
#pragma unroll
        for (int pp = 0; pp < kParts; pp++)
#pragma unroll
            for (int i = 0; i < 16; i++) acc[pp][i] = 0.0f;
        float *stg = reinterpret_cast<float *>(smem + CP_OFF_STG + ew * CP_STG_WARP);
        asm volatile("griddepcontrol.wait;" ::: "memory");   // wflag is a prepass output
        int b = 0, njob = 0;
        uint32_t fph = 0;
        CpJob j;
        while (it.next(p, j)) {
            // suspended, not spinning: the converters need the issue slots
            mbar_wait_sleep(&c_full[b], (fph >> b) & 1);
            fph ^= 1u << b;
            tc_fence_after();
            const int64_t tl = (int64_t)j.ct * p.tiles + j.tile;
            const bool whole = j.head && j.complete;
            // the non-finite flags of a tile held whole are final once its last
            // job is converted: issue the loads now, under the fold
            int nf_t = 0, nf_w = 0;
            if (j.seg_last && whole) {
                nf_t = ld_relaxed(p.tileflag + tl);
                nf_w = ld_relaxed(p.wflag);
            }
#pragma unroll
            for (int pp = 0; pp < kParts; pp++) {
                // lanes 2c / 2c+1 hold the hi / lo filter rows of channel c for
                // the same 32 columns: the even lane keeps columns 0-15, the odd 16-31
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * NT + h * kCols + pp * 32);
                uint32_t r0[16], r1[16];
                tmem_ld16_issue(ta, r0);
                tmem_ld16_issue(ta + 16, r1);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 16; i++) {
                    const float mine = __uint_as_float(odd ? r1[i] : r0[i]);
                    const float give = __uint_as_float(odd ? r0[i] : r1[i]);
                    acc[pp][i] += mine + __shfl_xor_sync(0xffffffffu, give, 1);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&c_empty[b]);
            if (ew == 0 && lane == 0) cp_stamp(p, 31 + min(njob, 14));
            njob++;
            b ^= 1;
            if (!j.seg_last) continue;

            const int n = j.tile / p.tpi, Ft = (j.tile - n * p.tpi) * NT;
            if (whole && j.last) {
                // the CTA's last segment holds its tile whole (every tile, when the
                // tiles fit one wave): no job remains, so both halo buffers are
                // free -- stage the whole tile there and store it by output rows
                cp_store_tile<NT>(p, reinterpret_cast<float *>(smem), acc, q, h, lane, ew, n, Ft, j.ct,
                                  nf_t == p.gen || nf_w == p.gen);
                if (ew == 0 && lane == 0) cp_stamp(p, 49);
                break;
            }
            // ---- otherwise: this warp's 16 channels x kCols columns, 32 columns
            // (one part) at a time through its smem block
            const int F0 = Ft + h * kCols;
            const int co0 = j.ct * 64 + 16 * q;
            int k0 = 0, k1 = 0;
            bool store = whole;
            if (!whole) {
                // the tile is split over CTAs k0..k1 (segment i = CTA k0 + i): every
                // segment publishes its partial (slot 2 cta + (head ? 1 : 0): a CTA
                // holds at most a tail-of-tile first segment and a head last
                // segment), then counts in; the LAST to arrive sums all partials in
                // segment order -- deterministic whoever it is -- and stores.
                const int slot = 2 * cta + (j.head ? 1 : 0);
                float *dst = p.part + ((int64_t)slot * 64 + 16 * q) * NT + h * kCols;
#pragma unroll
                for (int pp = 0; pp < kParts; pp++) {
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        *reinterpret_cast<float4 *>(stg + (lane >> 1) * CP_STG_ROW + (odd ? 16 : 0) + i) =
                            make_float4(acc[pp][i], acc[pp][i + 1], acc[pp][i + 2], acc[pp][i + 3]);
                    __syncwarp();
#pragma unroll
                    for (int cr = 0; cr < 16; cr++)
                        __stcg(dst + (int64_t)cr * NT + pp * 32 + lane, stg[cr * CP_STG_ROW + lane]);
                    __syncwarp();
                }
                asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
                const int t0u = j.tile_end - p.stages;
                k0 = cp_cta_of(p.units, ctas, t0u);
                k1 = cp_cta_of(p.units, ctas, j.tile_end - 1);
                if (ew == 0 && lane == 0) {
                    int old;
                    asm volatile("fence.acq_rel.gpu;\n\tatom.relaxed.gpu.global.add.s32 %0, [%1], 1;"
                                 : "=r"(old)
                                 : "l"(p.tilecnt + tl)
                                 : "memory");
                    const bool last = old == k1 - k0;
                    if (last) {
                        p.tilecnt[tl] = 0;   // re-armed for the next launch
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    }
                    *last_flag = last ? 1 : 0;
                }
                asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
                store = *last_flag;
                if (store) {
                    // every segment's converters counted in after converting
                    nf_t = ld_relaxed(p.tileflag + tl);
                    nf_w = ld_relaxed(p.wflag);
                }
            }
            if (store) {
                const bool nf = nf_t == p.gen || nf_w == p.gen;
                // NCHW stores: lane -> one flat column per part (32 consecutive
                // positions per instruction), 16 channels unrolled
                const int64_t so1 = p.so[1];
                const int nco = min(16, p.CO - co0);
#pragma unroll
                for (int pp = 0; pp < kParts; pp++) {
                    if (whole) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            *reinterpret_cast<float4 *>(stg + (lane >> 1) * CP_STG_ROW + (odd ? 16 : 0) + i) =
                                make_float4(acc[pp][i], acc[pp][i + 1], acc[pp][i + 2], acc[pp][i + 3]);
                    } else {
                        // sum the k1 - k0 + 1 partials in segment order
                        for (int cr = 0; cr < 16; cr++) {
                            float a = 0.0f;
                            for (int k = k0; k <= k1; k++) {
                                const int sl = 2 * k + (k == k0 ? 1 : 0);   // the tile's head is CTA k0's last segment
                                a += __ldcg(p.part + ((int64_t)sl * 64 + 16 * q + cr) * NT + h * kCols + pp * 32 +
                                            lane);
                            }
                            stg[cr * CP_STG_ROW + lane] = a;
                        }
                    }
                    __syncwarp();
                    const int Fp = F0 + pp * 32;
                    if (nf) cp_recompute(p, stg, n, Fp, co0, lane);
                    if (p.epi.n) cp_epilogue_col(p, stg, n, Fp, co0, lane);
                    int ho, wo;
                    const bool ok = cp_pixel(p, Fp + lane, ho, wo) && !(p.dbg & 1);
                    const int64_t off = (int64_t)n * p.so[0] + (int64_t)ho * p.so[2] + (int64_t)wo * p.so[3] +
                                        (int64_t)co0 * so1;
                    if (ok) {
#pragma unroll
                        for (int cr = 0; cr < 16; cr++)
                            if (cr < nco) p.o[off + cr * so1] = stg[cr * CP_STG_ROW + lane];
                    }
                    __syncwarp();
                }
            }
            // last_flag is reused by the next segment
            if (!whole) asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
#pragma unroll
            for (int pp = 0; pp < kParts; pp++)
#pragma unroll
                for (int i = 0; i < 16; i++) acc[pp][i] = 0.0f;
        }
    }
    __syncwarp();   // warp 0's lanes 1-31 wait for lane 0 (bar.sync is warp-aligned)
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) cp_stamp(p, 63);
    if (p.trace && threadIdx.x == 0) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[cta * 64 + 61] = t;
    }
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

}  // namespace tc
}  // namespace lsb
