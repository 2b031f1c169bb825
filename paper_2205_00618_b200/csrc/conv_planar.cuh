// conv_planar.cuh -- single-pass NCHW direct convolution on the tensor cores
// (split TF32), stride 1, any padding / dilation, zero fill.
//
// Flat padded pixel space.  With Hp = HO + (R-1) dh, Wp = WO + (S-1) dw (the
// padded extent the taps reach; padded (hp, wp) = raw (hp - ph, wp - pw)), the output
// pixel (n, ho, wo) is computed at the flat position F = n Hp Wp + ho Wp + wo
// of the padded input grid, and its tap (r, s) reads the padded input at
// F + r dh Wp + s dw.  Over a tile of NT consecutive F every tap is therefore
// one contiguous run of NT rows of a "halo" of NT + (R-1) dh Wp + (S-1) dw
// rows: the implicit GEMM's B operand for tap (r, s) is the halo shifted by a
// row offset.  Positions with ho >= HO or wo >= WO are computed and dropped.
//
// Planar operands.  The halo lives in smem as K-major SWIZZLE_NONE "planes":
// plane g holds channels 4g..4g+3 of every halo row, rows 16 B apart
// ([plane][row][4]), so core matrices (8 rows x 16 B) are contiguous for ANY
// start row: descriptor LBO = plane stride, SBO = 128 B, and the tap shift is
// just start + off * 16 B (verified on B200: tools/umma_planar_probe.cu;
// 128 cycles per 128x256x8 MMA, the same as the swizzled layouts).
//
// Split TF32 without a prepass.  The tensor core truncates fp32 operands to
// tf32 (probe mode 1), so the raw value IS the hi part; lo = x - trunc(x) is
// exact in fp32.  The A operand stacks the filters as 128 rows, row 2c =
// W[c] (hi), row 2c+1 = W[c] - trunc(W[c]) (lo), and each 16-channel stage
// issues  D += A.Xhi, D += A.Xlo  per 8 channels: row 2c accumulates
// Whi.(Xhi + Xlo), row 2c+1 Wlo.(Xhi + Xlo); the epilogue adds the row pair
// (3xTF32 plus the lo.lo term).  Two N = NT MMAs per 8 channels for 64 output
// channels x NT pixels.
//
// Stream-K.  Work units are (co tile, pixel tile, stage), stage = (16-channel
// block cb, tap); a persistent grid of one CTA per SM takes equal unit ranges.
// A CTA's range is a sequence of segments (runs within one tile); the CTA
// holding a tile's stage 0 owns the tile: the other segments (always the
// first segment of a later CTA, computed first) publish fp32 partials to a
// per-CTA slot with an epoch-stamped flag, and the owner adds them in CTA
// order (deterministic) before the fused epilogue and the NCHW stores.  The
// launch is cooperative (all CTAs resident), and no CTA waits before it has
// published, so the waits cannot deadlock.
//
// Two-level accumulation.  TMEM holds two NT-column accumulators; each job
// (one halo = one cb of one segment, <= R*S stages = 144-channel K for 3x3)
// accumulates into one while the epilogue warps fold the other into fp32
// registers (round to nearest; the tensor core's accumulate truncates).
//
// Warp roles (448 threads, 1 CTA / SM):
//   warp 0      filter stages: cp.async.bulk of 8 KiB planar stage images
//               (built by all CTAs at the start, behind a grid barrier) into
//               a 6-slot ring
//   warp 1      TMEM allocator + tcgen05.mma issuer
//   warps 2-5   halo converters: NCHW fp32 (global) -> hi / lo planes (smem),
//               zero outside the image (the padding), non-finite flags
//   warps 6-13  epilogue: fold, hi/lo row-pair sum (shfl), publish / owner
//               fixup, smem transpose, coalesced NCHW stores
#pragma once

#include "conv_common.cuh"

namespace lsb {
namespace tc {

constexpr int CP_HALO = 384;                       // halo rows per buffer
constexpr int CP_PLANE = CP_HALO * 16;             // bytes per 4-channel plane
constexpr int CP_HALO_BYTES = 8 * CP_PLANE;        // hi planes 0-3, lo planes 4-7: 48 KiB
constexpr int CP_FSLOTS = 3;                       // filter ring slots, each a tap pair
constexpr int CP_FSTAGE = 4 * 128 * 16;            // 8 KiB per tap: 4 planes x 128 rows x 16 B
constexpr int CP_CONV_WARPS = 4;
constexpr int CP_EPI_WARPS = 8;
constexpr int CP_THREADS = 64 + 32 * (CP_CONV_WARPS + CP_EPI_WARPS);   // 448
constexpr int CP_STG_ROW = 132;                    // staged floats per channel row (128 + pad)
constexpr int CP_STG_WARP = 16 * CP_STG_ROW * 4;   // 8448 B per epilogue warp
constexpr int CP_OFF_FRING = 2 * CP_HALO_BYTES;
constexpr int CP_OFF_STG = CP_OFF_FRING + 2 * CP_FSLOTS * CP_FSTAGE;
constexpr int CP_OFF_BAR = CP_OFF_STG + CP_EPI_WARPS * CP_STG_WARP;
constexpr size_t CP_SMEM = (size_t)CP_OFF_BAR + 256 + 1024;

struct ConvPlanarArgs {
    const float *x;
    int64_t sx[4];                 // NCHW element strides
    int N, C, H, W, CO, R, S, HO, WO, ph, pw, dh, dw;
    int Hp, Wp, halo;              // padded grid, halo rows used (<= CP_HALO)
    int tiles, co_tiles, cbs, stages;   // stages per tile = cbs * R * S
    int64_t units;                 // co_tiles * tiles * stages
    const float *wimg;             // [co_tile][stage][4 planes][128][4] (built in the kernel)
    float *wimg_w;                 // the same buffer, written by the CTAs
    int *gridbar;                  // filter-image barrier: += 1 per CTA per launch
    int bar_target;                // its value once every CTA of this launch arrived
    float *o;
    int64_t so[4];
    float *part;                   // [cta][64][NT] published partial sums
    int *tilecnt;                  // [co_tile * tiles + tile] segments arrived (reset by the last)
    int *tileflag;                 // [co_tile * tiles + tile] == gen: non-finite X in the tile's halo
    int *wflag;                    // == gen: non-finite filter (set while building the filter images)
    int gen;
    const float *w;
    int64_t swt[4];
    EpiStages epi;
    long long *trace;              // debug (LSB_CONV_TRACE): [cta][64] globaltimer stamps
    int dbg;                       // experiments (LSB_CP_DBG): 1 skip output stores, 2 skip publish stores, 4 skip MMAs,
                                   // 8 MMAs do not wait for filter stages, 16 nor for halos
};

__device__ __forceinline__ void cp_stamp(const ConvPlanarArgs &p, int slot) {
    if (p.trace != nullptr && slot < 64) p.trace[blockIdx.x * 64 + slot] = clock64();
}

// stage-level clock64 stamps of the MMA issuer: [148 * 64 + cta * 128 + slot]
__device__ __forceinline__ void cp_stamp2(const ConvPlanarArgs &p, int slot) {
    if (slot < 128) p.trace[148 * 64 + blockIdx.x * 128 + slot] = clock64();
}

// one element of the planar filter stage images: stage (cb, tap) of co tile
// ct holds, for the 16 channels cb*16.., rows 2c = W[ct*64 + c] (the hi part:
// the tensor core truncates) and 2c+1 = W - trunc(W); channels >= C and
// filters >= CO are zero.  e = ((ct * stages + stage) * 64 + co) * 16 + ch.
// Returns true for a non-finite filter value.
__device__ __forceinline__ bool cp_filter_elem(const ConvPlanarArgs &p, int e) {
    const float inf = __int_as_float(0x7f800000);
    const int ch = e & 15, co_l = (e >> 4) & 63, ts = e >> 10;
    const int stage = ts % p.stages, ct = ts / p.stages;
    const int RS = p.R * p.S;
    const int cb = stage / RS, tap = stage - cb * RS;
    const int r = tap / p.S, s = tap - r * p.S;
    const int co = ct * 64 + co_l, c = cb * 16 + ch;
    float v = 0.0f;
    if (co < p.CO && c < p.C) v = __ldg(p.w + co * p.swt[0] + c * p.swt[1] + r * p.swt[2] + s * p.swt[3]);
    const bool fin = fabsf(v) < inf;
    const float lo = fin ? v - __uint_as_float(__float_as_uint(v) & 0xffffe000u) : 0.0f;
    float *st = p.wimg_w + (int64_t)ts * (CP_FSTAGE / 4);
    const int plane = ch >> 2, q = ch & 3;
    st[plane * 512 + (2 * co_l) * 4 + q] = v;
    st[plane * 512 + (2 * co_l + 1) * 4 + q] = lo;
    return !fin;
}

// cold path, out of line
// non-finite input in the tile: FP32 recompute of the warp's staged 16 x 128
// block (3xTF32 would turn inf x 0 in a cross term into NaN); out-of-range
// taps contribute 0 x w like the guarded view
__device__ __noinline__ void cp_recompute(const ConvPlanarArgs &p, float *stg, int F0, int co0, int lane, int ncols) {
    const int HpWp = p.Hp * p.Wp;
    for (int col = lane; col < ncols; col += 32) {
        const int F = F0 + col;
        const int n = F / HpWp, rem = F - n * HpWp, ho = rem / p.Wp, wo = rem - ho * p.Wp;
        if (n >= p.N || ho >= p.HO || wo >= p.WO) continue;
        for (int cr = 0; cr < 16 && co0 + cr < p.CO; cr++) {
            const int co = co0 + cr;
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
            stg[cr * CP_STG_ROW + col] = a;
        }
    }
    __syncwarp();
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

// one job = the stages of one (co tile, tile, cb) inside this CTA's range
struct CpJob {
    int ct, tile, cb, t0, t1;      // taps [t0, t1)
    bool seg_last;                 // the job ends its segment
    bool head;                     // the segment starts at stage 0 of the tile
    bool complete;                 // the segment ends at the tile's last stage
    int64_t tile_end;              // first unit after the tile
};

__device__ __forceinline__ bool cp_next(const ConvPlanarArgs &p, int64_t &u, int64_t u_begin, int64_t u_end,
                                        CpJob &j) {
    if (u >= u_end) return false;
    // 32-bit arithmetic throughout (units < 2^31, checked by the host): a
    // 64-bit division here cost ~0.3k cycles per job in every role
    const int RS = p.R * p.S;
    const int uu = (int)u, ue = (int)u_end;
    const int tl = uu / p.stages;
    const int st = uu - tl * p.stages;
    const int cb = st / RS, tap = st - cb * RS;
    const int tile_begin = tl * p.stages;
    const int job_end = min(ue, tile_begin + (cb + 1) * RS);
    j.ct = tl / p.tiles;
    j.tile = tl - j.ct * p.tiles;
    j.cb = cb;
    j.t0 = tap;
    j.t1 = tap + (job_end - uu);
    j.tile_end = tile_begin + p.stages;
    j.seg_last = job_end == ue || job_end == (int)j.tile_end;
    j.head = tile_begin >= (int)u_begin;
    j.complete = (int)j.tile_end <= ue;
    u = job_end;
    return true;
}

// a converter thread's share of a job's halo: rows t, t + 128, ... of the
// flat range [tile * NT, + halo), 16 channels of block cb (0 outside the image)
template <int NT, int kRows>
__device__ __forceinline__ void cp_gather(const ConvPlanarArgs &p, const CpJob &j, int t, float (&v)[kRows][16]) {
    const int HpWp = p.Hp * p.Wp, nflat = p.N * HpWp;
    const int F0 = j.tile * NT;
#pragma unroll
    for (int rr = 0; rr < kRows; rr++) {
        const int row = t + rr * 32 * CP_CONV_WARPS;
        const int F = F0 + row;
        int64_t base = -1;
        if (row < p.halo && F < nflat) {
            const int n = F / HpWp;
            const int rem = F - n * HpWp;
            const int hp = rem / p.Wp, wp = rem - hp * p.Wp;
            const int hi_ = hp - p.ph, wi = wp - p.pw;
            if (hi_ >= 0 && hi_ < p.H && wi >= 0 && wi < p.W) base = n * p.sx[0] + hi_ * p.sx[2] + wi * p.sx[3];
        }
        const float *src = p.x + (base < 0 ? 0 : base) + (int64_t)(j.cb * 16) * p.sx[1];
        const int nch = (base < 0 || (p.dbg & 128)) ? 0 : min(16, p.C - j.cb * 16);
#pragma unroll
        for (int c = 0; c < 16; c++) v[rr][c] = c < nch ? __ldg(src + c * p.sx[1]) : 0.0f;
    }
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

// fused epilogue stages applied in place to a warp's staged 16 x ncols block
// (out of line: most convs have none)
__device__ __noinline__ void cp_epilogue_block(const ConvPlanarArgs &p, float *stg, int F0, int co0, int lane,
                                               int ncols) {
    const int HpWp = p.Hp * p.Wp;
    for (int col = lane; col < ncols; col += 32) {
        const int F = F0 + col;
        const int n = F / HpWp, rem = F - n * HpWp, ho = rem / p.Wp, wo = rem - ho * p.Wp;
        if (n >= p.N || ho >= p.HO || wo >= p.WO) continue;
        for (int cr = 0; cr < 16 && co0 + cr < p.CO; cr++)
            stg[cr * CP_STG_ROW + col] = apply_epilogue(p.epi, stg[cr * CP_STG_ROW + col], n, co0 + cr, ho, wo);
    }
    __syncwarp();
}

template <int NT>
__global__ void __launch_bounds__(CP_THREADS, 1) conv_planar_kernel(const __grid_constant__ ConvPlanarArgs p) {
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
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(c_empty + 2);
    volatile int *last_flag = reinterpret_cast<volatile int *>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cta = blockIdx.x, ctas = gridDim.x;
    const int64_t u_begin = cp_range(p.units, ctas, cta), u_end = cp_range(p.units, ctas, cta + 1);
    if (p.trace && threadIdx.x == 0) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[cta * 64 + 62] = t;
    }

    // ---- before the setup barrier, the two global-latency-bound starts:
    // converters issue the first halo's loads, epilogue warps build this CTA's
    // share of the filter stage images and arrive on the grid barrier
    constexpr int kRows = CP_HALO / (32 * CP_CONV_WARPS);   // halo rows per converter thread
    float v[kRows][16];
    CpJob jc;
    int64_t uc = u_begin;
    bool conv_have = false;
    if (warp >= 2 && warp < 2 + CP_CONV_WARPS) {
        conv_have = cp_next(p, uc, u_begin, u_end, jc);
        if (conv_have) cp_gather<NT, kRows>(p, jc, threadIdx.x - 64, v);
    } else if (warp >= 2 + CP_CONV_WARPS) {
        // this CTA's share of the planar filter stage images (they would
        // otherwise need their own launch), then one arrival on the grid
        // barrier the filter producers wait on (cooperative launch: all
        // CTAs are resident)
        const int ew = warp - 2 - CP_CONV_WARPS;
        const int E = p.co_tiles * p.stages * 1024;
        const int e0 = (int)((int64_t)E * cta / ctas), e1 = (int)((int64_t)E * (cta + 1) / ctas);
        bool bad = false;
        for (int e = e0 + ew * 32 + lane; e < e1; e += 32 * CP_EPI_WARPS) bad |= cp_filter_elem(p, e);
        if (bad) *p.wflag = p.gen;
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
        if (ew == 0 && lane == 0)
            asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(p.gridbar) : "memory");
    }

    if (threadIdx.x == 0) {
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
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
        // images every CTA helped build (epilogue warps, below) -- wait for all
        if (lane == 0) {
            int arrived;
            do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(arrived) : "l"(p.gridbar) : "memory");
            } while (arrived - p.bar_target < 0);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            int slot = 0;
            uint32_t ph = 0;
            int64_t u = u_begin;
            CpJob j;
            while (cp_next(p, u, u_begin, u_end, j)) {
                for (int tap = j.t0; tap < j.t1; tap += 2) {   // slots hold tap pairs
                    const int n = min(2, j.t1 - tap);
                    mbar_wait(&f_empty[slot], ph ^ 1);
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
        // per-MMA broadcasts) and one elected lane issues each tcgen05 op;
        // per stage the loop must stay under the 4 MMAs' 512 cycles
        constexpr uint32_t idesc = idesc_tf32(128, NT);
        constexpr uint64_t kPlane = CP_PLANE >> 4, kAPlane = 2048 >> 4;
        int slot = 0, b = 0, njob = 0, nst = 0;
        uint32_t fph = 0, hph[2] = {0, 0}, cph[2] = {0, 0};
        const uint64_t adesc0 = desc_planar(smem_u32(smem + CP_OFF_FRING), 2048);
        const uint32_t rowoff = (uint32_t)(p.dh * p.Wp);
        int64_t u = u_begin;
        CpJob j;
        while (cp_next(p, u, u_begin, u_end, j)) {
            if (p.trace && lane == 0) cp_stamp2(p, 100 + 3 * min(njob, 8));
            if (!(p.dbg & 16)) mbar_wait(&halo_full[b], hph[b]);
            hph[b] ^= 1;
            if (p.trace && lane == 0) cp_stamp2(p, 101 + 3 * min(njob, 8));
            mbar_wait(&c_empty[b], cph[b] ^ 1);
            cph[b] ^= 1;
            if (p.trace && lane == 0) cp_stamp2(p, 102 + 3 * min(njob, 8));
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(b * NT);
            const uint64_t bdesc0 = desc_planar(smem_u32(smem + b * CP_HALO_BYTES), CP_PLANE);
            int r = j.t0 / p.S, s = j.t0 - r * p.S;
            for (int tap = j.t0; tap < j.t1; tap += 2) {
                // one filter slot = a tap pair: one barrier wait per 8 MMAs keeps
                // this loop (~500 cycles) under the tensor time it feeds
                const int n = min(2, j.t1 - tap);
                if (p.trace && lane == 0) cp_stamp2(p, 2 * nst);
                if (!(p.dbg & 8)) mbar_wait(&f_full[slot], fph);
                tc_fence_after();
                if (p.trace && lane == 0) cp_stamp2(p, 2 * nst + 1);
                nst++;
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
                        umma_tf32(d, a0, b0 + 4 * kPlane, idesc, 1u);
                        umma_tf32(d, a0 + 2 * kAPlane, b0 + 2 * kPlane, idesc, 1u);
                        umma_tf32(d, a0 + 2 * kAPlane, b0 + 6 * kPlane, idesc, 1u);
                        if (n == 2) {
                            umma_tf32(d, a1, b1, idesc, 1u);
                            umma_tf32(d, a1, b1 + 4 * kPlane, idesc, 1u);
                            umma_tf32(d, a1 + 2 * kAPlane, b1 + 2 * kPlane, idesc, 1u);
                            umma_tf32(d, a1 + 2 * kAPlane, b1 + 6 * kPlane, idesc, 1u);
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
        // ---------------- halo converters: NCHW fp32 -> planar hi / lo
        const int t = threadIdx.x - 64;
        const float inf = __int_as_float(0x7f800000);
        int b = 0, njob = 0;
        uint32_t eph[2] = {0, 0};
        // the loads of job k + 1 are issued as soon as job k is written, so the
        // gather overlaps the MMAs of job k (the first job's were issued before
        // the setup barrier)
        while (conv_have) {
            const CpJob j = jc;
            mbar_wait(&halo_empty[b], eph[b] ^ 1);
            eph[b] ^= 1;
            float *hb = reinterpret_cast<float *>(smem + b * CP_HALO_BYTES);
            bool bad = false;
#pragma unroll
            for (int rr = 0; rr < kRows; rr++) {
                const int row = t + rr * 32 * CP_CONV_WARPS;
                if (row >= p.halo) break;
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    float4 hv = make_float4(v[rr][4 * g], v[rr][4 * g + 1], v[rr][4 * g + 2], v[rr][4 * g + 3]);
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
                    *reinterpret_cast<float4 *>(hb + (4 + g) * (CP_PLANE / 4) + row * 4) = lv;
                }
            }
            if (bad) {
                p.tileflag[(int64_t)j.ct * p.tiles + j.tile] = p.gen;
                __threadfence();
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&halo_full[b]);
            if (t == 0) cp_stamp(p, 16 + min(njob, 14));
            njob++;
            b ^= 1;
            conv_have = cp_next(p, uc, u_begin, u_end, jc);
            if (conv_have) cp_gather<NT, kRows>(p, jc, t, v);
        }
    } else {
        // ---------------- epilogue
        const int ew = warp - 2 - CP_CONV_WARPS;   // 0..7
        const int q = warp & 3;                    // TMEM lane quadrant (warp id % 4)
        const int h = ew >> 2;                     // column half
        const bool odd = lane & 1;
        constexpr int kParts = NT / 64;            // 32-column parts per warp (NT / 2 columns)
        float acc[kParts][16];
#pragma unroll
        for (int pp = 0; pp < kParts; pp++)
#pragma unroll
            for (int i = 0; i < 16; i++) acc[pp][i] = 0.0f;
        float *stg = reinterpret_cast<float *>(smem + CP_OFF_STG + ew * CP_STG_WARP);
        const int HpWp = p.Hp * p.Wp;
        int b = 0, njob = 0, nseg = 0;
        uint32_t fph[2] = {0, 0};
        int64_t u = u_begin;
        CpJob j;
        while (cp_next(p, u, u_begin, u_end, j)) {
            mbar_wait(&c_full[b], fph[b]);
            fph[b] ^= 1;
            tc_fence_after();
            // non-finite flags of a tile this CTA holds whole are final once its
            // last job is converted: issue the loads now, under the fold
            int nf_tile = 0, nf_w = 0;
            if (j.seg_last && j.head && j.complete) {
                nf_tile = ld_relaxed(p.tileflag + (int64_t)j.ct * p.tiles + j.tile);
                nf_w = ld_relaxed(p.wflag);
            }
#pragma unroll
            for (int pp = 0; pp < kParts; pp++) {
                if (p.dbg & 32) break;
                // lanes 2c / 2c+1 hold the hi / lo filter rows of channel c for
                // the same 32 columns: the even lane keeps columns 0-15, the odd 16-31
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * NT + h * (NT / 2) + pp * 32);
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

            // ---- segment finished: this warp's 16 channels x NT/2 columns go to
            // its smem block, then publish, or (owner) fix up and store
#pragma unroll
            for (int pp = 0; pp < kParts; pp++)
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4 *>(stg + (lane >> 1) * CP_STG_ROW + pp * 32 + (odd ? 16 : 0) + i) =
                        make_float4(acc[pp][i], acc[pp][i + 1], acc[pp][i + 2], acc[pp][i + 3]);
            __syncwarp();
            constexpr int kCols = NT / 2;
            constexpr int kVec = 16 * kCols / 128;   // float4s per lane of the warp's block
            const int64_t tl = (int64_t)j.ct * p.tiles + j.tile;
            if (!(j.head && j.complete)) {
                // the tile is split over CTAs k0..k1 (segment i = CTA k0 + i): every
                // segment publishes its partial (slot 2 cta + (head ? 1 : 0): a CTA
                // holds at most a tail-of-tile first segment and a head last
                // segment), then counts in; the LAST to arrive sums all partials in
                // segment order -- deterministic whoever it is -- and stores.  No
                // CTA ever waits for another.
                const int slot = 2 * cta + (j.head ? 1 : 0);
                float *dst = p.part + ((int64_t)slot * 64 + 16 * q) * NT + h * kCols;
#pragma unroll
                for (int v = 0; v < kVec; v++) {
                    const int e = v * 128 + lane * 4, row = e / kCols, col = e % kCols;
                    const float4 x = *reinterpret_cast<const float4 *>(stg + row * CP_STG_ROW + col);
                    __stcg(reinterpret_cast<float4 *>(dst + (int64_t)row * NT + col), x);
                }
                asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
                const int64_t t0u = j.tile_end - p.stages;
                const int k0 = cp_cta_of(p.units, ctas, t0u), k1 = cp_cta_of(p.units, ctas, j.tile_end - 1);
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
                    cp_stamp(p, 46);
                }
                asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
                if (*last_flag) {
                    // sum the k1 - k0 + 1 partials in segment order
                    for (int v = 0; v < kVec; v++) {
                        const int e = v * 128 + lane * 4, row = e / kCols, col = e % kCols;
                        float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
                        for (int k = k0; k <= k1; k++) {
                            const int sl = 2 * k + (k == k0 ? 1 : 0);   // the tile's head is CTA k0's last segment
                            const float4 x = __ldcg(reinterpret_cast<const float4 *>(
                                p.part + ((int64_t)sl * 64 + 16 * q) * NT + h * kCols + (int64_t)row * NT + col));
                            acc4.x += x.x;
                            acc4.y += x.y;
                            acc4.z += x.z;
                            acc4.w += x.w;
                        }
                        *reinterpret_cast<float4 *>(stg + row * CP_STG_ROW + col) = acc4;
                    }
                    __syncwarp();
                }
            }
            const bool store = (j.head && j.complete) || *last_flag;
            __syncwarp();
            if (store) {
                if (ew == 0 && lane == 0) cp_stamp(p, 48 + 4 * min(nseg, 3));
                const int F0 = j.tile * NT + h * kCols, co0 = j.ct * 64 + 16 * q;
                if (!(j.head && j.complete)) {   // partial tile: every segment's converters have counted in
                    nf_tile = ld_relaxed(p.tileflag + tl);
                    nf_w = ld_relaxed(p.wflag);
                }
                if (nf_tile == p.gen || nf_w == p.gen)
                    cp_recompute(p, stg, F0, co0, lane, kCols);
                if (p.epi.n) cp_epilogue_block(p, stg, F0, co0, lane, kCols);
                // NCHW stores: lane -> kCols/32 columns (32 consecutive flat positions
                // per instruction), addresses computed once, 16 channels unrolled
                int64_t off[kCols / 32];
                bool ok[kCols / 32];
#pragma unroll
                for (int k = 0; k < kCols / 32; k++) {
                    const int F = F0 + k * 32 + lane;
                    const int n = F / HpWp, rem = F - n * HpWp, ho = rem / p.Wp, wo = rem - ho * p.Wp;
                    ok[k] = n < p.N && ho < p.HO && wo < p.WO && !(p.dbg & 1);
                    off[k] = n * p.so[0] + (int64_t)ho * p.so[2] + (int64_t)wo * p.so[3] + (int64_t)co0 * p.so[1];
                }
                float *o = p.o;
                const int64_t so1 = p.so[1];
                const int nco = min(16, p.CO - co0);
#pragma unroll
                for (int cr = 0; cr < 16; cr++) {
                    if (cr < nco) {
#pragma unroll
                        for (int k = 0; k < kCols / 32; k++)
                            if (ok[k]) o[off[k] + cr * so1] = stg[cr * CP_STG_ROW + k * 32 + lane];
                    }
                }
                if (ew == 0 && lane == 0) cp_stamp(p, 49 + 4 * min(nseg, 3));
            }
            // the smem block and last_flag are reused by the next segment
            asm volatile("bar.sync 1, %0;" ::"r"(CP_EPI_WARPS * 32) : "memory");
            nseg++;
#pragma unroll
            for (int pp = 0; pp < kParts; pp++)
#pragma unroll
                for (int i = 0; i < 16; i++) acc[pp][i] = 0.0f;
        }
    }
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
