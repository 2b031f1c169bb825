// maxplus_fast.cuh -- (add, max|min) stream-K contraction for row-major,
// 16-byte aligned operands (C2's layout): cp.async multi-stage tiles, no
// register staging, pointer-bumped addressing.
//
// Same arithmetic as semiring_streamk_kernel (semiring_gemm.cuh): each thread
// owns an 8x8 output block, two k steps fold into one 3-input max/min
// (FADD2 with a broadcast scalar + FMNMX3), partial tiles of a stream-K
// segment merge into C (pre-filled with the identity) through exact integer
// atomics -- so the result is bit-identical to the reference's sequential
// max over k (max is exact and order-free).  What changes is the per-slice
// overhead: the generic kernel's slice is 8 deep and re-derives 64-bit
// addresses, layout branches and an smem transpose for A every slice
// (~30 % of issued instructions at C2, profiles/r01_ncu_c2_streamk.json);
// here a slice is 16 deep, A stays k-contiguous in smem ([m][k], read as
// k-pairs), both tiles arrive by cp.async straight from global memory, and
// the loop body is the math plus ~20 instructions.
//
// Preconditions (checked by the host, lsb_api.cu): A [M][K] with sa_k = 1,
// sa_m % 4 == 0; B [K][N] with sb_n = 1, sb_k % 4 == 0; both 16-B aligned;
// N % 4 == 0; K % 16 == 0; batch 1.  Rows/columns past M/N read clamped
// (valid) addresses and are never stored.
#pragma once

#include "semiring_gemm.cuh"

#ifndef LSB_MP_STAGES
#define LSB_MP_STAGES 3
#endif

namespace lsb {

constexpr int kMpBM = 128, kMpBN = 128, kMpBK = 16, kMpStages = LSB_MP_STAGES;
constexpr int kMpApitch = kMpBK + 4;   // [m][k] rows of 20 floats (80 B: 16-B aligned, conflict-free)
constexpr int kMpStageFloats = kMpBM * kMpApitch + kMpBK * kMpBN;
constexpr size_t kMpSmemBytes = sizeof(float) * kMpStages * kMpStageFloats;

__device__ __forceinline__ void cp_async16(float *smem_dst, const float *gsrc) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// one output tile's contribution from slices [k0 / 16, k0 / 16 + nsl) into
// acc (pre-set to the identity); every stage of the smem ring is free on
// entry and on exit
template <int OPR>
__device__ __forceinline__ void mp_tile_slices(const GemmArgs &p, float *mp_smem, int64_t m0, int64_t n0,
                                               int64_t k0, int nsl, float2 (&acc)[8][4]) {
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    // this thread's cp.async chunks: A rows (t >> 2) and 64 + (t >> 2), k
    // quarter t & 3; B k rows (t >> 5) and 8 + (t >> 5), column quad t & 31
    const int a_row = t >> 2, a_kq = (t & 3) * 4;
    const int b_k = t >> 5, b_nq = (t & 31) * 4;
    const int64_t ra0 = min(m0 + a_row, p.M - 1), ra1 = min(m0 + 64 + a_row, p.M - 1);
    const float *ga0 = p.A + ra0 * p.sa_m + k0 + a_kq;
    const float *ga1 = p.A + ra1 * p.sa_m + k0 + a_kq;
    const float *gb0 = p.B + (k0 + b_k) * p.sb_k + min(n0 + b_nq, p.N - 4);
    const int64_t b_step = kMpBK * p.sb_k, b_half = 8 * p.sb_k;

    auto issue = [&](int slice, int stage) {
        float *As = mp_smem + stage * kMpStageFloats;
        float *Bs = As + kMpBM * kMpApitch;
        cp_async16(As + a_row * kMpApitch + a_kq, ga0 + slice * kMpBK);
        cp_async16(As + (64 + a_row) * kMpApitch + a_kq, ga1 + slice * kMpBK);
        cp_async16(Bs + b_k * kMpBN + b_nq, gb0 + slice * b_step);
        cp_async16(Bs + (8 + b_k) * kMpBN + b_nq, gb0 + slice * b_step + b_half);
    };

#pragma unroll
    for (int s = 0; s < kMpStages - 1; s++) {
        if (s < nsl) issue(s, s);
        cp_async_commit();
    }
    for (int sl = 0; sl < nsl; sl++) {
        cp_async_wait<kMpStages - 2>();
        __syncthreads();   // slice sl visible to all; stage (sl - 1) % S free
        if (sl + kMpStages - 1 < nsl) issue(sl + kMpStages - 1, (sl + kMpStages - 1) % kMpStages);
        cp_async_commit();
        const float *As = mp_smem + (sl % kMpStages) * kMpStageFloats;
        const float *Bs = As + kMpBM * kMpApitch;
#pragma unroll
        for (int kk = 0; kk < kMpBK; kk += 2) {
            float2 a[8];
#pragma unroll
            for (int i = 0; i < 8; i++)
                a[i] = *reinterpret_cast<const float2 *>(As + row_of<8>(ty, i) * kMpApitch + kk);
            float b0[8], b1[8];
            {
                const float4 x0 = *reinterpret_cast<const float4 *>(Bs + kk * kMpBN + tx * 4);
                const float4 x1 = *reinterpret_cast<const float4 *>(Bs + kk * kMpBN + 64 + tx * 4);
                const float4 y0 = *reinterpret_cast<const float4 *>(Bs + (kk + 1) * kMpBN + tx * 4);
                const float4 y1 = *reinterpret_cast<const float4 *>(Bs + (kk + 1) * kMpBN + 64 + tx * 4);
                b0[0] = x0.x; b0[1] = x0.y; b0[2] = x0.z; b0[3] = x0.w;
                b0[4] = x1.x; b0[5] = x1.y; b0[6] = x1.z; b0[7] = x1.w;
                b1[0] = y0.x; b1[1] = y0.y; b1[2] = y0.z; b1[3] = y0.w;
                b1[4] = y1.x; b1[5] = y1.y; b1[6] = y1.z; b1[7] = y1.w;
            }
#pragma unroll
            for (int i = 0; i < 8; i++) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float2 s = __fadd2_rn(make_float2(a[i].x, a[i].x), make_float2(b0[2 * j], b0[2 * j + 1]));
                    const float2 v = __fadd2_rn(make_float2(a[i].y, a[i].y), make_float2(b1[2 * j], b1[2 * j + 1]));
                    acc[i][j].x = Op<OPR>::apply(acc[i][j].x, Op<OPR>::apply(s.x, v.x));
                    acc[i][j].y = Op<OPR>::apply(acc[i][j].y, Op<OPR>::apply(s.y, v.y));
                }
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();   // every stage free again
}

template <int OPR>
__device__ __forceinline__ void mp_acc_init(float2 (&acc)[8][4]) {
    const float id = Op<OPR>::identity();
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = make_float2(id, id);
}

// stream-K: partial tiles merge into C (pre-filled with the identity)
// through exact integer atomics
template <int OPR>
__global__ void __launch_bounds__(kThreads, 2) maxplus_streamk_fast_kernel(const GemmArgs p) {
    extern __shared__ __align__(16) float mp_smem[];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t m_tiles = (p.M + kMpBM - 1) / kMpBM, n_tiles = (p.N + kMpBN - 1) / kMpBN;
    const int64_t kslices = p.K / kMpBK;
    const int64_t units = m_tiles * n_tiles * kslices;
    const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    for (int64_t u = u0; u < u1;) {
        const int64_t tile = u / kslices, ks = u % kslices;
        const int64_t seg_end = min(u1, (tile + 1) * kslices);
        const int64_t m0 = (tile / n_tiles) * kMpBM, n0 = (tile % n_tiles) * kMpBN;
        float2 acc[8][4];
        mp_acc_init<OPR>(acc);
        mp_tile_slices<OPR>(p, mp_smem, m0, n0, ks * kMpBK, (int)(seg_end - u), acc);
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int64_t m = m0 + row_of<8>(ty, i);
            if (m >= p.M) continue;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int64_t n = n0 + col_of(tx, j);
                if (n >= p.N) continue;
                const float v = (j & 1) ? acc[i][j >> 1].y : acc[i][j >> 1].x;
                float *dst = p.C + m * p.sc_m + n * p.sc_n;
                if constexpr (OPR == LSB_OP_MAX) atomic_max_f32(dst, v);
                else atomic_min_f32(dst, v);
            }
        }
        u = seg_end;
    }
}

// split-K inside a thread-block cluster: the cluster's CTAs (rank r of
// S = %cluster_nctarank) take the K slices [r*ks/S, (r+1)*ks/S) of one output
// tile, publish their partial tiles in their own shared memory, and after a
// cluster barrier each reduces a row band across all S partials through
// distributed shared memory and stores it -- one launch, no identity fill,
// no global atomics, and max/min is exact in any order.
constexpr int kMpCPitch = kMpBN + 4;   // partial tile rows in smem
constexpr int kMpMaxCluster = 16;      // non-portable cluster sizes up to 16
constexpr size_t kMpClusterSmemBytes =
    sizeof(float) * (kMpBM * kMpCPitch > kMpStages * kMpStageFloats ? kMpBM * kMpCPitch : kMpStages * kMpStageFloats);

__device__ __forceinline__ uint32_t mp_cluster_nrank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mp_cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void mp_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 16 bytes of a peer CTA's shared memory (same offset as `local` here).
// Not volatile: the loads of one fold are independent and may overlap; the
// cluster barriers around the fold order them against the writes.
__device__ __forceinline__ float4 mp_ld_dsmem4(const float *local, uint32_t rank) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local), r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    float4 v;
    asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(r));
    return v;
}

template <int OPR>
__global__ void __launch_bounds__(kThreads, 2) maxplus_cluster_kernel(const GemmArgs p) {
    extern __shared__ __align__(16) float mp_smem[];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const uint32_t S = mp_cluster_nrank(), r = mp_cluster_rank();
    const int64_t n_tiles = (p.N + kMpBN - 1) / kMpBN;
    const int64_t tile = blockIdx.x / S;
    const int64_t m0 = (tile / n_tiles) * kMpBM, n0 = (tile % n_tiles) * kMpBN;
    const int64_t kslices = p.K / kMpBK;
    const int64_t s0 = kslices * r / S, s1 = kslices * (r + 1) / S;
    float2 acc[8][4];
    mp_acc_init<OPR>(acc);
    mp_tile_slices<OPR>(p, mp_smem, m0, n0, s0 * kMpBK, (int)(s1 - s0), acc);
    // publish the partial tile (the stage ring is free)
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int h = 0; h < 2; h++)
            *reinterpret_cast<float4 *>(mp_smem + row_of<8>(ty, i) * kMpCPitch + h * 64 + tx * 4) =
                make_float4(acc[i][2 * h].x, acc[i][2 * h].y, acc[i][2 * h + 1].x, acc[i][2 * h + 1].y);
    mp_cluster_sync();
    // row band [b0, b1) of the tile: fold the S partials, store
    const int b0 = (int)(kMpBM * r / S), b1 = (int)(kMpBM * (r + 1) / S);
    constexpr int kQ = kMpBN / 4;   // float4 column quads per row
    for (int e = b0 * kQ + (int)threadIdx.x; e < b1 * kQ; e += kThreads) {
        const int row = e / kQ, c4 = (e % kQ) * 4;
        const int64_t m = m0 + row, n = n0 + c4;
        const float *src = mp_smem + row * kMpCPitch + c4;
        float4 w[kMpMaxCluster];
#pragma unroll
        for (int q = 0; q < kMpMaxCluster; q++)
            if (q < (int)S) w[q] = mp_ld_dsmem4(src, (uint32_t)q);
        const float id = Op<OPR>::identity();
        float4 v = make_float4(id, id, id, id);
#pragma unroll
        for (int q = 0; q < kMpMaxCluster; q++) {
            if (q < (int)S) {
                v.x = Op<OPR>::apply(v.x, w[q].x);
                v.y = Op<OPR>::apply(v.y, w[q].y);
                v.z = Op<OPR>::apply(v.z, w[q].z);
                v.w = Op<OPR>::apply(v.w, w[q].w);
            }
        }
        if (m < p.M) {
            float *dst = p.C + m * p.sc_m;
            if (p.c_vec && n + 3 < p.N) {
                *reinterpret_cast<float4 *>(dst + n) = v;
            } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (n + q < p.N) dst[(n + q) * p.sc_n] = vv[q];
            }
        }
    }
    mp_cluster_sync();   // peers may still read this CTA's partial tile
}

// stream-K with an in-kernel fixup: a persistent grid of G co-resident CTAs
// (cooperative launch, 2 per SM) splits the tiles x 16-deep k-slices work
// into G equal ranges (C2: 4096 units / 296 CTAs, every SM gets the same
// 27-28 slices -- the cluster split-K leaves 40 SMs with one CTA and the
// rest with two).  A range is at most two tile segments: the first, if it
// starts mid-tile, is published as a partial tile (plain stores to a
// per-CTA workspace slot, then a release flag stamped with the launch
// epoch); the segment holding a tile's slice 0 is the tile's owner, which
// after its own slices waits (acquire) on every later CTA whose range
// reaches into the tile, folds their partials and stores C.  Contributors
// publish before they wait on anything, so with every CTA resident there
// is no cycle.  One launch, no fill, no atomics; max/min are exact in any
// order, so C is bit-identical to the sequential reference.
__device__ __forceinline__ void mp_flag_release(int *f, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ int mp_flag_acquire(const int *f) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    return v;
}

// Timeline probe (tools/dbg/mp_trace.cu defines LSB_MP_TRACE): thread 0 of
// every CTA stamps %globaltimer at phase boundaries; nothing in product builds.
#ifdef LSB_MP_TRACE
__device__ long long *g_mp_trace;   // [ctas][16]: smid, then (tag << 56 | ns) stamps
__device__ __forceinline__ void mp_stamp(int &n, int tag) {
    if (threadIdx.x == 0 && n < 16) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_mp_trace[blockIdx.x * 16 + n++] = ((long long)tag << 56) | (t & 0x00ffffffffffffffll);
    }
}
#define MP_STAMP(tag) mp_stamp(mp_tn, tag)
#else
#define MP_STAMP(tag)
#endif

template <int OPR>
__global__ void __launch_bounds__(kThreads, 2) maxplus_fixup_kernel(const GemmArgs p, float4 *part, int *flags,
                                                                     int epoch) {
    extern __shared__ __align__(16) float mp_smem[];
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    const int64_t n_tiles = (p.N + kMpBN - 1) / kMpBN, m_tiles = (p.M + kMpBM - 1) / kMpBM;
    const int64_t ks = p.K / kMpBK;
    const int64_t U = m_tiles * n_tiles * ks, G = gridDim.x, b = blockIdx.x;
    const int64_t u0 = U * b / G, u1 = U * (b + 1) / G;
    for (int64_t u = u0; u < u1;) {
        const int64_t tile = u / ks, s0 = u % ks, tile_end = (tile + 1) * ks;
        const int64_t seg_end = min(u1, tile_end);
        const int64_t m0 = (tile / n_tiles) * kMpBM, n0 = (tile % n_tiles) * kMpBN;
        float2 acc[8][4];
        mp_acc_init<OPR>(acc);
        mp_tile_slices<OPR>(p, mp_smem, m0, n0, s0 * kMpBK, (int)(seg_end - u), acc);
        if (s0 != 0) {
            // contributor: this CTA's (only) partial tile, thread-major float4s
            float4 *dst = part + b * (16 * kThreads);
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int h = 0; h < 2; h++)
                    __stcg(dst + (i * 2 + h) * kThreads + t,
                           make_float4(acc[i][2 * h].x, acc[i][2 * h].y, acc[i][2 * h + 1].x, acc[i][2 * h + 1].y));
            __syncthreads();
            if (t == 0) {
                __threadfence();
                mp_flag_release(flags + b, epoch);
            }
        } else {
            // owner: fold the partials of the later CTAs reaching into the tile
            for (int64_t c = b + 1; seg_end < tile_end && c < G && U * c / G < tile_end; c++) {
                if (t == 0)
                    while (mp_flag_acquire(flags + c) != epoch) __nanosleep(32);
                __syncthreads();
                const float4 *src = part + c * (16 * kThreads);
#pragma unroll
                for (int i = 0; i < 8; i++)
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const float4 w = __ldcg(src + (i * 2 + h) * kThreads + t);
                        acc[i][2 * h].x = Op<OPR>::apply(acc[i][2 * h].x, w.x);
                        acc[i][2 * h].y = Op<OPR>::apply(acc[i][2 * h].y, w.y);
                        acc[i][2 * h + 1].x = Op<OPR>::apply(acc[i][2 * h + 1].x, w.z);
                        acc[i][2 * h + 1].y = Op<OPR>::apply(acc[i][2 * h + 1].y, w.w);
                    }
            }
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int64_t m = m0 + row_of<8>(ty, i);
                if (m >= p.M) continue;
                float *dst = p.C + m * p.sc_m;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int64_t n = n0 + h * 64 + tx * 4;
                    const float v[4] = {acc[i][2 * h].x, acc[i][2 * h].y, acc[i][2 * h + 1].x, acc[i][2 * h + 1].y};
                    if (p.c_vec && n + 3 < p.N) {
                        *reinterpret_cast<float4 *>(dst + n) = make_float4(v[0], v[1], v[2], v[3]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; q++)
                            if (n + q < p.N) dst[(n + q) * p.sc_n] = v[q];
                    }
                }
            }
        }
        u = seg_end;
    }
}

// ---------------------------------------------------------------------------
// "duo" fixup kernel: ONE 512-thread CTA per SM, two 256-thread groups.
//
// Why (B200 timeline of maxplus_fixup_kernel, tools/dbg/mp_trace.cu): with two
// 256-thread CTAs per SM and equal ranges the warp scheduler gives one CTA
// ~65 % of the issue slots, so it finishes its 13.8 slices at ~45 us while the
// other ends at ~62 us after a solo phase that reaches only ~71 % of the
// FADD2 + FMNMX3 ceiling (2 warps per scheduler); static weighting of the
// ranges measured slower (which CTA is favoured is not fixed).  Here both
// groups work on the SAME segment and pull its slices from a shared-memory
// counter, each with its own cp.async ring and accumulators, so whichever
// group the scheduler favours simply takes more slices and both finish within
// one slice of each other.  At the end of a segment the groups swap halves of
// their accumulators through shared memory (group g ends up with rows
// [64 g, 64 g + 64) of the merged tile) and BOTH run the fixup on their half:
// publish / fold / store use all 512 threads.  Ranges are twice as long as the
// two-CTA kernel's, so a tile has 2-3 contributors instead of 4-5.  A partial's
// release flag is deferred to the top of the CTA's next segment (only thread
// 0's group waits for the stores to land), and an owner folds two published
// partials per pass.
// Same protocol otherwise (epoch flags, contributors publish before anyone
// waits, cooperative launch); max/min are exact in any order: bit-identical.
constexpr int kDuoThreads = 2 * kThreads;
// slice depth BK (8, 16 or 32): what the groups pull from the counter.  Every
// slice costs a group barrier and a pop (~450 cycles measured), and at the end
// of a segment the faster group waits for the slower one's last slice: 32-deep
// slices measured best on C2 (0.0745 ms; 16: 0.0764; 8: 0.0823).
template <int BK>
struct DuoCfg {
    static constexpr int kStages = BK == 8 ? 5 : 3;
    static constexpr int kApitch = BK + 4;
    static constexpr int kStageFloats = kMpBM * kApitch + BK * kMpBN;
    static constexpr int kRingFloats = kStages * kStageFloats;
    // the accumulator exchange of a segment's end reuses the rings (each group sends
    // into its own, free by then: 8 float4 slots x 256 threads = 32 KB)
    static constexpr size_t kSmemBytes = sizeof(float) * (2 * kRingFloats);
    static_assert(sizeof(float) * kRingFloats >= sizeof(float4) * 8 * kThreads, "ring holds the exchange");
};

__device__ __forceinline__ void mp_group_bar(int g) { asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory"); }

// this group's share of slices [0, nsl) of the segment starting at k0, pulled
// from *next (shared, zeroed before the call) -- q: this group's staged slice
// indices (shared, kStages ints).  Every stage of the ring is free on exit.
template <int OPR, int BK>
__device__ __forceinline__ void mp_group_slices(const GemmArgs &p, float *ring, int64_t m0, int64_t n0, int64_t k0,
                                                int nsl, float2 (&acc)[8][4], int *next, volatile int *q, int g) {
    using Cf = DuoCfg<BK>;
    constexpr int S = Cf::kStages, kPer = BK / 8;   // 16-B chunks per thread and operand
    const int t = threadIdx.x & (kThreads - 1), tx = t & 15, ty = t >> 4;
    // 16-B chunk j of this thread: A row t / (BK / 4) + j * (1024 / BK), k quad t % (BK / 4);
    // B k row (t >> 5) + 8 j, column quad t & 31.  Addresses are rebuilt per
    // issue from two base pointers (per-chunk pointers spill at BK = 32).
    constexpr int kQuads = BK / 4, kRowsPerPass = kThreads / kQuads;
    const int a_row0 = t / kQuads, a_kq = (t % kQuads) * 4;
    const int b_k0 = t >> 5, b_nq = (t & 31) * 4;
    const float *ga = p.A + k0 + a_kq;
    const float *gb = p.B + (k0 + b_k0) * p.sb_k + min(n0 + b_nq, p.N - 4);
    const int64_t b_step = BK * p.sb_k;

    auto issue = [&](int slice, int stage) {
        float *st = ring + stage * Cf::kStageFloats;
#pragma unroll
        for (int j = 0; j < kPer; j++) {
            const int a_row = a_row0 + j * kRowsPerPass;
            cp_async16(st + a_row * Cf::kApitch + a_kq, ga + min(m0 + a_row, p.M - 1) * p.sa_m + slice * BK);
            cp_async16(st + kMpBM * Cf::kApitch + (b_k0 + 8 * j) * kMpBN + b_nq,
                       gb + slice * b_step + (int64_t)(8 * j) * p.sb_k);
        }
    };

    if (t == 0) {
#pragma unroll
        for (int s = 0; s < S - 1; s++) q[s] = atomicAdd(next, 1);
    }
    mp_group_bar(g);
#pragma unroll
    for (int s = 0; s < S - 1; s++) {
        const int sl = q[s];
        if (sl < nsl) issue(sl, s);
        cp_async_commit();
    }
    for (int it = 0;; it++) {
        const int cur = q[it % S];
        if (cur >= nsl) break;   // pops are monotonic: nothing later is staged either
        if (t == 0) q[(it + S - 1) % S] = atomicAdd(next, 1);
        cp_async_wait<S - 2>();
        mp_group_bar(g);   // slice cur visible to the group; stage (it - 1) % S free; next pop visible
        {
            const int nxt = q[(it + S - 1) % S];
            if (nxt < nsl) issue(nxt, (it + S - 1) % S);
            cp_async_commit();
        }
        const float *As = ring + (it % S) * Cf::kStageFloats;
        const float *Bs = As + kMpBM * Cf::kApitch;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 2) {
            float2 a[8];
#pragma unroll
            for (int i = 0; i < 8; i++)
                a[i] = *reinterpret_cast<const float2 *>(As + row_of<8>(ty, i) * Cf::kApitch + kk);
            float b0[8], b1[8];
            {
                const float4 x0 = *reinterpret_cast<const float4 *>(Bs + kk * kMpBN + tx * 4);
                const float4 x1 = *reinterpret_cast<const float4 *>(Bs + kk * kMpBN + 64 + tx * 4);
                const float4 y0 = *reinterpret_cast<const float4 *>(Bs + (kk + 1) * kMpBN + tx * 4);
                const float4 y1 = *reinterpret_cast<const float4 *>(Bs + (kk + 1) * kMpBN + 64 + tx * 4);
                b0[0] = x0.x; b0[1] = x0.y; b0[2] = x0.z; b0[3] = x0.w;
                b0[4] = x1.x; b0[5] = x1.y; b0[6] = x1.z; b0[7] = x1.w;
                b1[0] = y0.x; b1[1] = y0.y; b1[2] = y0.z; b1[3] = y0.w;
                b1[4] = y1.x; b1[5] = y1.y; b1[6] = y1.z; b1[7] = y1.w;
            }
#pragma unroll
            for (int i = 0; i < 8; i++) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float2 s = __fadd2_rn(make_float2(a[i].x, a[i].x), make_float2(b0[2 * j], b0[2 * j + 1]));
                    const float2 v = __fadd2_rn(make_float2(a[i].y, a[i].y), make_float2(b1[2 * j], b1[2 * j + 1]));
                    acc[i][j].x = Op<OPR>::apply(acc[i][j].x, Op<OPR>::apply(s.x, v.x));
                    acc[i][j].y = Op<OPR>::apply(acc[i][j].y, Op<OPR>::apply(s.y, v.y));
                }
            }
        }
    }
    cp_async_wait<0>();
    mp_group_bar(g);   // every stage free again
}

// group GI's tail of a segment (GI is the compile-time group index, so the
// accumulator halves are addressed statically)
template <int OPR, int GI>
struct MpDuoTail {
    static constexpr int kOwn = 4 * GI, kOther = 4 * (1 - GI);
    // send the other group's rows
    static __device__ __forceinline__ void send(float4 *xch, int t, const float2 (&acc)[8][4]) {
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int h = 0; h < 2; h++)
                xch[(i * 2 + h) * kThreads + t] = make_float4(acc[kOther + i][2 * h].x, acc[kOther + i][2 * h].y,
                                                                       acc[kOther + i][2 * h + 1].x, acc[kOther + i][2 * h + 1].y);
    }
    static __device__ __forceinline__ void fold4(float2 (&acc)[8][4], int i, int h, const float4 w) {
        acc[kOwn + i][2 * h].x = Op<OPR>::apply(acc[kOwn + i][2 * h].x, w.x);
        acc[kOwn + i][2 * h].y = Op<OPR>::apply(acc[kOwn + i][2 * h].y, w.y);
        acc[kOwn + i][2 * h + 1].x = Op<OPR>::apply(acc[kOwn + i][2 * h + 1].x, w.z);
        acc[kOwn + i][2 * h + 1].y = Op<OPR>::apply(acc[kOwn + i][2 * h + 1].y, w.w);
    }
    // fold the rows the other group sent
    static __device__ __forceinline__ void recv(const float4 *xch, int t, float2 (&acc)[8][4]) {
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int h = 0; h < 2; h++) fold4(acc, i, h, xch[(i * 2 + h) * kThreads + t]);
    }
    // partial tile slots of this group: (kOwn + i) * 2 + h
    static __device__ __forceinline__ void publish(float4 *dst, int t, const float2 (&acc)[8][4]) {
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int h = 0; h < 2; h++)
                __stcg(dst + ((kOwn + i) * 2 + h) * kThreads + t,
                       make_float4(acc[kOwn + i][2 * h].x, acc[kOwn + i][2 * h].y, acc[kOwn + i][2 * h + 1].x,
                                   acc[kOwn + i][2 * h + 1].y));
    }
    static __device__ __forceinline__ void fold_part(const float4 *src, int t, float2 (&acc)[8][4]) {
        float4 w[8];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int h = 0; h < 2; h++) w[i * 2 + h] = __ldcg(src + ((kOwn + i) * 2 + h) * kThreads + t);
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int h = 0; h < 2; h++) fold4(acc, i, h, w[i * 2 + h]);
    }
    static __device__ __forceinline__ void fold_part2(const float4 *s0, const float4 *s1, int t, float2 (&acc)[8][4]) {
        float4 w[8], x[8];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                w[i * 2 + h] = __ldcg(s0 + ((kOwn + i) * 2 + h) * kThreads + t);
                x[i * 2 + h] = __ldcg(s1 + ((kOwn + i) * 2 + h) * kThreads + t);
            }
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                fold4(acc, i, h, w[i * 2 + h]);
                fold4(acc, i, h, x[i * 2 + h]);
            }
    }
    static __device__ __forceinline__ void store(const GemmArgs &p, int64_t m0, int64_t n0, int tx, int ty,
                                                 const float2 (&acc)[8][4]) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int64_t m = m0 + row_of<8>(ty, kOwn + i);
            if (m >= p.M) continue;
            float *dst = p.C + m * p.sc_m;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int64_t n = n0 + h * 64 + tx * 4;
                const float v[4] = {acc[kOwn + i][2 * h].x, acc[kOwn + i][2 * h].y, acc[kOwn + i][2 * h + 1].x,
                                    acc[kOwn + i][2 * h + 1].y};
                if (p.c_vec && n + 3 < p.N) {
                    *reinterpret_cast<float4 *>(dst + n) = make_float4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (n + q < p.N) dst[(n + q) * p.sc_n] = v[q];
                }
            }
        }
    }
};

template <int OPR, int BK>
__global__ void __launch_bounds__(kDuoThreads, 1) maxplus_duo_kernel(const GemmArgs p, float4 *part, int *flags,
                                                                      int epoch) {
    using Cf = DuoCfg<BK>;
    extern __shared__ __align__(16) float mp_smem[];
    __shared__ int s_next;
    __shared__ int s_q[2][Cf::kStages];
    const int g = threadIdx.x >> 8, t = threadIdx.x & (kThreads - 1), tx = t & 15, ty = t >> 4;
    float *ring = mp_smem + g * Cf::kRingFloats;
    // exchange areas: a group sends into its own ring and receives from the other's
    float4 *xch_mine = reinterpret_cast<float4 *>(ring);
    const float4 *xch_other = reinterpret_cast<const float4 *>(mp_smem + (1 - g) * Cf::kRingFloats);
    const int64_t n_tiles = (p.N + kMpBN - 1) / kMpBN, m_tiles = (p.M + kMpBM - 1) / kMpBM;
    const int64_t ks = p.K / BK;
    const int64_t U = m_tiles * n_tiles * ks, G = gridDim.x, b = blockIdx.x;
    const int64_t u0 = U * b / G, u1 = U * (b + 1) / G;
#ifdef LSB_MP_TRACE
    int mp_tn = 1;
    if (threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_mp_trace[b * 16] = sm;
    }
#endif
    MP_STAMP(1);   // start
    bool release_due = false;   // partial stored, flag not yet released (uniform)
    for (int64_t u = u0; u < u1;) {
        const int64_t tile = u / ks, s0 = u % ks, tile_end = (tile + 1) * ks;
        const int64_t seg_end = min(u1, tile_end);
        const int64_t m0 = (tile / n_tiles) * kMpBM, n0 = (tile % n_tiles) * kMpBN;
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();   // also: the previous segment's exchange reads and partial stores are done
        if (release_due) {
            // the previous segment's partial: every thread's stores precede the
            // barrier above, so thread 0's release publishes them all.  Done
            // here, not right after the stores: the release waits for the
            // stores to land (~1-2 us) and only delays thread 0's group, whose
            // slices the other group picks up meanwhile.
            if (threadIdx.x == 0) mp_flag_release(flags + b, epoch);
            release_due = false;
            MP_STAMP(3);   // published
        }
        float2 acc[8][4];
        mp_acc_init<OPR>(acc);
        mp_group_slices<OPR, BK>(p, ring, m0, n0, s0 * BK, (int)(seg_end - u), acc, &s_next, s_q[g], g);
        MP_STAMP(2);   // group 0's slices done
        if (g == 0) MpDuoTail<OPR, 0>::send(xch_mine, t, acc);
        else MpDuoTail<OPR, 1>::send(xch_mine, t, acc);
        __syncthreads();
        if (g == 0) MpDuoTail<OPR, 0>::recv(xch_other, t, acc);
        else MpDuoTail<OPR, 1>::recv(xch_other, t, acc);
        MP_STAMP(6);   // halves merged
        if (s0 != 0) {
            // contributor: this CTA's (only) partial tile, thread-major float4s
            float4 *dst = part + b * (16 * kThreads);
            if (g == 0) MpDuoTail<OPR, 0>::publish(dst, t, acc);
            else MpDuoTail<OPR, 1>::publish(dst, t, acc);
            release_due = true;
        } else {
            // owner: fold the partials of the later CTAs reaching into the tile,
            // two at a time when both are already published
            int64_t c = b + 1;
            int nc = 0;
            if (seg_end < tile_end)
                while (c + nc < G && U * (c + nc) / G < tile_end) nc++;
            while (nc > 0) {
                if (threadIdx.x == 0) {
                    while (mp_flag_acquire(flags + c) != epoch) __nanosleep(32);
                    s_next = (nc > 1 && mp_flag_acquire(flags + c + 1) == epoch) ? 2 : 1;
                }
                __syncthreads();
                const int r = s_next;
                __syncthreads();   // everyone has read it: thread 0 may rewrite s_next
                MP_STAMP(4);   // r contributors ready
                const float4 *src = part + c * (16 * kThreads);
                if (r == 2) {
                    if (g == 0) MpDuoTail<OPR, 0>::fold_part2(src, src + 16 * kThreads, t, acc);
                    else MpDuoTail<OPR, 1>::fold_part2(src, src + 16 * kThreads, t, acc);
                } else {
                    if (g == 0) MpDuoTail<OPR, 0>::fold_part(src, t, acc);
                    else MpDuoTail<OPR, 1>::fold_part(src, t, acc);
                }
                c += r;
                nc -= r;
            }
            if (g == 0) MpDuoTail<OPR, 0>::store(p, m0, n0, tx, ty, acc);
            else MpDuoTail<OPR, 1>::store(p, m0, n0, tx, ty, acc);
            MP_STAMP(5);   // tile stored
        }
        u = seg_end;
    }
    if (release_due) {
        __syncthreads();
        if (threadIdx.x == 0) mp_flag_release(flags + b, epoch);
        MP_STAMP(3);
    }
}

}  // namespace lsb
