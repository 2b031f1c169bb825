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

}  // namespace lsb
