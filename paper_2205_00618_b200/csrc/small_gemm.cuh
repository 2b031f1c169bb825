// small_gemm.cuh -- one-launch SIMT contraction for latency-bound sizes
// (C1: 256^3, every small acceptance graph).
//
// At C1 the work is ~1 us of FFMA on the whole chip; what costs is launches
// and DRAM round trips.  The register-blocked kernel (semiring_gemm.cuh)
// needs split-K plus a fold launch to put enough CTAs on the SMs there
// (14.3 us).  Here one CTA owns a 32 x TN output tile (TN = 16 or 32, picked
// so the grid covers the SMs) and its 8 warps split K among themselves:
// operand chunks arrive by cp.async (double-buffered, 128 k per chunk),
// warp w folds k-steps [w*16, w*16 + 16) of every chunk into a 4 x TN/4
// register block per lane, and the 8 warp partials meet in shared memory,
// folded in warp order (deterministic), epilogue fused, one store.
//
// Arithmetic per operator pair as in the reference VM's vop/vfma body
// (vm.py:112-136): (mul, add) is one FFMA per point; every other pair is
// combine then reduce with round-to-nearest FP32 ops, so (add, max|min) stays
// bit-identical to float32(reference_eval) (max/min are exact and the fold
// order does not matter for them).
//
// Preconditions (host, lsb_api.cu): A [M][K] with sa_k = 1, sa_m % 4 == 0;
// B [K][N] with sb_n = 1, sb_k % 4 == 0; batch strides % 4 == 0; both 16-B
// aligned; K % 4 == 0; N % 4 == 0; no beta inside the loop.  Rows / columns
// past M / N read clamped (valid) addresses and are never stored.
#pragma once

#include "maxplus_fast.cuh"   // cp_async16 / commit / wait

namespace lsb {

constexpr int kSgTM = 32, kSgKC = 128, kSgWarps = 8, kSgThreads = 256;
constexpr int kSgKW = kSgKC / kSgWarps;   // k-steps per warp per chunk (16)
constexpr int kSgApitch = kSgKC + 4;      // As[m][k]: 16-B rows, 2 rows 16 words apart per quarter-warp

template <int TN>
struct SgSmem {
    static constexpr int kA = kSgTM * kSgApitch;   // floats per A stage
    static constexpr int kB = kSgKC * TN;          // floats per B stage
    static constexpr int kStage = kA + kB;
    static constexpr size_t kBytes = sizeof(float) * 2 * kStage;
    static_assert(kSgWarps * kSgTM * TN <= 2 * kStage, "partials reuse the stage buffers");
};

template <int OPC, int OPR>
__device__ __forceinline__ float sg_step(float acc, float a, float b) {
    if constexpr (OPC == LSB_OP_MUL && OPR == LSB_OP_ADD) return fmaf(a, b, acc);
    else return Op<OPR>::apply(acc, Op<OPC>::apply(a, b));
}

template <int OPC, int OPR, int TN>
__global__ void __launch_bounds__(kSgThreads) small_gemm_kernel(const GemmArgs p) {
    using S = SgSmem<TN>;
    constexpr int CW = TN / 4;                     // columns per lane
    extern __shared__ __align__(16) float sg_smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int rg = lane >> 2, cg = lane & 3;       // rows rg*4 .. +3, columns cg*CW .. +CW-1
    const int64_t n_tiles = (p.N + TN - 1) / TN;
    const int64_t m0 = (blockIdx.x / n_tiles) * kSgTM, n0 = (blockIdx.x % n_tiles) * TN;
    const int64_t bz = blockIdx.y;
    const float *A = p.A + bz * p.sa_b;
    const float *B = p.B + bz * p.sb_b;

    // cp.async chunk assignment: A is 32 rows x 128 k = 1024 float4 (4 per
    // thread), B is 128 k x TN columns = 32*TN float4 (TN/8 per thread)
    auto issue = [&](int64_t k0, int stage) {
        float *As = sg_smem + stage * S::kStage;
        float *Bs = As + S::kA;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int e = t + j * kSgThreads;          // 0..1023
            const int r = e >> 5, kq = (e & 31) * 4;   // row, k offset
            const int64_t gr = min(m0 + r, p.M - 1);
            const int64_t gk = min(k0 + kq, p.K - 4);
            cp_async16(As + r * kSgApitch + kq, A + gr * p.sa_m + gk);
        }
#pragma unroll
        for (int j = 0; j < TN / 8; j++) {
            const int e = t + j * kSgThreads;          // 0 .. 32*TN - 1
            const int kr = e / (TN / 4), nq = (e % (TN / 4)) * 4;
            const int64_t gk = min(k0 + kr, p.K - 1);
            const int64_t gn = min(n0 + nq, p.N - 4);
            cp_async16(Bs + kr * TN + nq, B + gk * p.sb_k + gn);
        }
    };

    float acc[4][CW];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < CW; j++) acc[i][j] = Op<OPR>::identity();

    const int64_t chunks = (p.K + kSgKC - 1) / kSgKC;
    issue(0, 0);
    cp_async_commit();
    for (int64_t c = 0; c < chunks; c++) {
        if (c + 1 < chunks) issue((c + 1) * kSgKC, (int)((c + 1) & 1));
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const float *As = sg_smem + (c & 1) * S::kStage;
        const float *Bs = As + S::kA;
        const int kbase = warp * kSgKW;
        const int64_t krem = p.K - c * kSgKC - kbase;
        const int kvalid = krem < kSgKW ? (int)krem : kSgKW;   // ragged last chunk
        if (kvalid == kSgKW) {
#pragma unroll
            for (int k4 = 0; k4 < kSgKW; k4 += 4) {
                float4 a[4];
#pragma unroll
                for (int i = 0; i < 4; i++)
                    a[i] = *reinterpret_cast<const float4 *>(As + (rg * 4 + i) * kSgApitch + kbase + k4);
#pragma unroll
                for (int kk = 0; kk < 4; kk++) {
                    float b[CW];
#pragma unroll
                    for (int q = 0; q < CW; q += 4) {
                        const float4 v = *reinterpret_cast<const float4 *>(Bs + (kbase + k4 + kk) * TN + cg * CW + q);
                        b[q] = v.x; b[q + 1] = v.y; b[q + 2] = v.z; b[q + 3] = v.w;
                    }
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const float av = kk == 0 ? a[i].x : kk == 1 ? a[i].y : kk == 2 ? a[i].z : a[i].w;
#pragma unroll
                        for (int j = 0; j < CW; j++) acc[i][j] = sg_step<OPC, OPR>(acc[i][j], av, b[j]);
                    }
                }
            }
        } else {
            for (int kk = 0; kk < kvalid; kk++) {
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const float av = As[(rg * 4 + i) * kSgApitch + kbase + kk];
#pragma unroll
                    for (int j = 0; j < CW; j++)
                        acc[i][j] = sg_step<OPC, OPR>(acc[i][j], av, Bs[(kbase + kk) * TN + cg * CW + j]);
                }
            }
        }
        __syncthreads();   // stage (c & 1) is refilled by the next issue
    }
    cp_async_wait<0>();

    // warp partials -> smem [warp][row][col], then fold in warp order
    float *part = sg_smem;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < CW; j += 4)
            *reinterpret_cast<float4 *>(part + (warp * kSgTM + rg * 4 + i) * TN + cg * CW + j) =
                make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
    __syncthreads();
    float *C = p.C + bz * p.sc_b;
    for (int e = t; e < kSgTM * TN / 4; e += kSgThreads) {
        const int r = e / (TN / 4), cq = (e % (TN / 4)) * 4;
        float v[4];
        {
            const float4 x = *reinterpret_cast<const float4 *>(part + r * TN + cq);
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        }
#pragma unroll
        for (int w = 1; w < kSgWarps; w++) {
            const float4 x = *reinterpret_cast<const float4 *>(part + (w * kSgTM + r) * TN + cq);
            v[0] = Op<OPR>::apply(v[0], x.x); v[1] = Op<OPR>::apply(v[1], x.y);
            v[2] = Op<OPR>::apply(v[2], x.z); v[3] = Op<OPR>::apply(v[3], x.w);
        }
        const int64_t m = m0 + r, n = n0 + cq;
        if (m >= p.M) continue;
        if (n + 3 < p.N) {
            if (p.epi.n) apply_epilogue4(p.epi, v, bz, m, n, 0);
            if (p.c_vec) {
                *reinterpret_cast<float4 *>(C + m * p.sc_m + n) = make_float4(v[0], v[1], v[2], v[3]);
                continue;
            }
        } else if (p.epi.n) {
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (n + q < p.N) v[q] = apply_epilogue(p.epi, v[q], bz, m, n + q, 0);
        }
#pragma unroll
        for (int q = 0; q < 4; q++)
            if (n + q < p.N) C[m * p.sc_m + (n + q) * p.sc_n] = v[q];
    }
}

}  // namespace lsb
