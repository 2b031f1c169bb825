// nest_fast.cuh -- the affine loop nest (affine_nest.cuh) for the shapes the
// acceptance nests have: at most 4 output dims, 3 reduction dims, 2 operands,
// 2 guards per operand, every offset inside 32 bits.  Same arithmetic and
// order as the general kernel (combine left to right, beta, reduce from the
// identity, epilogue), so results are bit-identical to it; what changes is
// the addressing cost, which bound the general kernel (ncu: ~790 warp
// instructions per max-pool output, 5-12 % of HBM bandwidth):
//
//  * nest_rows_kernel: a CTA is TX x TY threads, TX lanes on consecutive
//    points of the innermost output dim (coalesced stores, and coalesced loads
//    for every operand whose innermost coefficient is 1), TY rows of the outer
//    dims.  The outer coordinates are decoded once per row (two 32-bit
//    divisions), a thread then walks its row in steps of the grid width, four
//    points per trip with their loads independent.  The reduction space is
//    three nested 32-bit loops with running addresses.  Templated on the
//    operand count, on whether any guard exists and on whether there is a
//    reduction, so reduction-free unguarded nests (broadcast_add) compile to
//    load / op / store.
//  * nest_transpose_kernel: a reduction-free single-operand nest whose operand
//    is contiguous along another output dim than the output is (transpose,
//    any permutation) goes through 32 x 32 shared-memory tiles so both sides
//    move whole 128-byte lines.
#pragma once

#include "lsb_common.cuh"

namespace lsb {

constexpr int kNfOut = 4, kNfRed = 3, kNfOps = 2, kNfGuards = 2;

struct NfAffine {
    int base;
    int co[kNfOut];   // output dims, right-aligned (co[3] = innermost)
    int cr[kNfRed];   // reduction dims, right-aligned
};

struct NfOperand {
    const float *ptr;
    NfAffine addr;
    int n_guards;
    NfAffine guard[kNfGuards];
    unsigned guard_size[kNfGuards];
    float fill;
};

struct NestFastArgs {
    int eo[kNfOut], er[kNfRed];   // extents, right-aligned, padded with 1
    int shift;                    // kNfOut - n_out: epilogue coordinate k is padded dim k + shift
    int n_rows;                   // eo[0] * eo[1] * eo[2]
    NfOperand op[kNfOps];
    float *out;
    NfAffine out_addr;
    float beta;
    int combine, reduce;
    EpiStages epi;
    // transpose kernel: q = the operand's contiguous output dim (0..2), the two batch dims
    int tq, tb0, tb1;
};

__device__ __forceinline__ int nf_dot3(const int (&co)[kNfOut], int p0, int p1, int p2) {
    return co[0] * p0 + co[1] * p1 + co[2] * p2;
}

template <int NOPS, bool GUARDS, bool RED>
__device__ __forceinline__ float nf_point(const NestFastArgs &p, const int (&ab)[kNfOps],
                                          const int (&gb)[kNfOps][kNfGuards], int i) {
    int a[NOPS], g[NOPS][kNfGuards];
#pragma unroll
    for (int o = 0; o < NOPS; o++) {
        a[o] = ab[o] + p.op[o].addr.co[3] * i;
        if (GUARDS) {
#pragma unroll
            for (int q = 0; q < kNfGuards; q++) g[o][q] = gb[o][q] + p.op[o].guard[q].co[3] * i;
        }
    }
    auto term = [&](int d0, int d1, int d2) {
        float t = 0.0f;
#pragma unroll
        for (int o = 0; o < NOPS; o++) {
            const NfOperand &od = p.op[o];
            bool ok = true;
            if (GUARDS) {
#pragma unroll
                for (int q = 0; q < kNfGuards; q++)
                    if (q < od.n_guards) {
                        const int gv = g[o][q] + (RED ? od.guard[q].cr[0] * d0 + od.guard[q].cr[1] * d1 +
                                                            od.guard[q].cr[2] * d2
                                                      : 0);
                        ok = ok && (unsigned)gv < od.guard_size[q];
                    }
            }
            const int off = a[o] + (RED ? od.addr.cr[0] * d0 + od.addr.cr[1] * d1 + od.addr.cr[2] * d2 : 0);
            const float v = ok ? __ldg(od.ptr + off) : od.fill;
            t = (o == 0) ? v : op_rt(p.combine, t, v);
        }
        if (p.beta != 1.0f) t = __fmul_rn(p.beta, t);
        return t;
    };
    if (!RED) return term(0, 0, 0);
    float acc = identity_rt(p.reduce);
    for (int d0 = 0; d0 < p.er[0]; d0++)
        for (int d1 = 0; d1 < p.er[1]; d1++)
            for (int d2 = 0; d2 < p.er[2]; d2++) acc = op_rt(p.reduce, acc, term(d0, d1, d2));
    return acc;
}

// grid: x over the innermost dim (TX * 4 points per CTA trip), y over rows
template <int NOPS, bool GUARDS, bool RED>
__global__ void __launch_bounds__(256) nest_rows_kernel(const NestFastArgs p, int tx_log2) {
    const int TX = 1 << tx_log2, TY = 256 >> tx_log2;
    const int tx = threadIdx.x & (TX - 1), ty = threadIdx.x >> tx_log2;
    const int inner = p.eo[3];
    const int stride = gridDim.x * TX;
    for (int row = blockIdx.y * TY + ty; row < p.n_rows; row += gridDim.y * TY) {
        const int p2 = row % p.eo[2], r1 = row / p.eo[2];
        const int p1 = r1 % p.eo[1], p0 = r1 / p.eo[1];
        int ab[kNfOps], gb[kNfOps][kNfGuards];
#pragma unroll
        for (int o = 0; o < NOPS; o++) {
            ab[o] = p.op[o].addr.base + nf_dot3(p.op[o].addr.co, p0, p1, p2);
#pragma unroll
            for (int q = 0; q < kNfGuards; q++)
                gb[o][q] = GUARDS ? p.op[o].guard[q].base + nf_dot3(p.op[o].guard[q].co, p0, p1, p2) : 0;
        }
        const int ob = p.out_addr.base + nf_dot3(p.out_addr.co, p0, p1, p2);
        for (int i0 = blockIdx.x * TX + tx; i0 < inner; i0 += 4 * stride) {
            float x[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int i = i0 + u * stride;
                x[u] = i < inner ? nf_point<NOPS, GUARDS, RED>(p, ab, gb, i) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int i = i0 + u * stride;
                if (i < inner) {
                    float v = x[u];
                    if (p.epi.n) {
                        const int c[kNfOut] = {p0, p1, p2, i};
                        int64_t e[4];
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            int s = 0;
#pragma unroll
                            for (int d = 0; d < kNfOut; d++) s = (d == k + p.shift) ? c[d] : s;
                            e[k] = s;
                        }
                        v = apply_epilogue(p.epi, v, e[0], e[1], e[2], e[3]);
                    }
                    p.out[ob + p.out_addr.co[3] * i] = v;
                }
            }
        }
    }
}

// out[.., q, .., i] = in[..]: operand contiguous along output dim q, output
// along dim 3.  grid: x tiles of dim 3, y tiles of dim q, z the two batch dims.
__global__ void __launch_bounds__(256) nest_transpose_kernel(const NestFastArgs p) {
    __shared__ float tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int eq = p.eo[p.tq], inner = p.eo[3];
    const NfOperand &od = p.op[0];
    for (int z = blockIdx.z; z < p.eo[p.tb0] * p.eo[p.tb1]; z += gridDim.z) {
        const int c1 = z % p.eo[p.tb1], c0 = z / p.eo[p.tb1];
        const int ain = od.addr.base + od.addr.co[p.tb0] * c0 + od.addr.co[p.tb1] * c1;
        const int aout = p.out_addr.base + p.out_addr.co[p.tb0] * c0 + p.out_addr.co[p.tb1] * c1;
        const int q0 = blockIdx.y * 32, i0 = blockIdx.x * 32;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int i = i0 + ty + 8 * k, q = q0 + tx;
            if (i < inner && q < eq) tile[ty + 8 * k][tx] = __ldg(od.ptr + ain + od.addr.co[p.tq] * q + od.addr.co[3] * i);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int q = q0 + ty + 8 * k, i = i0 + tx;
            if (i < inner && q < eq) p.out[aout + p.out_addr.co[p.tq] * q + p.out_addr.co[3] * i] = tile[tx][ty + 8 * k];
        }
        __syncthreads();
    }
}

}  // namespace lsb
