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
//    divisions), a thread then walks its row in steps of the grid width, eight
//    points per trip (four under a reduction) with their loads independent.
//    The reduction space is three nested 32-bit loops, outside the points.  Templated on the
//    operand count, on whether any guard exists and on whether there is a
//    reduction, so reduction-free unguarded nests (broadcast_add) compile to
//    load / op / store.
//  * nest_vec4_kernel: reduction-free nests with 16-byte aligned contiguous
//    rows (elementwise / broadcast / concat): float4 loads and stores; a
//    group of four points that straddles a guard boundary loads by element.
//  * nest_pool_kernel: non-overlapping pooling along the innermost dim (window
//    == stride, contiguous): the window's inputs of four outputs are one
//    contiguous run, read as float4s.
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

// U consecutive trips of one thread's row walk (points i0 + u * stride): the
// reduction loops are outermost and the U points innermost, so every
// reduction step issues U independent loads per operand; per point the terms
// still arrive in the reference order.
template <int NOPS, bool GUARDS, bool RED, int U>
__device__ __forceinline__ void nf_strip(const NestFastArgs &p, const int (&ab)[kNfOps],
                                         const int (&gb)[kNfOps][kNfGuards], int i0, int stride, int inner,
                                         float (&x)[U]) {
    const float id = RED ? identity_rt(p.reduce) : 0.0f;
#pragma unroll
    for (int u = 0; u < U; u++) x[u] = id;
    auto step = [&](int d0, int d1, int d2) {
        int ra[NOPS], rg[NOPS][kNfGuards];   // this step's offsets (uniform)
#pragma unroll
        for (int o = 0; o < NOPS; o++) {
            const NfOperand &od = p.op[o];
            ra[o] = ab[o] + (RED ? od.addr.cr[0] * d0 + od.addr.cr[1] * d1 + od.addr.cr[2] * d2 : 0);
#pragma unroll
            for (int q = 0; q < kNfGuards; q++)
                rg[o][q] = GUARDS ? gb[o][q] + (RED ? od.guard[q].cr[0] * d0 + od.guard[q].cr[1] * d1 +
                                                          od.guard[q].cr[2] * d2
                                                    : 0)
                                  : 0;
        }
        float v[NOPS][U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = i0 + u * stride;
#pragma unroll
            for (int o = 0; o < NOPS; o++) {
                const NfOperand &od = p.op[o];
                bool ok = i < inner;
                if (GUARDS) {
#pragma unroll
                    for (int q = 0; q < kNfGuards; q++)
                        if (q < od.n_guards) ok = ok && (unsigned)(rg[o][q] + od.guard[q].co[3] * i) < od.guard_size[q];
                }
                v[o][u] = ok ? __ldg(od.ptr + ra[o] + od.addr.co[3] * i) : od.fill;
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            float t = v[0][u];
            if (NOPS == 2) t = op_rt(p.combine, t, v[NOPS - 1][u]);
            if (p.beta != 1.0f) t = __fmul_rn(p.beta, t);
            x[u] = RED ? op_rt(p.reduce, x[u], t) : t;
        }
    };
    if (!RED) {
        step(0, 0, 0);
    } else {
        for (int d0 = 0; d0 < p.er[0]; d0++)
            for (int d1 = 0; d1 < p.er[1]; d1++)
                for (int d2 = 0; d2 < p.er[2]; d2++) step(d0, d1, d2);
    }
}

// grid: x over the innermost dim (TX * U points per CTA trip), y over rows
template <int NOPS, bool GUARDS, bool RED>
__global__ void __launch_bounds__(256, 6) nest_rows_kernel(const NestFastArgs p, int tx_log2) {
    constexpr int U = RED ? 4 : 8;
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
        for (int i0 = blockIdx.x * TX + tx; i0 < inner; i0 += U * stride) {
            float x[U];
            nf_strip<NOPS, GUARDS, RED, U>(p, ab, gb, i0, stride, inner, x);
#pragma unroll
            for (int u = 0; u < U; u++) {
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

// Reduction-free nests whose operands are contiguous (or constant) along the
// innermost output dim, 16-byte aligned rows, guarded or not: four float4 groups per
// thread per trip (64 B per operand in flight per thread).  i counts float4s.
template <int NOPS, bool GUARDS>
__device__ __forceinline__ void nest_vec4_body(const NestFastArgs &p, int tx_log2) {
    const int TX = 1 << tx_log2, TY = 256 >> tx_log2;
    const int tx = threadIdx.x & (TX - 1), ty = threadIdx.x >> tx_log2;
    const int inner4 = p.eo[3] >> 2;
    const int stride = gridDim.x * TX;
    for (int row = blockIdx.y * TY + ty; row < p.n_rows; row += gridDim.y * TY) {
        const int p2 = row % p.eo[2], r1 = row / p.eo[2];
        const int p1 = r1 % p.eo[1], p0 = r1 / p.eo[1];
        const float *src[NOPS];
        int gb[NOPS][kNfGuards];
#pragma unroll
        for (int o = 0; o < NOPS; o++) {
            src[o] = p.op[o].ptr + p.op[o].addr.base + nf_dot3(p.op[o].addr.co, p0, p1, p2);
#pragma unroll
            for (int q = 0; q < kNfGuards; q++)
                gb[o][q] = GUARDS ? p.op[o].guard[q].base + nf_dot3(p.op[o].guard[q].co, p0, p1, p2) : 0;
        }
        float *dst = p.out + p.out_addr.base + nf_dot3(p.out_addr.co, p0, p1, p2);
        for (int i0 = blockIdx.x * TX + tx; i0 < inner4; i0 += 4 * stride) {
            float4 v[NOPS][4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int i = i0 + u * stride;
                if (i < inner4) {
#pragma unroll
                    for (int o = 0; o < NOPS; o++) {
                        const NfOperand &od = p.op[o];
                        bool ok[4] = {true, true, true, true};
                        bool all = true, any = true;
                        if (GUARDS) {
                            // a group of four points is all inside its guards (vector load), all
                            // outside (the fill) or straddles a boundary (element by element).
                            // A guard is an interval of an affine form, so the ends decide "all";
                            // the middle points are only evaluated when the ends disagree or are
                            // both outside (a window narrower than the group).
                            bool first = true, last = true;
#pragma unroll
                            for (int q = 0; q < kNfGuards; q++)
                                if (q < od.n_guards) {
                                    const int g0 = gb[o][q] + od.guard[q].co[3] * (4 * i);
                                    first = first && (unsigned)g0 < od.guard_size[q];
                                    last = last && (unsigned)(g0 + 3 * od.guard[q].co[3]) < od.guard_size[q];
                                }
                            all = first && last;
                            if (!all) {
                                ok[0] = first;
                                ok[3] = last;
#pragma unroll
                                for (int e = 1; e < 3; e++)
#pragma unroll
                                    for (int q = 0; q < kNfGuards; q++)
                                        if (q < od.n_guards)
                                            ok[e] = ok[e] && (unsigned)(gb[o][q] + od.guard[q].co[3] * (4 * i + e)) < od.guard_size[q];
                                any = ok[0] || ok[1] || ok[2] || ok[3];
                            }
                        }
                        if (!any) {
                            v[o][u] = make_float4(od.fill, od.fill, od.fill, od.fill);
                        } else if (od.addr.co[3]) {
                            if (all) {
                                v[o][u] = __ldg(reinterpret_cast<const float4 *>(src[o]) + i);
                            } else {
                                v[o][u].x = ok[0] ? __ldg(src[o] + 4 * i) : od.fill;
                                v[o][u].y = ok[1] ? __ldg(src[o] + 4 * i + 1) : od.fill;
                                v[o][u].z = ok[2] ? __ldg(src[o] + 4 * i + 2) : od.fill;
                                v[o][u].w = ok[3] ? __ldg(src[o] + 4 * i + 3) : od.fill;
                            }
                        } else {
                            const float b = __ldg(src[o]);
                            v[o][u] = make_float4(ok[0] ? b : od.fill, ok[1] ? b : od.fill, ok[2] ? b : od.fill,
                                                  ok[3] ? b : od.fill);
                        }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int i = i0 + u * stride;
                if (i < inner4) {
                    float4 t = v[0][u];
                    if (NOPS == 2) {
                        t.x = op_rt(p.combine, t.x, v[NOPS - 1][u].x);
                        t.y = op_rt(p.combine, t.y, v[NOPS - 1][u].y);
                        t.z = op_rt(p.combine, t.z, v[NOPS - 1][u].z);
                        t.w = op_rt(p.combine, t.w, v[NOPS - 1][u].w);
                    }
                    if (p.beta != 1.0f) {
                        t.x = __fmul_rn(p.beta, t.x);
                        t.y = __fmul_rn(p.beta, t.y);
                        t.z = __fmul_rn(p.beta, t.z);
                        t.w = __fmul_rn(p.beta, t.w);
                    }
                    reinterpret_cast<float4 *>(dst)[i] = t;
                }
            }
        }
    }
}

// Two entry points: the unguarded body fits 48 registers (5 CTAs per SM:
// broadcast_add 5432 -> 5580 GB/s); the guarded one is fastest at the
// compiler's own 58 (capped to 48 or pushed to 64+ it lost 8-19 % on concat).
template <int NOPS>
__global__ void __launch_bounds__(256, 5) nest_vec4_kernel(const NestFastArgs p, int tx_log2) {
    nest_vec4_body<NOPS, false>(p, tx_log2);
}
template <int NOPS>
__global__ void __launch_bounds__(256) nest_vec4_guarded_kernel(const NestFastArgs p, int tx_log2) {
    nest_vec4_body<NOPS, true>(p, tx_log2);
}

// Non-overlapping pooling along the innermost dim: one operand, no guards, the
// innermost reduction dim contiguous with extent E equal to the operand's
// stride along the innermost output dim (window == stride), 16-byte aligned
// rows.  A thread owns groups of four consecutive outputs: per outer reduction
// step their 4 E inputs are one contiguous run, read as E float4s, and the
// window's terms fold in the reference order (outer reduction dims, then the
// window).  Four groups per trip.
template <int E>
__global__ void __launch_bounds__(256) nest_pool_kernel(const NestFastArgs p, int tx_log2) {
    const int TX = 1 << tx_log2, TY = 256 >> tx_log2;
    const int tx = threadIdx.x & (TX - 1), ty = threadIdx.x >> tx_log2;
    const int inner4 = p.eo[3] >> 2;
    const int stride = gridDim.x * TX;
    const NfOperand &od = p.op[0];
    const float id = identity_rt(p.reduce);
    for (int row = blockIdx.y * TY + ty; row < p.n_rows; row += gridDim.y * TY) {
        const int p2 = row % p.eo[2], r1 = row / p.eo[2];
        const int p1 = r1 % p.eo[1], p0 = r1 / p.eo[1];
        const float *src = od.ptr + od.addr.base + nf_dot3(od.addr.co, p0, p1, p2);
        float *dst = p.out + p.out_addr.base + nf_dot3(p.out_addr.co, p0, p1, p2);
        for (int i0 = blockIdx.x * TX + tx; i0 < inner4; i0 += 4 * stride) {
            float acc[4][4];
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[u][j] = id;
            for (int d0 = 0; d0 < p.er[0]; d0++)
                for (int d1 = 0; d1 < p.er[1]; d1++) {
                    const float4 *line = reinterpret_cast<const float4 *>(src + od.addr.cr[0] * d0 + od.addr.cr[1] * d1);
                    float4 w[4][E];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int i = i0 + u * stride;
                        if (i < inner4) {
#pragma unroll
                            for (int e = 0; e < E; e++) w[u][e] = __ldg(line + i * E + e);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        if (i0 + u * stride < inner4) {
#pragma unroll
                            for (int j = 0; j < 4; j++)
#pragma unroll
                                for (int d2 = 0; d2 < E; d2++) {
                                    const int f = j * E + d2;   // float f of the run: float4 f / 4, lane f % 4
                                    const float4 q = w[u][f >> 2];
                                    float t = (f & 3) == 0 ? q.x : (f & 3) == 1 ? q.y : (f & 3) == 2 ? q.z : q.w;
                                    if (p.beta != 1.0f) t = __fmul_rn(p.beta, t);
                                    acc[u][j] = op_rt(p.reduce, acc[u][j], t);
                                }
                        }
                    }
                }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int i = i0 + u * stride;
                if (i < inner4) reinterpret_cast<float4 *>(dst)[i] = make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
            }
        }
    }
}

// out[.., q, .., i] = in[..]: operand contiguous along output dim q, output
// along dim 3.  grid: x tiles of dim 3, y tiles of dim q, z the two batch dims.
constexpr int kNfTileQ = 32, kNfTileI = 64;   // tile: 32 along the operand's line, 64 along the output's
__global__ void __launch_bounds__(256) nest_transpose_kernel(const NestFastArgs p) {
    __shared__ float tile[kNfTileI][kNfTileQ + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    const int eq = p.eo[p.tq], inner = p.eo[3];
    const NfOperand &od = p.op[0];
    for (int z = blockIdx.z; z < p.eo[p.tb0] * p.eo[p.tb1]; z += gridDim.z) {
        const int c1 = z % p.eo[p.tb1], c0 = z / p.eo[p.tb1];
        const int ain = od.addr.base + od.addr.co[p.tb0] * c0 + od.addr.co[p.tb1] * c1;
        const int aout = p.out_addr.base + p.out_addr.co[p.tb0] * c0 + p.out_addr.co[p.tb1] * c1;
        const int q0 = blockIdx.y * kNfTileQ, i0 = blockIdx.x * kNfTileI;
        const int cq = od.addr.co[p.tq], ci = od.addr.co[3], oq = p.out_addr.co[p.tq];
        // read: lanes along q (the operand's contiguous dim), 8 rows of i per pass
#pragma unroll
        for (int k = 0; k < kNfTileI / 8; k++) {
            const int il = ty + 8 * k, i = i0 + il, q = q0 + tx;
            if (i < inner && q < eq) tile[il][tx] = __ldg(od.ptr + ain + cq * q + ci * i);
        }
        __syncthreads();
        // write: lanes along i (the output's contiguous dim), 4 rows of q per pass
#pragma unroll
        for (int k = 0; k < kNfTileQ / 4; k++) {
            const int il = threadIdx.x & (kNfTileI - 1), ql = (threadIdx.x >> 6) + 4 * k;
            const int i = i0 + il, q = q0 + ql;
            if (i < inner && q < eq) p.out[aout + oq * q + i] = tile[il][ql];
        }
        __syncthreads();
    }
}

// The same permutation with 16-byte aligned rows on both sides: 64 x 64 tiles,
// float4 loads along q and float4 stores along i (four float4 in flight per
// thread each way); the 4 x 4 transposition happens in the shared-memory tile.
__global__ void __launch_bounds__(256) nest_transpose4_kernel(const NestFastArgs p) {
    constexpr int T = 64;
    __shared__ float tile[T][T + 1];
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;   // 16 float4 columns x 16 rows
    const int eq = p.eo[p.tq], inner = p.eo[3];
    const NfOperand &od = p.op[0];
    for (int z = blockIdx.z; z < p.eo[p.tb0] * p.eo[p.tb1]; z += gridDim.z) {
        const int c1 = z % p.eo[p.tb1], c0 = z / p.eo[p.tb1];
        const int ain = od.addr.base + od.addr.co[p.tb0] * c0 + od.addr.co[p.tb1] * c1;
        const int aout = p.out_addr.base + p.out_addr.co[p.tb0] * c0 + p.out_addr.co[p.tb1] * c1;
        const int q0 = blockIdx.y * T, i0 = blockIdx.x * T;
        const int ci = od.addr.co[3], oq = p.out_addr.co[p.tq];
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int i = i0 + ly + 16 * k, q = q0 + 4 * lx;
            if (i < inner && q < eq) v[k] = __ldg(reinterpret_cast<const float4 *>(od.ptr + ain + q + ci * i));
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int il = ly + 16 * k;
            tile[il][4 * lx] = v[k].x;
            tile[il][4 * lx + 1] = v[k].y;
            tile[il][4 * lx + 2] = v[k].z;
            tile[il][4 * lx + 3] = v[k].w;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int ql = ly + 16 * k, q = q0 + ql, i = i0 + 4 * lx;
            if (i < inner && q < eq)
                *reinterpret_cast<float4 *>(p.out + aout + oq * q + i) =
                    make_float4(tile[4 * lx][ql], tile[4 * lx + 1][ql], tile[4 * lx + 2][ql], tile[4 * lx + 3][ql]);
        }
        __syncthreads();
    }
}

}  // namespace lsb
