// affine_nest.cuh -- general affine loop nest for one Arith node (coverage
// path).  One thread per output point (grid-stride); the reduction space is
// walked with an odometer so each step costs a few integer adds per operand.
//
// This is the B200 form of what the reference VM does for arbitrary
// (scalar-fallback) nests: guarded sload / sop / sfma over affine addresses
// (vm.py:172-213, backend.py:357-395) -- every access is
// base + Σ coeff[d] * iter[d], guarded coordinates read the view's oob fill
// (ir.py:238-245).  Ops are applied in the reference order: combine over the
// node's inputs left to right, beta per term, reduce (feedback.py:144-170).
#pragma once

#include "lsb_common.cuh"

namespace lsb {

struct NestArgs {
    int n_out, n_red, n_ops;
    int64_t extent[LSB_MAX_NEST_DIMS];
    lsb_nest_operand op[LSB_MAX_NEST_OPERANDS];
    float *out;
    lsb_affine out_addr;
    float beta;
    int64_t n_points;   // product of output extents
    EpiStages epi;
};

__device__ __forceinline__ bool guards_ok(const lsb_nest_operand &o, const int64_t *g) {
    for (int q = 0; q < o.n_guards; q++)
        if ((uint64_t)g[q] >= (uint64_t)o.guard_size[q]) return false;
    return true;
}

template <int OPC, int OPR>
__global__ void __launch_bounds__(256) affine_nest_kernel(const NestArgs p) {
    for (int64_t pt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pt < p.n_points;
         pt += (int64_t)gridDim.x * blockDim.x) {
        // output coordinates (row-major over the first n_out dims)
        int64_t coord[LSB_MAX_NEST_DIMS];
        int64_t rem = pt;
        for (int d = p.n_out - 1; d >= 0; d--) {
            coord[d] = rem % p.extent[d];
            rem /= p.extent[d];
        }
        // per-operand running address / guard values at reduction origin
        int64_t addr[LSB_MAX_NEST_OPERANDS];
        int64_t gv[LSB_MAX_NEST_OPERANDS][LSB_MAX_GUARDS];
        for (int o = 0; o < p.n_ops; o++) {
            int64_t a = p.op[o].addr.base;
            for (int d = 0; d < p.n_out; d++) a += p.op[o].addr.coeff[d] * coord[d];
            addr[o] = a;
            for (int q = 0; q < p.op[o].n_guards; q++) {
                int64_t v = p.op[o].guard[q].base;
                for (int d = 0; d < p.n_out; d++) v += p.op[o].guard[q].coeff[d] * coord[d];
                gv[o][q] = v;
            }
        }
        int64_t rcoord[LSB_MAX_NEST_DIMS];
        for (int d = 0; d < p.n_red; d++) rcoord[d] = 0;
        float acc = Op<OPR>::identity();
        bool first = true;
        int64_t red_total = 1;
        for (int d = 0; d < p.n_red; d++) red_total *= p.extent[p.n_out + d];
        for (int64_t r = 0; r < red_total; r++) {
            float t = 0.0f;
            for (int o = 0; o < p.n_ops; o++) {
                const lsb_nest_operand &od = p.op[o];
                float v = guards_ok(od, gv[o]) ? __ldg(od.ptr + addr[o]) : od.fill;
                t = (o == 0) ? v : Op<OPC>::apply(t, v);
            }
            if (p.beta != 1.0f) t = __fmul_rn(p.beta, t);
            if (p.n_red == 0) {
                acc = t;   // reduction-free node: the combined value itself
            } else {
                acc = first ? Op<OPR>::apply(Op<OPR>::identity(), t) : Op<OPR>::apply(acc, t);
            }
            first = false;
            // odometer step over the reduction dims (innermost last)
            for (int d = p.n_red - 1; d >= 0; d--) {
                const int D = p.n_out + d;
                if (++rcoord[d] < p.extent[D]) {
                    for (int o = 0; o < p.n_ops; o++) {
                        addr[o] += p.op[o].addr.coeff[D];
                        for (int q = 0; q < p.op[o].n_guards; q++) gv[o][q] += p.op[o].guard[q].coeff[D];
                    }
                    break;
                }
                const int64_t back = p.extent[D] - 1;
                rcoord[d] = 0;
                for (int o = 0; o < p.n_ops; o++) {
                    addr[o] -= p.op[o].addr.coeff[D] * back;
                    for (int q = 0; q < p.op[o].n_guards; q++) gv[o][q] -= p.op[o].guard[q].coeff[D] * back;
                }
            }
        }
        float x = acc;
        if (p.epi.n) {
            int64_t c[4] = {0, 0, 0, 0};
            for (int d = 0; d < p.n_out && d < 4; d++) c[d] = coord[d];
            x = apply_epilogue(p.epi, x, c[0], c[1], c[2], c[3]);
        }
        int64_t oa = p.out_addr.base;
        for (int d = 0; d < p.n_out; d++) oa += p.out_addr.coeff[d] * coord[d];
        p.out[oa] = x;
    }
}

}  // namespace lsb
