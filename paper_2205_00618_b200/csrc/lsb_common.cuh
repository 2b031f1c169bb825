// lsb_common.cuh -- operator functors and the fused epilogue shared by all
// B200 loop-nest kernels.
//
// Semantics follow the reference Arith node (ir.py:194-222) as evaluated by
// feedback.reference_eval (feedback.py:144-170) and the VM (vm.py:112-228):
//   combine / reduce ops add, mul, max, min   (program.py:182 KIND_CODE)
//   pre / post ops identity, relu, sigmoid    (program.py:183 EW_CODE)
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/lsb.h"

namespace lsb {

// max/min with NaN propagation, like the reference's np.max / np.maximum
// (feedback.py:29-42): fmaxf/fminf are IEEE maxNum and drop a NaN operand.
// Same cost: nested pairs still fuse into FMNMX3 (as FMNMX3.NAN).
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float fmin_nan(float a, float b) {
    float d;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

template <int OP>
struct Op;
template <>
struct Op<LSB_OP_ADD> {
    static __device__ __forceinline__ float apply(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float identity() { return 0.0f; }
};
template <>
struct Op<LSB_OP_MUL> {
    static __device__ __forceinline__ float apply(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float identity() { return 1.0f; }
};
template <>
struct Op<LSB_OP_MAX> {
    static __device__ __forceinline__ float apply(float a, float b) { return fmax_nan(a, b); }
    static __device__ __forceinline__ float identity() { return -INFINITY; }
};
template <>
struct Op<LSB_OP_MIN> {
    static __device__ __forceinline__ float apply(float a, float b) { return fmin_nan(a, b); }
    static __device__ __forceinline__ float identity() { return INFINITY; }
};

__device__ __forceinline__ float op_rt(int op, float a, float b) {
    switch (op) {
    case LSB_OP_ADD: return __fadd_rn(a, b);
    case LSB_OP_MUL: return __fmul_rn(a, b);
    case LSB_OP_MAX: return fmax_nan(a, b);
    default: return fmin_nan(a, b);
    }
}

__host__ __device__ __forceinline__ float identity_rt(int op) {
    switch (op) {
    case LSB_OP_ADD: return 0.0f;
    case LSB_OP_MUL: return 1.0f;
    case LSB_OP_MAX: return -INFINITY;
    default: return INFINITY;
    }
}

// vm.py:214-228: sigmoid evaluated in f64 then rounded, with the same
// two-branch formulation.  Out of line: inlining the f64 exp/div into every
// epilogue element blew the tf32x3 kernel up to 15k SASS instructions.
static __device__ __noinline__ float sigmoid_f64(float x) {
    double d = (double)x;
    if (d >= 0.0) return (float)(1.0 / (1.0 + exp(-d)));
    double e = exp(d);
    return (float)(e / (1.0 + e));
}

// vm.py:214-228: relu = max(x, 0)
__device__ __forceinline__ float ew_rt(int ew, float x) {
    if (ew == LSB_EW_RELU) return fmax_nan(x, 0.0f);
    if (ew == LSB_EW_SIGMOID) return sigmoid_f64(x);
    return x;
}

struct EpiStages {
    int n;
    lsb_epi_stage s[LSB_MAX_EPI];
};

// Fused epilogue (lsb.h lsb_epi_stage): x is the reduced value of one output
// point, c0..c3 its coordinates in the kernel's output index space.
__device__ __forceinline__ float apply_epilogue(const EpiStages &e, float x, int64_t c0,
                                                int64_t c1, int64_t c2, int64_t c3) {
    // fully unrolled over the static bound: e.s[i] must be a compile-time
    // offset, or the whole stage table (kernel-parameter space) is copied to
    // local memory for dynamic indexing (measured: 2.3x slower C4 epilogue)
#pragma unroll
    for (int i = 0; i < LSB_MAX_EPI; i++) {
        if (i >= e.n) break;
        const lsb_epi_stage &st = e.s[i];
        float t = x;
        if (st.combine >= 0) {
            float v = __ldg(st.operand + c0 * st.so[0] + c1 * st.so[1] + c2 * st.so[2] +
                            c3 * st.so[3]);
            t = op_rt(st.combine, t, v);
        }
        if (st.beta != 1.0f) t = __fmul_rn(st.beta, t);
        if (st.alpha != 0.0f) {
            float c = __ldg(st.c_in + c0 * st.sc[0] + c1 * st.sc[1] + c2 * st.sc[2] + c3 * st.sc[3]);
            c = __fmul_rn(st.alpha, ew_rt(st.pre, c));
            t = op_rt(st.reduce, c, t);
        }
        x = ew_rt(st.post, t);
    }
    return x;
}

// four consecutive points along coordinate 2 (a GEMM row segment n..n+3):
// per-stage row offsets are formed once and unit-stride operands (bias[n],
// C_in rows) are read as one 128-bit load
__device__ __forceinline__ float4 ldg4(const float *base, int64_t idx, int64_t stride) {
    const float *p = base + idx;
    if (stride == 1 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) return __ldg(reinterpret_cast<const float4 *>(p));
    if (stride == 0) {
        const float v = __ldg(p);
        return make_float4(v, v, v, v);
    }
    return make_float4(__ldg(p), __ldg(p + stride), __ldg(p + 2 * stride), __ldg(p + 3 * stride));
}

__device__ __forceinline__ void apply_epilogue4(const EpiStages &e, float (&x)[4], int64_t c0, int64_t c1,
                                                int64_t c2, int64_t c3) {
#pragma unroll
    for (int i = 0; i < LSB_MAX_EPI; i++) {
        if (i >= e.n) break;
        const lsb_epi_stage &st = e.s[i];
        float t[4] = {x[0], x[1], x[2], x[3]};
        if (st.combine >= 0) {
            const float4 v = ldg4(st.operand, c0 * st.so[0] + c1 * st.so[1] + c2 * st.so[2] + c3 * st.so[3], st.so[2]);
            t[0] = op_rt(st.combine, t[0], v.x);
            t[1] = op_rt(st.combine, t[1], v.y);
            t[2] = op_rt(st.combine, t[2], v.z);
            t[3] = op_rt(st.combine, t[3], v.w);
        }
        if (st.beta != 1.0f) {
#pragma unroll
            for (int q = 0; q < 4; q++) t[q] = __fmul_rn(st.beta, t[q]);
        }
        if (st.alpha != 0.0f) {
            const float4 c = ldg4(st.c_in, c0 * st.sc[0] + c1 * st.sc[1] + c2 * st.sc[2] + c3 * st.sc[3], st.sc[2]);
            const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int q = 0; q < 4; q++) t[q] = op_rt(st.reduce, __fmul_rn(st.alpha, ew_rt(st.pre, cv[q])), t[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; q++) x[q] = ew_rt(st.post, t[q]);
    }
}

// GEMM-row variant of apply_epilogue4 (coordinates (0, m, n..n+3, 0)) whose
// row-invariant operands (so[1] == 0: bias[n], column vectors) were loaded
// once per column segment into pre[] by epi4_preload -- a per-row dependent
// L2 round trip made the C4 epilogue 4x slower than its stores
__device__ __forceinline__ void epi4_preload(const EpiStages &e, int64_t n, bool full4, float4 (&pre)[LSB_MAX_EPI]) {
#pragma unroll
    for (int i = 0; i < LSB_MAX_EPI; i++) {
        pre[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i >= e.n) break;
        const lsb_epi_stage &st = e.s[i];
        if (st.combine >= 0 && st.so[1] == 0) {
            if (full4) {
                pre[i] = ldg4(st.operand, n * st.so[2], st.so[2]);
            } else {
                pre[i].x = __ldg(st.operand + n * st.so[2]);   // n < N always holds for the first
            }
        }
    }
}

__device__ __forceinline__ void apply_epilogue4_pre(const EpiStages &e, float (&x)[4], int64_t m, int64_t n,
                                                    const float4 (&pre)[LSB_MAX_EPI]) {
#pragma unroll
    for (int i = 0; i < LSB_MAX_EPI; i++) {
        if (i >= e.n) break;
        const lsb_epi_stage &st = e.s[i];
        float t[4] = {x[0], x[1], x[2], x[3]};
        if (st.combine >= 0) {
            const float4 v = st.so[1] == 0 ? pre[i] : ldg4(st.operand, m * st.so[1] + n * st.so[2], st.so[2]);
            t[0] = op_rt(st.combine, t[0], v.x);
            t[1] = op_rt(st.combine, t[1], v.y);
            t[2] = op_rt(st.combine, t[2], v.z);
            t[3] = op_rt(st.combine, t[3], v.w);
        }
        if (st.beta != 1.0f) {
#pragma unroll
            for (int q = 0; q < 4; q++) t[q] = __fmul_rn(st.beta, t[q]);
        }
        if (st.alpha != 0.0f) {
            const float4 c = ldg4(st.c_in, m * st.sc[1] + n * st.sc[2], st.sc[2]);
            const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int q = 0; q < 4; q++) t[q] = op_rt(st.reduce, __fmul_rn(st.alpha, ew_rt(st.pre, cv[q])), t[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; q++) x[q] = ew_rt(st.post, t[q]);
    }
}

}  // namespace lsb
