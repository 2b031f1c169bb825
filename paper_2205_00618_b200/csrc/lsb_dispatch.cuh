// lsb_dispatch.cuh -- launcher tables shared by the API TU (lsb_api.cu) and
// the kernel-instantiation TUs (kern_*.cu, compiled in parallel).
#pragma once

#include "affine_nest.cuh"
#include "semiring_gemm.cuh"

namespace lsb {

using GemmFn = void (*)(const GemmArgs &, dim3, cudaStream_t);
using ConvFn = void (*)(const ConvArgs &, dim3, size_t, cudaStream_t);
using SplitFn = void (*)(const GemmArgs &, int64_t, cudaStream_t);
using NestFn = void (*)(const NestArgs &, cudaStream_t);

int device_sms();                               // lsb_api.cu

GemmFn fast_gemm(int combine, int reduce, int bm, bool two_level);   // kern_fast.cu (nullptr if untuned)
void launch_conv_fast(const ConvArgs &a, dim3 grid, size_t dyn, cudaStream_t s);
extern const GemmFn kGemmGeneric[4][4];          // kern_generic.cu
extern const SplitFn kSplit[4];                  // kern_generic.cu
extern const NestFn kNest[4][4];                 // kern_nest.cu

template <int C, int R, bool B, int BM, bool TWO = false>
void launch_gemm(const GemmArgs &a, dim3 grid, cudaStream_t s) {
    constexpr size_t dyn = gemm_dyn_smem<BM>();
    static bool attr = false;   // > 48 KiB dynamic smem needs an opt-in, once per kernel
    if (!attr) {
        cudaFuncSetAttribute(semiring_gemm_kernel<C, R, B, BM, TWO>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        attr = true;
    }
    semiring_gemm_kernel<C, R, B, BM, TWO><<<grid, kThreads, dyn, s>>>(a);
}

}  // namespace lsb
