// kern_fast.cu -- tuned instantiations: (mul, add) FFMA2, (add, max|min)
// FADD2 + FMNMX3, for BM = 128 and 64, and the (mul, add) implicit-GEMM conv.
#include "lsb_dispatch.cuh"
#include "maxplus_fast.cuh"
#include "small_gemm.cuh"

namespace lsb {

GemmFn fast_gemm(int c, int r, int bm, bool two_level) {
    if (c == LSB_OP_MUL && r == LSB_OP_ADD) {
        if (two_level)
            return bm == 64 ? launch_gemm<1, 0, false, 64, true> : launch_gemm<1, 0, false, 128, true>;
        return bm == 64 ? launch_gemm<1, 0, false, 64> : launch_gemm<1, 0, false, 128>;
    }
    if (c == LSB_OP_ADD && r == LSB_OP_MAX)
        return bm == 64 ? launch_gemm<0, 2, false, 64> : launch_gemm<0, 2, false, 128>;
    if (c == LSB_OP_ADD && r == LSB_OP_MIN)
        return bm == 64 ? launch_gemm<0, 3, false, 64> : launch_gemm<0, 3, false, 128>;
    return nullptr;
}

// stream-K (add, max|min): identity fill of C, then the balanced kernel
void launch_streamk(int reduce, const GemmArgs &a, int ctas, cudaStream_t s) {
    const float id = reduce == LSB_OP_MAX ? -INFINITY : INFINITY;
    const int64_t total = a.M * a.N;
    const int fb = (int)std::min<int64_t>((total + 255) / 256, 2048);
    fill_kernel<0><<<fb, 256, 0, s>>>(a.C, a.M, a.N, a.sc_m, a.sc_n, id);
    if (reduce == LSB_OP_MAX)
        semiring_streamk_kernel<LSB_OP_ADD, LSB_OP_MAX, 128><<<ctas, kThreads, 0, s>>>(a);
    else
        semiring_streamk_kernel<LSB_OP_ADD, LSB_OP_MIN, 128><<<ctas, kThreads, 0, s>>>(a);
}

// the same with the cp.async row-major kernel (maxplus_fast.cuh)
void launch_streamk_fast(int reduce, const GemmArgs &a, int ctas, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(maxplus_streamk_fast_kernel<LSB_OP_MAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kMpSmemBytes);
        cudaFuncSetAttribute(maxplus_streamk_fast_kernel<LSB_OP_MIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kMpSmemBytes);
        attr = true;
    }
    const float id = reduce == LSB_OP_MAX ? -INFINITY : INFINITY;
    const int64_t total = a.M * a.N;
    const int fb = (int)std::min<int64_t>((total + 255) / 256, 2048);
    fill_kernel<0><<<fb, 256, 0, s>>>(a.C, a.M, a.N, a.sc_m, a.sc_n, id);
    if (reduce == LSB_OP_MAX)
        maxplus_streamk_fast_kernel<LSB_OP_MAX><<<ctas, kThreads, kMpSmemBytes, s>>>(a);
    else
        maxplus_streamk_fast_kernel<LSB_OP_MIN><<<ctas, kThreads, kMpSmemBytes, s>>>(a);
}

// split-K across a thread-block cluster of `splits` CTAs per output tile,
// DSMEM reduction (maxplus_cluster_kernel): one launch
int launch_maxplus_cluster(int reduce, const GemmArgs &a, int splits, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        for (auto fn : {maxplus_cluster_kernel<LSB_OP_MAX>, maxplus_cluster_kernel<LSB_OP_MIN>}) {
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMpClusterSmemBytes);
            cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
        attr = true;
    }
    const int64_t tiles = ((a.M + kMpBM - 1) / kMpBM) * ((a.N + kMpBN - 1) / kMpBN);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(tiles * splits));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kMpClusterSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)splits;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = reduce == LSB_OP_MAX ? cudaLaunchKernelEx(&cfg, maxplus_cluster_kernel<LSB_OP_MAX>, a)
                                         : cudaLaunchKernelEx(&cfg, maxplus_cluster_kernel<LSB_OP_MIN>, a);
    return e == cudaSuccess ? 0 : -1;
}

// latency-bound contractions: one launch, K split across the CTA's warps
// (small_gemm.cuh).  32 x 16 tiles while 32 x 32 ones would not cover the
// SMs.  Returns -1 for operator pairs without an instantiation.
template <int C, int R, int TN>
static int launch_small_tn(const GemmArgs &a, int64_t batch, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(small_gemm_kernel<C, R, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SgSmem<TN>::kBytes);
        attr = true;
    }
    const int64_t tiles = ((a.M + kSgTM - 1) / kSgTM) * ((a.N + TN - 1) / TN);
    small_gemm_kernel<C, R, TN><<<dim3((unsigned)tiles, (unsigned)batch), kSgThreads, SgSmem<TN>::kBytes, s>>>(a);
    return 0;
}

template <int C, int R>
static int launch_small_pair(const GemmArgs &a, int64_t batch, cudaStream_t s) {
    const int64_t t32 = ((a.M + kSgTM - 1) / kSgTM) * ((a.N + 31) / 32) * batch;
    return t32 < device_sms() ? launch_small_tn<C, R, 16>(a, batch, s) : launch_small_tn<C, R, 32>(a, batch, s);
}

int launch_small_gemm(int c, int r, const GemmArgs &a, int64_t batch, cudaStream_t s) {
    if (c == LSB_OP_MUL && r == LSB_OP_ADD) return launch_small_pair<LSB_OP_MUL, LSB_OP_ADD>(a, batch, s);
    if (c == LSB_OP_ADD && r == LSB_OP_MAX) return launch_small_pair<LSB_OP_ADD, LSB_OP_MAX>(a, batch, s);
    if (c == LSB_OP_ADD && r == LSB_OP_MIN) return launch_small_pair<LSB_OP_ADD, LSB_OP_MIN>(a, batch, s);
    return -1;
}

// stream-K with the in-kernel fixup (maxplus_fixup_kernel): cooperative
// launch so every CTA is resident; returns the CTA count used, or -1
int maxplus_fixup_ctas(int64_t units) {
    static int occ = -1;
    if (occ < 0) {
        for (auto fn : {maxplus_fixup_kernel<LSB_OP_MAX>, maxplus_fixup_kernel<LSB_OP_MIN>})
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMpSmemBytes);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, maxplus_fixup_kernel<LSB_OP_MAX>, kThreads,
                                                          kMpSmemBytes) != cudaSuccess)
            occ = 0;
    }
    return (int)std::min<int64_t>(units, (int64_t)occ * device_sms());
}

int launch_maxplus_fixup(int reduce, const GemmArgs &a, int ctas, float4 *part, int *flags, int epoch,
                         cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kMpSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = reduce == LSB_OP_MAX
                        ? cudaLaunchKernelEx(&cfg, maxplus_fixup_kernel<LSB_OP_MAX>, a, part, flags, epoch)
                        : cudaLaunchKernelEx(&cfg, maxplus_fixup_kernel<LSB_OP_MIN>, a, part, flags, epoch);
    return e == cudaSuccess ? 0 : -1;
}

// the one-CTA-per-SM variant (maxplus_duo_kernel): two groups per CTA share
// a segment's slices (bk deep) dynamically; returns the CTA count used, or -1
template <int BK>
static int duo_ctas(int64_t units) {
    static int occ = -1;
    if (occ < 0) {
        for (auto fn : {maxplus_duo_kernel<LSB_OP_MAX, BK>, maxplus_duo_kernel<LSB_OP_MIN, BK>})
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DuoCfg<BK>::kSmemBytes);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, maxplus_duo_kernel<LSB_OP_MAX, BK>, kDuoThreads,
                                                          DuoCfg<BK>::kSmemBytes) != cudaSuccess)
            occ = 0;
    }
    return (int)std::min<int64_t>(units, (int64_t)occ * device_sms());
}
int maxplus_duo_ctas(int64_t units, int bk) {
    return bk == 8 ? duo_ctas<8>(units) : bk == 32 ? duo_ctas<32>(units) : duo_ctas<16>(units);
}

template <int BK>
static int launch_duo(int reduce, const GemmArgs &a, int ctas, float4 *part, int *flags, int epoch, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(kDuoThreads);
    cfg.dynamicSmemBytes = DuoCfg<BK>::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = reduce == LSB_OP_MAX
                        ? cudaLaunchKernelEx(&cfg, maxplus_duo_kernel<LSB_OP_MAX, BK>, a, part, flags, epoch)
                        : cudaLaunchKernelEx(&cfg, maxplus_duo_kernel<LSB_OP_MIN, BK>, a, part, flags, epoch);
    return e == cudaSuccess ? 0 : -1;
}
int launch_maxplus_duo(int reduce, const GemmArgs &a, int bk, int ctas, float4 *part, int *flags, int epoch,
                       cudaStream_t s) {
    return bk == 8    ? launch_duo<8>(reduce, a, ctas, part, flags, epoch, s)
           : bk == 32 ? launch_duo<32>(reduce, a, ctas, part, flags, epoch, s)
                      : launch_duo<16>(reduce, a, ctas, part, flags, epoch, s);
}

void launch_conv_fold(const ConvArgs &a, int64_t n_img, cudaStream_t s) {
    const int64_t total = n_img * a.M * a.N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
    conv_splitk_fold_kernel<0><<<blocks, 256, 0, s>>>(a, n_img);
}

void launch_conv_fast(const ConvArgs &a, dim3 grid, size_t dyn, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(conv_igemm_kernel<1, 0, false, 64>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr = true;
    }
    conv_igemm_kernel<1, 0, false, 64><<<grid, kThreads, dyn, s>>>(a);
}

}  // namespace lsb
