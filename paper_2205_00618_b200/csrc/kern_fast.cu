// kern_fast.cu -- tuned instantiations: (mul, add) FFMA2, (add, max|min)
// FADD2 + FMNMX3, for BM = 128 and 64, and the (mul, add) implicit-GEMM conv.
#include "lsb_dispatch.cuh"

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
