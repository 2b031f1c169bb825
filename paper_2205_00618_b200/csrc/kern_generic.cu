// kern_generic.cu -- every (combine, reduce) pair with beta applied per term
// (exact reference order, ir.py:194-222), and the split-K fold kernels.
#include <algorithm>

#include "lsb_dispatch.cuh"

namespace lsb {

template <int R>
void launch_split(const GemmArgs &a, int64_t batch, cudaStream_t s) {
    int64_t total = batch * a.M * a.N;
    int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)device_sms() * 8);
    splitk_epilogue_kernel<R><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(a, batch);
}

#define GEN_ROW(C) {launch_gemm<C, 0, true, 128>, launch_gemm<C, 1, true, 128>, \
                    launch_gemm<C, 2, true, 128>, launch_gemm<C, 3, true, 128>}
const GemmFn kGemmGeneric[4][4] = {GEN_ROW(0), GEN_ROW(1), GEN_ROW(2), GEN_ROW(3)};
#undef GEN_ROW

const SplitFn kSplit[4] = {launch_split<0>, launch_split<1>, launch_split<2>, launch_split<3>};

}  // namespace lsb
