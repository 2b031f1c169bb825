// kern_nest.cu -- general affine loop-nest kernels, one per operator pair.
#include <algorithm>

#include "lsb_dispatch.cuh"

namespace lsb {

template <int C, int R>
void launch_nest(const NestArgs &a, cudaStream_t s) {
    int64_t blocks = std::min<int64_t>((a.n_points + 255) / 256, (int64_t)device_sms() * 16);
    affine_nest_kernel<C, R><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(a);
}

#define NEST_ROW(C) {launch_nest<C, 0>, launch_nest<C, 1>, launch_nest<C, 2>, launch_nest<C, 3>}
const NestFn kNest[4][4] = {NEST_ROW(0), NEST_ROW(1), NEST_ROW(2), NEST_ROW(3)};
#undef NEST_ROW

}  // namespace lsb
