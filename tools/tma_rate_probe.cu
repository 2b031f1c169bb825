// Probe: time per raw-X box on every SM -- a 4-D TMA box {64 w, 7 h, 16 c, 1}
// (the planar conv's raw halo load) vs the same bytes as 112 1-D bulk copies
// of 256 B, vs 2-D boxes {64, 112 rows} -- with 1 or 2 boxes in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/tma_rate_probe tools/tma_rate_probe.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2205_00618_b200/csrc/tf32x3_gemm.cuh"
using namespace lsb::tc;

constexpr int W = 64, H = 56, C = 64, N = 8, RB = 7, SLOT = 16 * RB * W * 4;

__global__ void k(const __grid_constant__ CUtensorMap m4, const __grid_constant__ CUtensorMap m2, const float *x,
                  int mode, int iters, int inflight, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 4 * SLOT);
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 4; i++) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int n = blockIdx.x % N, cb = (blockIdx.x / N) % 4;
    long long c0 = clock64();
    uint32_t ph[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters + inflight; it++) {
        const int s = it % inflight;
        if (it >= inflight) {
            mbar_wait(&bar[s], ph[s]);
            ph[s] ^= 1;
        }
        if (it >= iters) continue;
        const int h0 = (it * 5) % 48;
        unsigned char *dst = sm + s * SLOT;
        mbar_expect_tx(&bar[s], SLOT);
        if (mode == 0) {
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
                "%5, %6}], [%2];" ::"r"(smem_u32(dst)),
                "l"(reinterpret_cast<uint64_t>(&m4)), "r"(smem_u32(&bar[s])), "r"(0), "r"(h0), "r"(cb * 16), "r"(n)
                : "memory");
        } else if (mode == 1) {
            for (int c = 0; c < 16; c++)
                for (int r = 0; r < RB; r++) {
                    const float *src = x + (((size_t)n * C + cb * 16 + c) * H + h0 + r) * W;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(dst + (c * RB + r) * W * 4)),
                        "l"(reinterpret_cast<uint64_t>(src)), "r"(W * 4), "r"(smem_u32(&bar[s]))
                        : "memory");
                }
        } else {
            // 16 2-D boxes {64 w, 7 rows} of the [N*C*H][W] view
            for (int c = 0; c < 16; c++) {
                const int row = ((n * C + cb * 16 + c) * H + h0);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
                    "[%2];" ::"r"(smem_u32(dst + c * RB * W * 4)),
                    "l"(reinterpret_cast<uint64_t>(&m2)), "r"(smem_u32(&bar[s])), "r"(0), "r"(row)
                    : "memory");
            }
        }
    }
    long long c1 = clock64();
    cyc[blockIdx.x] = c1 - c0;
}

int main() {
    const size_t n = (size_t)N * C * H * W;
    float *dx;
    long long *dc;
    cudaMalloc(&dx, n * 4);
    cudaMemset(dx, 0, n * 4);
    cudaMalloc(&dc, 148 * 8);
    CUtensorMap m4, m2;
    {
        cuuint64_t dims[4] = {W, H, C, N};
        cuuint64_t str[3] = {W * 4, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * C * 4};
        cuuint32_t box[4] = {W, RB, 16, 1}, es[4] = {1, 1, 1, 1};
        cuTensorMapEncodeTiled(&m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    {
        cuuint64_t dims[2] = {W, (cuuint64_t)N * C * H};
        cuuint64_t str[1] = {W * 4};
        cuuint32_t box[2] = {W, RB}, es[2] = {1, 1};
        cuTensorMapEncodeTiled(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dx, dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    const int smem = 4 * SLOT + 64 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char *names[3] = {"4-D box", "112 x 1-D bulk", "16 x 2-D box"};
    for (int grid : {1, 148})
        for (int inflight : {1, 2, 4})
            for (int mode = 0; mode < 3; mode++) {
                k<<<grid, 32, smem>>>(m4, m2, dx, mode, 64, inflight, dc);   // warm
                k<<<grid, 32, smem>>>(m4, m2, dx, mode, 64, inflight, dc);
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<long long> c(grid);
                cudaMemcpy(c.data(), dc, grid * 8, cudaMemcpyDeviceToHost);
                long long mx = 0, sum = 0;
                for (auto v : c) mx = v > mx ? v : mx, sum += v;
                printf("grid %3d inflight %d %-16s: %6.0f cycles per 28 KB box (max CTA %6.0f) %s\n", grid, inflight,
                       names[mode], (double)sum / grid / 64, (double)mx / 64, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
