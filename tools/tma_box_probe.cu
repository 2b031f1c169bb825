// Probe: 4-D TMA box loads of an NCHW tensor with boxes wider than the image
// (zero fill = conv padding).  Usage: tma_box_probe W wb rb
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/tma_box_probe tools/tma_box_probe.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2205_00618_b200/csrc/tf32x3_gemm.cuh"
using namespace lsb::tc;

__global__ void k(const __grid_constant__ CUtensorMap map, float *out, int n, int x0, int y0) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 63 * 1024);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(bar, n * 4);
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
            "[%2];" ::"r"(smem_u32(sm)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(bar)), "r"(x0), "r"(y0), "r"(0), "r"(0)
            : "memory");
    }
    __syncthreads();
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = reinterpret_cast<float *>(sm)[i];
}

int main(int argc, char **argv) {
    const int W = atoi(argv[1]), wb = atoi(argv[2]), rb = atoi(argv[3]), H = 16, C = 16;
    const int swz = argc > 4 ? atoi(argv[4]) : 0;   // 0 none, 1 32B, 2 64B, 3 128B
    const int x0 = argc > 5 ? atoi(argv[5]) : -1, y0 = argc > 6 ? atoi(argv[6]) : -1;
    std::vector<float> x((size_t)C * H * W);
    for (size_t i = 0; i < x.size(); i++) x[i] = (float)(i + 1);
    float *dx, *dout;
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&dout, 64 * 1024);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, 1};
    cuuint64_t strides[3] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * C * 4};
    cuuint32_t box[4] = {(cuuint32_t)wb, (cuuint32_t)rb, 16, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)swz,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("W=%d wb=%d rb=%d encode failed %d\n", W, wb, rb, (int)r);
        return 0;
    }
    const int n = wb * rb * 16;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    k<<<1, 128, 66 * 1024>>>(map, dout, n, x0, y0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("W=%d wb=%d rb=%d swz %d at (%d,%d): %s\n", W, wb, rb, swz, x0, y0, cudaGetErrorString(e));
        return 0;
    }
    std::vector<float> o(n);
    cudaMemcpy(o.data(), dout, n * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int c = 0; c < 16; c++)
        for (int rr = 0; rr < rb; rr++)
            for (int w = 0; w < wb; w++) {
                const int h = rr + y0, ww = w + x0;
                const float ref = (h >= 0 && h < H && ww >= 0 && ww < W) ? x[((size_t)c * H + h) * W + ww] : 0.f;
                bad += o[(c * rb + rr) * wb + w] != ref;
            }
    printf("W=%d wb=%d rb=%d swz %d at (%d,%d): ok, %d mismatches\n", W, wb, rb, swz, x0, y0, bad);
    return 0;
}
