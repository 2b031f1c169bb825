// Probe: 4-D TMA box {32 w, 4 c, 4 h, 1 n} of an NCHW tensor with
// SWIZZLE_128B_ATOM_32B lands as the MN-major SW128_BASE32B tf32 UMMA operand
// (4 atoms of [4 taps][32 px]); MMA against a K-major B and compare.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda.h>
#include "../paper_2205_00618_b200/csrc/tf32x3_conv.cuh"
using namespace lsb::tc;

__device__ __forceinline__ void tma_load_4d(const CUtensorMap *map, uint64_t *bar, void *dst, int x, int y, int z, int w) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w)
        : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap mx, const float *B, float *D, int w0, int h0) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    float *sb = reinterpret_cast<float *>(smem + 4096);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 8192);
    uint64_t *bar2 = bar + 1;
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem + 8208);
    int t = threadIdx.x;
    for (int e = t; e < 64 * 8; e += blockDim.x) {   // B: 64 x 8 taps, K-major SW64 rows of 16 taps (only 8 used)
        int n = e / 8, k = e % 8;
        uint32_t off = n * 64 + (((k >> 2) ^ ((n >> 1) & 3)) << 4) + (k & 3) * 4;
        sb[off / 4] = B[n * 8 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) { mbar_init(bar, 1); mbar_init(bar2, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tmem = *slot;
    if (t == 0) {
        mbar_expect_tx(bar, 4096);
        tma_load_4d(&mx, bar, smem, w0, 0, h0, 0);          // taps c = 0..3
        tma_load_4d(&mx, bar, smem + 2048, w0, 4, h0, 0);   // taps c = 4..7
        mbar_wait(bar, 0);
        uint32_t idesc = idesc_tf32(128, 64) | (1u << 15);
        uint64_t a = sdesc_mn_sw128_32b(smem_u32(smem));
        uint64_t b = sdesc_k_sw<64>(smem_u32(sb));
        umma_tf32(tmem, a, b, idesc, 0u);
        umma_commit(bar2);
    }
    __syncthreads();
    mbar_wait(bar2, 0);
    tc_fence_after();
    if (t < 128) {
        int q = t >> 5;
        float v[16];
        for (int part = 0; part < 4; part++) {
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + part * 16, v);
            for (int i = 0; i < 16; i++) D[t * 64 + part * 16 + i] = v[i];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main(int argc, char **argv) {
    const int C = 8, H = 6, W = 40;   // NCHW, N = 1
    static float hx[C * H * W], hB[64 * 8], hD[128 * 64];
    srand(3);
    for (auto &v : hx) v = (float)(rand() % 9 - 4);
    for (auto &v : hB) v = (float)(rand() % 5 - 2);
    float *x, *B, *D;
    cudaMalloc(&x, sizeof hx); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
    cudaMemcpy(x, hx, sizeof hx, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)C, (cuuint64_t)H, 1};
    cuuint64_t strides[3] = {(cuuint64_t)H * W * 4, (cuuint64_t)W * 4, (cuuint64_t)C * H * W * 4};
    cuuint32_t box[4] = {32, 4, 4, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, argc > 3 ? (CUtensorMapSwizzle)atoi(argv[3]) : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    if (r) return 1;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288);
    {
        int w0 = atoi(argv[1]), h0 = atoi(argv[2]);
        cudaMemset(D, 0, sizeof hD);
        probe<<<1, 128, 12288>>>(m, B, D, w0, h0);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
        double err = 0; int bad = 0;
        for (int mm = 0; mm < 128; mm++)
            for (int n = 0; n < 64; n++) {
                int h = h0 + mm / 32, w = w0 + mm % 32;
                double s = 0;
                for (int c = 0; c < 8; c++) {
                    float xv = (h >= 0 && h < H && w >= 0 && w < W) ? hx[(c * H + h) * W + w] : 0.f;
                    s += xv * hB[n * 8 + c];
                }
                double d = fabs(s - hD[mm * 64 + n]);
                err = d > err ? d : err; bad += d > 1e-3;
            }
        printf("w0=%d h0=%d %s maxerr=%g bad=%d\n", w0, h0, cudaGetErrorString(e), err, bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
