// Probe: cycles per job of the planar conv's halo converter loop (raw smem
// slot [16 c][rb][wb] -> hi / lo planes [8][384 rows][4]), 4 converter warps,
// variants: 0 = the kernel's loop (per-row division), 1 = no division
// (row offsets stepped), 2 = 1 + all rows' loads issued before any store.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/conv_cvt_probe tools/conv_cvt_probe.cu
#include <cstdio>

#include "../paper_2205_00618_b200/csrc/tf32x3_gemm.cuh"
using namespace lsb::tc;

constexpr int HALO = 384, PLANE = HALO * 16, RAW = 28 * 1024;

__device__ __forceinline__ float lo_of(float x, bool &bad) {
    const bool fin = fabsf(x) < __int_as_float(0x7f800000);
    bad |= !fin;
    return fin ? x - __uint_as_float(__float_as_uint(x) & 0xffffe000u) : 0.0f;
}

template <int V>
__global__ void __launch_bounds__(128) k(int halo, int Wp, int wb, int rb, int wsh, int F0, int jobs, long long *cyc,
                                          int *sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const float *raw = reinterpret_cast<const float *>(sm + 8 * PLANE);
    float *hb = reinterpret_cast<float *>(sm);
    const int t = threadIdx.x, cstride = rb * wb;
    for (int i = t; i < RAW / 4; i += 128) reinterpret_cast<float *>(sm + 8 * PLANE)[i] = (float)i * 1.0001f;
    __syncthreads();
    long long c0 = clock64();
    bool bad = false;
    for (int job = 0; job < jobs; job++) {
        if (V == 0) {
            for (int row = t; row < halo; row += 128) {
                const int F = F0 + row;
                const int hp = F / Wp, wp = F - hp * Wp;
                const float *src = raw + (hp - F0 / Wp) * wb + wp + wsh;
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    float4 hv = make_float4(src[(4 * g) * cstride], src[(4 * g + 1) * cstride],
                                            src[(4 * g + 2) * cstride], src[(4 * g + 3) * cstride]);
                    float4 lv = make_float4(lo_of(hv.x, bad), lo_of(hv.y, bad), lo_of(hv.z, bad), lo_of(hv.w, bad));
                    *reinterpret_cast<float4 *>(hb + g * (PLANE / 4) + row * 4) = hv;
                    *reinterpret_cast<float4 *>(hb + (4 + g) * (PLANE / 4) + row * 4) = lv;
                }
            }
        } else {
            constexpr int kR = 3;   // rows per thread (halo <= 384)
            int off[kR];
            {
                const int hp0 = F0 / Wp;
                int F = F0 + t, hp = F / Wp, wp = F - hp * Wp;
                const int dh = 128 / Wp, dw = 128 - dh * Wp;
#pragma unroll
                for (int r = 0; r < kR; r++) {
                    off[r] = (hp - hp0) * wb + wp + wsh;
                    wp += dw;
                    hp += dh;
                    if (wp >= Wp) {
                        wp -= Wp;
                        hp++;
                    }
                }
            }
            if (V == 1) {
#pragma unroll
                for (int r = 0; r < kR; r++) {
                    const int row = t + 128 * r;
                    if (row < halo) {
#pragma unroll
                        for (int g = 0; g < 4; g++) {
                            const float *src = raw + off[r] + 4 * g * cstride;
                            float4 hv = make_float4(src[0], src[cstride], src[2 * cstride], src[3 * cstride]);
                            float4 lv = make_float4(lo_of(hv.x, bad), lo_of(hv.y, bad), lo_of(hv.z, bad), lo_of(hv.w, bad));
                            *reinterpret_cast<float4 *>(hb + g * (PLANE / 4) + row * 4) = hv;
                            *reinterpret_cast<float4 *>(hb + (4 + g) * (PLANE / 4) + row * 4) = lv;
                        }
                    }
                }
            } else {
                float v[kR][16];
#pragma unroll
                for (int r = 0; r < kR; r++)
#pragma unroll
                    for (int c = 0; c < 16; c++) v[r][c] = (t + 128 * r < halo) ? raw[off[r] + c * cstride] : 0.f;
#pragma unroll
                for (int r = 0; r < kR; r++) {
                    const int row = t + 128 * r;
                    if (row < halo) {
#pragma unroll
                        for (int g = 0; g < 4; g++) {
                            float4 hv = make_float4(v[r][4 * g], v[r][4 * g + 1], v[r][4 * g + 2], v[r][4 * g + 3]);
                            float4 lv = make_float4(lo_of(hv.x, bad), lo_of(hv.y, bad), lo_of(hv.z, bad), lo_of(hv.w, bad));
                            *reinterpret_cast<float4 *>(hb + g * (PLANE / 4) + row * 4) = hv;
                            *reinterpret_cast<float4 *>(hb + (4 + g) * (PLANE / 4) + row * 4) = lv;
                        }
                    }
                }
            }
        }
        __syncwarp();
        F0 += 7;   // vary the wrap points
        F0 %= 64;
    }
    long long c1 = clock64();
    if (t == 0) cyc[blockIdx.x] = (c1 - c0) / jobs;
    if (bad) sink[0] = 1;
}

int main() {
    long long *dc, h;
    int *ds;
    cudaMalloc(&dc, 8 * 148);
    cudaMalloc(&ds, 4);
    const int smem = 8 * PLANE + RAW;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int v = 0; v < 3; v++) {
        auto fn = v == 0 ? k<0> : v == 1 ? k<1> : k<2>;
        fn<<<1, 128, smem>>>(310, 58, 64, 7, 3, 0, 200, dc, ds);
        fn<<<1, 128, smem>>>(310, 58, 64, 7, 3, 0, 200, dc, ds);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
        printf("variant %d: %lld cycles per job (310 rows x 16 channels) %s\n", v, h, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
