// Microbenchmark of sm_100a issue / pipe rates for the max-plus instruction
// mix, with exact SASS via inline PTX (add.rn.f32x2, 3-input max.f32).
#include <cstdio>
#include <cuda_runtime.h>

#define FADD2(d, a, b) asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b))
#define MAX3(d, a, b, c) asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c))
#define MAX2(d, a, b) asm volatile("max.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b))
#define FFMA2(d, a, b, c) asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c))

template <int MODE>
__global__ void __launch_bounds__(256, 2) k(float *out, int iters) {
    unsigned long long s[16], x[16];
    float m[16];
    for (int i = 0; i < 16; i++) {
        float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        s[i] = *reinterpret_cast<unsigned long long *>(&v);
        x[i] = s[i] ^ 0x100;
        m[i] = -1e30f;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            if (MODE == 0) {        // FADD2 + FMNMX3 (one of each per 2 points)
                unsigned long long t;
                FADD2(t, s[i], x[i]);
                float2 tv = *reinterpret_cast<float2 *>(&t);
                MAX3(m[i], m[i], tv.x, tv.y);
            } else if (MODE == 1) { // FADD2 only
                FADD2(s[i], s[i], x[i]);
            } else if (MODE == 2) { // FMNMX3 only
                float2 xv = *reinterpret_cast<float2 *>(&x[i]);
                MAX3(m[i], m[i], xv.x, xv.y);
            } else if (MODE == 3) { // FMNMX (2-input) only
                float2 xv = *reinterpret_cast<float2 *>(&x[i]);
                MAX2(m[i], m[i], xv.x);
            } else if (MODE == 4) { // FFMA2 only
                FFMA2(s[i], s[i], x[i], s[i]);
            } else if (MODE == 5) { // FADD2 + 2 x FMNMX (one FADD2 per 2 points)
                unsigned long long t;
                FADD2(t, s[i], x[i]);
                float2 tv = *reinterpret_cast<float2 *>(&t);
                MAX2(m[i], m[i], tv.x);
                MAX2(m[(i + 8) & 15], m[(i + 8) & 15], tv.y);
            } else {                // scalar FADD + FMNMX per point
                float2 xv = *reinterpret_cast<float2 *>(&x[i]);
                float t;
                asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(t) : "f"(xv.x), "f"(m[(i + 3) & 15]));
                MAX2(m[i], m[i], t);
            }
        }
    }
    float r = 0;
    for (int i = 0; i < 16; i++) {
        float2 v = *reinterpret_cast<float2 *>(&s[i]);
        r += m[i] + v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char *name, int instr_per_i) {
    float *out;
    cudaMalloc(&out, 148 * 2 * 4 * 256 * sizeof(float));
    int iters = 40000;
    dim3 grid(148 * 2 * 4), block(256);
    k<MODE><<<grid, block>>>(out, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    double warp_instr = (double)grid.x * (block.x / 32) * iters * 16 * instr_per_i;
    double cycles = ms * 1e-3 * 1965e6;   // at max clock
    printf("%-26s %8.2f ms   %.3f warp-instr/clk/SMSP (at 1965 MHz)\n", name, ms, warp_instr / cycles / (148 * 4));
    cudaFree(out);
}

int main() {
    run<0>("FADD2+FMNMX3", 2);
    run<1>("FADD2", 1);
    run<2>("FMNMX3", 1);
    run<3>("FMNMX", 1);
    run<4>("FFMA2", 1);
    run<5>("FADD2+2xFMNMX", 3);
    run<6>("FADD+FMNMX", 2);
    return 0;
}
