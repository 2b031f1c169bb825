// Timeline of maxplus_fixup_kernel on C2 (1024^3): per-CTA %globaltimer stamps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2205_00618_b200/csrc -I include \
//      tools/dbg/mp_trace.cu -o tools/dbg/mp_trace && tools/dbg/mp_trace > gpurun_out/mp_trace.txt
#define LSB_MP_TRACE 1
#ifndef DUO_BK
#define DUO_BK 8
#endif
#include <cstdio>
#include <vector>
#include "maxplus_fast.cuh"
using namespace lsb;
int main(int argc, char **argv) {
    const int64_t M = 1024, N = 1024, K = 1024;
    const int coop = argc > 1 ? atoi(argv[1]) : 1;
    const int duo = argc > 2 ? atoi(argv[2]) : 1;
    float *A, *B, *C;
    cudaMalloc(&A, M * K * 4); cudaMalloc(&B, K * N * 4); cudaMalloc(&C, M * N * 4);
    std::vector<float> h(M * K);
    for (size_t i = 0; i < h.size(); i++) h[i] = (float)((i * 2654435761u) % 20000) / 1000.f - 10.f;
    cudaMemcpy(A, h.data(), M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(B, h.data(), K * N * 4, cudaMemcpyHostToDevice);
    GemmArgs a = {};
    a.M = M; a.N = N; a.K = K;
    a.A = A; a.sa_m = K; a.sa_k = 1;
    a.B = B; a.sb_k = N; a.sb_n = 1;
    a.C = C; a.sc_m = N; a.sc_n = 1; a.c_vec = 1; a.beta = 1.f;
    cudaFuncSetAttribute(maxplus_fixup_kernel<LSB_OP_MAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMpSmemBytes);
    int occ = 0, sms = 0;
    cudaFuncSetAttribute(maxplus_duo_kernel<LSB_OP_MAX, DUO_BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DuoCfg<DUO_BK>::kSmemBytes);
    if (duo) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, maxplus_duo_kernel<LSB_OP_MAX, DUO_BK>, kDuoThreads, DuoCfg<DUO_BK>::kSmemBytes);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, maxplus_fixup_kernel<LSB_OP_MAX>, kThreads, kMpSmemBytes);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int G = occ * sms;
    float4 *part; int *flags; long long *trace;
    cudaMalloc(&part, sizeof(float4) * 16 * kThreads * G);
    cudaMalloc(&flags, 4 * G); cudaMemset(flags, 0, 4 * G);
    cudaMalloc(&trace, 8 * 16 * G);
    cudaMemcpyToSymbol(g_mp_trace, &trace, sizeof(trace));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int epoch = 1; epoch <= 6; epoch++) {
        cudaMemset(trace, 0, 8 * 16 * G);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G); cfg.blockDim = dim3(duo ? kDuoThreads : kThreads); cfg.dynamicSmemBytes = duo ? DuoCfg<DUO_BK>::kSmemBytes : kMpSmemBytes;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = coop;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaEventRecord(e0);
        cudaError_t e = duo ? cudaLaunchKernelEx(&cfg, maxplus_duo_kernel<LSB_OP_MAX, DUO_BK>, a, part, flags, epoch)
                            : cudaLaunchKernelEx(&cfg, maxplus_fixup_kernel<LSB_OP_MAX>, a, part, flags, epoch);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        cudaEventElapsedTime(&ms, e0, e1);
        if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    }
    std::vector<long long> t(16 * G);
    cudaMemcpy(t.data(), trace, 8 * 16 * G, cudaMemcpyDeviceToHost);
    long long t0 = -1;
    for (int b = 0; b < G; b++) { long long v = t[b * 16 + 1] & 0x00ffffffffffffffll; if (t0 < 0 || v < t0) t0 = v; }
    printf("# duo=%d G=%d coop=%d last launch %.4f ms; per CTA: cta sm then tag:ns-since-first-start\n", duo, G, coop, ms);
    for (int b = 0; b < G; b++) {
        printf("%3d %3lld", b, t[b * 16]);
        for (int i = 1; i < 16 && t[b * 16 + i]; i++)
            printf(" %lld:%lld", t[b * 16 + i] >> 56, (t[b * 16 + i] & 0x00ffffffffffffffll) - t0);
        printf("\n");
    }
    return 0;
}
