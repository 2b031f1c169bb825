// Probe: tcgen05.mma kind::tf32 with an MN-major SWIZZLE_128B A operand.
// D[128][64] = A[128][16] * B[64][16]^T, A MN-major (pixel-contiguous atoms),
// B K-major SWIZZLE_64B; tries LBO/SBO variants and reports max error.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_2205_00618_b200/csrc/tf32x3_conv.cuh"
using namespace lsb::tc;

__global__ void probe(const float *A, const float *B, float *D, uint32_t lbo, uint32_t sbo, int kmajor_a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    float *sa = reinterpret_cast<float *>(smem);            // 8 KB
    float *sb = reinterpret_cast<float *>(smem + 8192);     // 4 KB
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 12288);
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem + 12296);
    int t = threadIdx.x;
    for (int e = t; e < 128 * 16; e += blockDim.x) {
        int m = e / 16, k = e % 16;
        uint32_t off;
        if (kmajor_a) {
            off = (k >> 3) * 0 + m * 64 + (((k >> 2) ^ ((m >> 1) & 3)) << 4) + (k & 3) * 4;   // sw64 K-major (16 taps/row)
        } else {
            int r = k & 3;   // SWIZZLE_128B_BASE32B: 32-B granules XOR row (4-row atoms)
            off = (k >> 2) * (sbo ? sbo : 2048) + (m >> 5) * (lbo ? lbo : 512) + r * 128 + ((((m & 31) >> 3) ^ r) << 5) + (m & 7) * 4;
        }
        sa[off / 4] = A[m * 16 + k];
    }
    for (int e = t; e < 64 * 16; e += blockDim.x) {
        int n = e / 16, k = e % 16;
        uint32_t off = n * 64 + (((k >> 2) ^ ((n >> 1) & 3)) << 4) + (k & 3) * 4;
        sb[off / 4] = B[n * 16 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tmem = *slot;
    if (t == 0) {
        uint32_t idesc = idesc_tf32(128, 64) | (kmajor_a ? 0u : (1u << 15));
        uint32_t abase = smem_u32(sa), bbase = smem_u32(sb);
        for (int k = 0; k < 2; k++) {
            uint64_t a;
            if (kmajor_a) a = sdesc_k_sw<64>(abase) + (uint64_t)((k * 32) >> 4);
            else {
                a = 0;
                a |= (uint64_t)(((abase + k * 2 * sbo) >> 4) & 0x3FFF);
                a |= (uint64_t)(lbo >> 4) << 16;
                a |= (uint64_t)(sbo >> 4) << 32;
                a |= (uint64_t)1 << 46;
                a |= (uint64_t)1 << 61;
            }
            uint64_t b = sdesc_k_sw<64>(bbase) + (uint64_t)((k * 32) >> 4);
            umma_tf32(tmem, a, b, idesc, k ? 1u : 0u);
        }
        umma_commit(bar);
    }
    mbar_wait(bar, 0);
    tc_fence_after();
    if (t < 128) {
        int q = (t >> 5);
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

// conv-pattern stage: for k in 0..1: N=128 (A hi, SW128 K-major) + N=64 (A lo at +64 B);
// B K-major SW64 (128 rows).  mode 0: that; mode 1: A SW64 (separate hi/lo tiles);
// mode 2: three N=64 MMAs per k (the old pattern); mode 3: N=256 x 2 per k (GEMM-like)
__global__ void conv_pattern(int mode, int n_iter, long long *out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 65536);
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem + 65600);
    int t = threadIdx.x;
    for (int e = t; e < 16384; e += blockDim.x) reinterpret_cast<float *>(smem)[e] = 0.5f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) { mbar_init(bar, 1); mbar_init(bar + 2, 1 << 20); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tmem = *slot;
    if (t == 0) {
        const uint32_t base = smem_u32(smem);
        const uint32_t i64 = idesc_tf32(128, 64), i128 = idesc_tf32(128, 128), i256 = idesc_tf32(128, 256);
        long long t0 = clock64();
        for (int it = 0; it < n_iter; it++) {
            if (mode >= 9) {   // mode 9/10/11: channel-major conv stage, A = SW64 filter image
                               // (128 rows), B = SW128 X box (hi, lo at +64 B), N = 128 / 224 / 256
                const uint64_t b = sdesc_k_sw<128>(base), a = sdesc_k_sw<64>(base + 32768);
                const uint32_t id = mode == 9 ? idesc_tf32(128, 128) : mode == 10 ? idesc_tf32(128, 224) : idesc_tf32(128, 256);
                for (int k = 0; k < 2; k++) {
                    const uint64_t off = (uint64_t)((k * 32) >> 4);
                    umma_tf32(tmem, a + off, b + off, id, 1u);
                    umma_tf32(tmem, a + off, b + 4 + off, id, 1u);
                }
                continue;
            }
            if (mode >= 6) {   // mode 6/7/8: M=64 N=256 / M=64 N=128 / M=128 N=256, 2 per k
                const uint64_t a = sdesc_k_sw<64>(base), b = sdesc_k_sw<64>(base + 32768);
                const uint32_t id = mode == 6 ? idesc_tf32(64, 256) : mode == 7 ? idesc_tf32(64, 128) : idesc_tf32(128, 256);
                for (int k = 0; k < 2; k++) {
                    const uint64_t off = (uint64_t)((k * 32) >> 4);
                    umma_tf32(tmem, a + off, b + off, id, 1u);
                    umma_tf32(tmem, a + off, b + off, id, 1u);
                }
                continue;
            }
            if (mode >= 4) {   // mode 4: conv stage + commit every stage; 5: every 4th stage
                const uint64_t a = sdesc_k_sw<128>(base), b = sdesc_k_sw<64>(base + 32768);
                for (int k = 0; k < 2; k++) {
                    const uint64_t off = (uint64_t)((k * 32) >> 4);
                    umma_tf32(tmem, a + off, b + off, i128, 1u);
                    umma_tf32(tmem, a + 4 + off, b + off, i64, 1u);
                }
                if (mode == 4 || (it & 3) == 3) umma_commit(bar + 2);
                continue;
            }
            for (int k = 0; k < 2; k++) {
                const uint64_t off = (uint64_t)((k * 32) >> 4);
                if (mode == 0) {
                    const uint64_t a = sdesc_k_sw<128>(base), b = sdesc_k_sw<64>(base + 32768);
                    umma_tf32(tmem, a + off, b + off, i128, 1u);
                    umma_tf32(tmem, a + 4 + off, b + off, i64, 1u);
                } else if (mode == 1) {
                    const uint64_t a = sdesc_k_sw<64>(base), al = sdesc_k_sw<64>(base + 8192), b = sdesc_k_sw<64>(base + 32768);
                    umma_tf32(tmem, a + off, b + off, i128, 1u);
                    umma_tf32(tmem, al + off, b + off, i64, 1u);
                } else if (mode == 2) {
                    const uint64_t a = sdesc_k_sw<64>(base), al = sdesc_k_sw<64>(base + 8192), b = sdesc_k_sw<64>(base + 32768), bl = sdesc_k_sw<64>(base + 36864);
                    umma_tf32(tmem, a + off, b + off, i64, 1u);
                    umma_tf32(tmem, a + off, bl + off, i64, 1u);
                    umma_tf32(tmem, al + off, b + off, i64, 1u);
                } else {
                    const uint64_t a = sdesc_k_sw<64>(base), al = sdesc_k_sw<64>(base + 8192), b = sdesc_k_sw<64>(base + 32768);
                    umma_tf32(tmem, a + off, b + off, i256, 1u);
                    umma_tf32(tmem, a + off, b + off, i256, 1u);
                    umma_tf32(tmem, al + off, b + off, i256, 1u);
                }
            }
        }
        umma_commit(bar);
        mbar_wait(bar, 0);
        long long t1 = clock64();
        out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

__global__ void mma_lat(int kmajor_a, int n_iter, int per, long long *out, int nn) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 32768);
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem + 32776);
    int t = threadIdx.x;
    for (int e = t; e < 8192; e += blockDim.x) reinterpret_cast<float *>(smem)[e] = 0.5f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) { mbar_init(bar, 1); mbar_init(bar + 2, 1 << 20); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tmem = *slot;
    if (t == 0) {
        uint32_t idesc = idesc_tf32(128, nn) | (kmajor_a ? 0u : (1u << 15));
        uint32_t base = smem_u32(smem);
        uint64_t a = kmajor_a ? sdesc_k_sw<64>(base) : sdesc_mn_sw128_32b(base);
        uint64_t b = sdesc_k_sw<64>(base + 16384);
        long long t0 = clock64();
        for (int it = 0; it < n_iter; it++) {
            for (int j = 0; j < per; j++) umma_tf32(tmem, a, b, idesc, 1u);
            umma_commit(bar);
            mbar_wait(bar, it & 1);
        }
        long long t1 = clock64();
        out[0] = t1 - t0;
        // throughput: no waits
        t0 = clock64();
        for (int it = 0; it < n_iter; it++)
            for (int j = 0; j < per; j++) umma_tf32(tmem, a, b, idesc, 1u);
        umma_commit(bar);
        mbar_wait(bar, n_iter & 1);
        t1 = clock64();
        out[1] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
    {
        long long *o2, hh;
        cudaMalloc(&o2, 8);
        cudaFuncSetAttribute(conv_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
        for (int mode = 0; mode < 12; mode++) {
            conv_pattern<<<1, 128, 70000>>>(mode, 200, o2);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(&hh, o2, 8, cudaMemcpyDeviceToHost);
            printf("conv pattern mode %d %s: %.1f cycles per 16-tap stage\n", mode, cudaGetErrorString(e), hh / 200.0);
        }
    }
    {
        long long *o, h[2];
        cudaMalloc(&o, 16);
        cudaFuncSetAttribute(mma_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
        for (int km = 0; km < 2; km++)
            for (int nn : {64, 128, 256})
            for (int per : {6}) {
                mma_lat<<<1, 128, 40000>>>(km, 200, per, o, nn);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
                printf("kmajor=%d N=%d per=%d %s: latency/iter %.1f cyc, throughput %.1f cyc/mma\n", km, nn, per,
                       cudaGetErrorString(e), h[0] / 200.0, h[1] / (200.0 * per));
            }
    }
    float hA[128 * 16], hB[64 * 16], hD[128 * 64], ref[128 * 64];
    srand(1);
    for (auto &x : hA) x = (float)(rand() % 7 - 3);
    for (auto &x : hB) x = (float)(rand() % 5 - 2);
    for (int m = 0; m < 128; m++)
        for (int n = 0; n < 64; n++) {
            float s = 0;
            for (int k = 0; k < 16; k++) s += hA[m * 16 + k] * hB[n * 16 + k];
            ref[m * 64 + n] = s;
        }
    float *A, *B, *D;
    cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
    cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    struct { uint32_t lbo, sbo; int km; } v[] = {{0, 0, 1}, {512, 2048, 0}, {2048, 512, 0}};
    for (auto &c : v) {
        cudaMemset(D, 0, sizeof hD);
        probe<<<1, 128, 16384>>>(A, B, D, c.lbo, c.sbo, c.km);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
        double err = 0; int bad = 0;
        for (int i = 0; i < 128 * 64; i++) { double d = fabs(hD[i] - ref[i]); if (d > err) err = d; bad += d > 1e-3; }
        printf("kmajor=%d lbo=%u sbo=%u err=%s maxerr=%g bad=%d D[0..3]=%g %g %g %g ref=%g %g %g %g\n", c.km, c.lbo, c.sbo,
               cudaGetErrorString(e), err, bad, hD[0], hD[1], hD[64], hD[65], ref[0], ref[1], ref[64], ref[65]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
