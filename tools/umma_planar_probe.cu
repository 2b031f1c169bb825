// Probe: tcgen05.mma kind::tf32 with K-major SWIZZLE_NONE "planar" operands
// (smem [k-chunk of 4][row][4 floats], rows 16 B apart, so an operand may
// start at ANY row: the implicit-conv tap shift becomes a descriptor offset).
//   mode 0: D[128][256] = A[128][8] . B[off + 0..255][8]^T, checks LBO/SBO
//           roles (lbo = plane stride, sbo = 128 B, and swapped)
//   mode 1: raw fp32 operands (low 13 mantissa bits set): reports whether
//           the tensor core truncates or rounds them to tf32
//   mode 2: throughput, cycles per 128x256x8 MMA (planar vs SWIZZLE_128B)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/umma_planar_probe tools/umma_planar_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2205_00618_b200/csrc/tf32x3_gemm.cuh"
using namespace lsb::tc;

constexpr int RB = 320;   // B rows held in smem (256 + max offset)

__device__ uint64_t desc_planar(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;   // version; layout bits 61-63 = 0 (SWIZZLE_NONE)
    return d;
}

__global__ void probe(const float *A, const float *B, float *D, int off, int swap, int iters, long long *cyc,
                      int sw128) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    float *sa = reinterpret_cast<float *>(smem);                    // 2 planes x 128 rows x 16 B = 4 KB
    float *sb = reinterpret_cast<float *>(smem + 4096);             // 2 planes x RB rows x 16 B
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 4096 + 2 * RB * 16 + 1024);
    uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 1);
    const int t = threadIdx.x;
    for (int e = t; e < 128 * 8; e += blockDim.x) {
        const int m = e / 8, k = e % 8;
        sa[(k >> 2) * 128 * 4 + m * 4 + (k & 3)] = A[m * 8 + k];
    }
    for (int e = t; e < RB * 8; e += blockDim.x) {
        const int n = e / 8, k = e % 8;
        sb[(k >> 2) * RB * 4 + n * 4 + (k & 3)] = B[n * 8 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (t == 0) {
        const uint32_t idesc = idesc_tf32(128, 256);
        uint64_t a, b;
        if (!swap) {
            a = desc_planar(smem_u32(sa), 128 * 16, 128);
            b = desc_planar(smem_u32(sb) + off * 16, RB * 16, 128);
        } else {
            a = desc_planar(smem_u32(sa), 128, 128 * 16);
            b = desc_planar(smem_u32(sb) + off * 16, 128, RB * 16);
        }
        if (sw128) {   // throughput reference: SWIZZLE_128B descriptors (values meaningless)
            a = sdesc_k_sw<128>(smem_u32(sa));
            b = sdesc_k_sw<128>(smem_u32(sb));
        }
        long long c0 = clock64();
        for (int i = 0; i < iters; i++) umma_tf32(tmem, a, b, idesc, i ? 1u : 0u);
        umma_commit(bar);
        mbar_wait(bar, 0);
        long long c1 = clock64();
        if (cyc) *cyc = c1 - c0;
    }
    __syncwarp();
    mbar_wait(bar, 0);
    tc_fence_after();
    if (t < 128) {
        const int q = t >> 5;
        float v[16];
        for (int part = 0; part < 16; part++) {
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + part * 16, v);
            for (int i = 0; i < 16; i++) D[t * 256 + part * 16 + i] = v[i];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// mode 3: the conv kernel's stage pattern on one CTA: per stage 2 k8 steps x
// (A . Bhi, A . Blo), A from a rotating 6-slot ring, B shifted by the tap
// offset, a tcgen05.commit per stage (variant bits: 1 = no per-stage commit,
// 2 = constant A slot, 4 = constant B offset)
__global__ void stage_probe(int stages, int variant, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    // halo 8 planes x 384 rows x 16 B = 48 KB, filter ring 6 x 8 KB
    const uint32_t halo = smem_u32(smem), fring = halo + 8 * 6144;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 8 * 6144 + 6 * 8192);
    uint64_t *fin = bar + 1;
    uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 2);
    const int t = threadIdx.x;
    if (t == 0) {
        mbar_init(bar, 1);
        mbar_init(fin, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (t == 0) {
        const uint32_t idesc = idesc_tf32(128, 256);
        long long c0 = clock64();
        for (int st = 0; st < stages; st++) {
            const int tap = st % 9, r = tap / 3, s2 = tap % 3;
            const uint32_t off = (variant & 4) ? 0u : (uint32_t)(r * 58 + s2) * 16u;
            const uint32_t fa = fring + ((variant & 2) ? 0 : (st % 6)) * 8192;
            for (int k = 0; k < 2; k++) {
                const uint64_t a = desc_planar(fa + k * 2 * 2048, 2048, 128);
                const uint64_t bhi = desc_planar(halo + k * 2 * 6144 + off, 6144, 128);
                const uint64_t blo = desc_planar(halo + (4 + k * 2) * 6144 + off, 6144, 128);
                umma_tf32(tmem, a, bhi, idesc, (st | k) ? 1u : 0u);
                umma_tf32(tmem, a, blo, idesc, 1u);
            }
            if (!(variant & 1)) umma_commit(bar);
        }
        umma_commit(fin);
        mbar_wait(fin, 0);
        long long c1 = clock64();
        *cyc = c1 - c0;
    }
    tc_fence_before();
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

static float trunc_tf32(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xffffe000u;
    memcpy(&x, &u, 4);
    return x;
}
static float rna_tf32_h(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u += 0x1000u;
    u &= 0xffffe000u;
    memcpy(&x, &u, 4);
    return x;
}

int main() {
    const size_t smem = 4096 + 2 * RB * 16 + 1024 + 64 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    std::vector<float> A(128 * 8), B(RB * 8), D(128 * 256);
    float *dA, *dB, *dD;
    long long *dc;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMalloc(&dc, 8);
    srand(1);
    // mode 0: tf32-exact small integers
    for (auto &x : A) x = (float)(rand() % 7 - 3);
    for (auto &x : B) x = (float)(rand() % 7 - 3);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int swap = 0; swap < 1; swap++)
        for (int off : {0, 1, 3, 7, 58, 59, 63}) {
            probe<<<1, 128, smem>>>(dA, dB, dD, off, swap, 1, nullptr, 0);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode0 swap=%d off=%d: %s\n", swap, off, cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
            double err = 0;
            for (int m = 0; m < 128; m++)
                for (int n = 0; n < 256; n++) {
                    double r = 0;
                    for (int k = 0; k < 8; k++) r += (double)A[m * 8 + k] * B[(n + off) * 8 + k];
                    err = fmax(err, fabs(r - D[m * 256 + n]));
                }
            printf("mode0 layout lbo=%s off=%d max_err=%g\n", swap ? "128(sbo=plane)" : "plane(sbo=128)", off, err);
        }
    // mode 1: raw fp32 operands with low bits set, one product per output
    for (int m = 0; m < 128; m++)
        for (int k = 0; k < 8; k++) A[m * 8 + k] = k == 0 ? 1.0f + (float)(m + 1) * 1.3e-4f + 3.1e-7f : 0.f;
    for (int n = 0; n < RB; n++)
        for (int k = 0; k < 8; k++) B[n * 8 + k] = k == 0 ? 1.0f + (float)(n + 1) * 0.77e-4f + 1.9e-7f : 0.f;
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    probe<<<1, 128, smem>>>(dA, dB, dD, 0, 0, 1, nullptr, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int same_tr = 0, same_rna = 0, same_full = 0;
    for (int m = 0; m < 128; m++)
        for (int n = 0; n < 256; n++) {
            const float a = A[m * 8], b = B[n * 8], d = D[m * 256 + n];
            same_tr += d == (float)((double)trunc_tf32(a) * trunc_tf32(b));
            same_rna += d == (float)((double)rna_tf32_h(a) * rna_tf32_h(b));
            same_full += d == (float)((double)a * b);
        }
    printf("mode1 raw fp32 inputs: matches trunc %d, rna %d, full %d of %d\n", same_tr, same_rna, same_full, 128 * 256);
    // mode 2: throughput by B start row (a misaligned 128-B core matrix may cost
    // two shared-memory wavefronts)
    for (int off : {0, 1, 2, 4, 8, 58, 59}) {
        probe<<<1, 128, smem>>>(dA, dB, dD, off, 0, 2048, dc, 0);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("mode2 planar off=%d: %.1f cycles per 128x256x8 MMA\n", off, (double)c / 2048);
    }
    {
        const size_t sm3 = 8 * 6144 + 6 * 8192 + 64 + 1024;
        cudaFuncSetAttribute(stage_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
        for (int v : {0, 1, 2, 4, 7}) {
            stage_probe<<<1, 128, sm3>>>(360, v, dc);
            cudaError_t e = cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
            printf("mode3 variant %d: %.1f cycles per stage (4 MMAs) %s\n", v, (double)c / 360,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
