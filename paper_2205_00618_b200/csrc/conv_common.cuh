// conv_common.cuh -- pieces shared by the tensor-core conv kernels: 1-D bulk
// copies, TMEM loads without a wait, and the SWIZZLE_64B filter stage images
// of the NHWC conv (tf32x3_conv_nhwc.cuh).
#pragma once

#include "tf32x3_gemm.cuh"

namespace lsb {
namespace tc {

constexpr int CT_BN = 64;                 // output channels per filter tile
constexpr int CT_BK = 16;                 // taps per stage

// 1-D bulk copy global -> shared, completion on an mbarrier (tx bytes)
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// 32 lanes x 16 columns, no wait (pair with tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
}

// 32 lanes x 32 columns, no wait (pair with tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

// filters W[co][c][r][s] -> the exact shared-memory image of every stage's B
// operand: [co tile][stage][hi | lo][64 co rows x 16 taps, K-major SWIZZLE_64B],
// taps in (r, s, c) order, so one 8 KiB bulk copy feeds a stage (a 2-D TMA
// box of 64-B rows costs one request per row)
// (tap k -> (r, s) = k / Cp, channel c = k % Cp; zero for c >= C or k >= K)
// One thread per element with 32-bit index decomposition (the int64 div/mod
// chain per element made this tiny prepass take 4.9 us on C3).  The body is
// shared with the NHWC conv's fused prepass (extra blocks of its X split).
struct FilterImgArgs {
    const float *w;
    int64_t CO, K, Kp, C, Cp, S;
    int64_t sw[4];
    float *img;
    // 0: rows 0-63 hi, 64-127 lo; 1: channel c's hi / lo rows at
    // 32 (c / 16) + 2 (c % 16) and +1 (tf32x3_conv_nhwc_t_kernel)
    int ilv_rows;
};

__device__ __forceinline__ void filter_image_body(const FilterImgArgs &f, int *any, int gen, int first, int step) {
    const int nkb = (int)(f.Kp / CT_BK);
    const int co_tiles = (int)((f.CO + CT_BN - 1) / CT_BN);
    const int total = co_tiles * nkb * CT_BN * CT_BK;
    const int cp = (int)f.Cp, sS = (int)f.S, kK = (int)f.K, cC = (int)f.C;
    for (int e = first; e < total; e += step) {
        const int kk = e & (CT_BK - 1), n = (e >> 4) & (CT_BN - 1);
        const int t = e >> 10;   // / (CT_BK * CT_BN)
        const int kb = t % nkb, ct = t / nkb;
        const int64_t co = (int64_t)ct * CT_BN + n;
        const int k = kb * CT_BK + kk;
        const int rs = k / cp, c = k - rs * cp;
        float v = 0.0f;
        if (co < f.CO && k < kK && c < cC) {
            const int r = rs / sS, sx = rs - r * sS;
            v = __ldg(f.w + co * f.sw[0] + c * f.sw[1] + r * f.sw[2] + sx * f.sw[3]);
        }
        const float h = rna_tf32(v);
        const float l = tf32_lo(v, h);
        if (any != nullptr && !(fabsf(v) < __int_as_float(0x7f800000))) *any = gen;
        float *base = f.img + ((int64_t)(ct * nkb + kb) * 2) * (CT_BN * CT_BK);
        // row R of the 128-row K-major SW64 image: 16 floats, 16-B chunks XOR (R >> 1) & 3
        const int rh = f.ilv_rows ? 32 * (n >> 4) + 2 * (n & 15) : n;
        const int rl = f.ilv_rows ? rh + 1 : CT_BN + n;
        base[rh * 16 + (((kk >> 2) ^ ((rh >> 1) & 3)) << 2) + (kk & 3)] = h;
        base[rl * 16 + (((kk >> 2) ^ ((rl >> 1) & 3)) << 2) + (kk & 3)] = l;
    }
}

__global__ void __launch_bounds__(256) filter_image_kernel(const FilterImgArgs f, int *__restrict__ any, int gen) {
    asm volatile("griddepcontrol.launch_dependents;");
    filter_image_body(f, any, gen, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

}  // namespace tc
}  // namespace lsb
