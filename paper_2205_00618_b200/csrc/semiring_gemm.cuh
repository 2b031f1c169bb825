// semiring_gemm.cuh -- register-blocked FP32 semiring contraction for sm_100a.
//
// One CTA owns a BM x 128 output tile (BM = 128 or 64) and walks the
// reduction in BK = 8 slices.  256 threads; each owns TM x 8 outputs
// (TM = BM/16) split in 4-row / 4-column quads 64 apart, so the per-k
// fragment reads from shared memory are 128-bit and bank-conflict free.
// Global -> register prefetch of slice t+1 overlaps the math on slice t;
// shared memory is double buffered (one __syncthreads per slice).
//
// The inner loop is where the reference VM spends all its time
// (vm.py:112-136, the vop/vfma body of a register-blocked region,
// backend.py:930-971).  Here it is specialised per operator pair:
//   (mul, add)  FFMA2      : 2 FMAs / instruction, a[i] broadcast (.F32)
//   (add, max)  FADD2+FMNMX3: two k-steps folded per 3-input max
//   (add, min)  FADD2+FMNMX3
//   others      scalar combine + reduce (+ beta per term when required)
// FADD/FMNMX round exactly like the VM's f32 vop.add / max, so max/min
// semirings are bit-identical to float32(reference_eval).
//
// Loaders (template): plain strided GEMM operands, or implicit-GEMM conv
// (A = filters, B = im2col gather with out-of-range taps reading `fill`).
#pragma once

#include "lsb_common.cuh"

namespace lsb {

constexpr int kBN = 128;
constexpr int kBK = 8;
constexpr int kThreads = 256;
constexpr int kChunkSlices = 32;   // two-level accumulation: fold every 32*BK = 256 k

// ---------------------------------------------------------------------------
// problem descriptors as seen by the device
// ---------------------------------------------------------------------------

enum LoadMode { LD_GENERIC = 0, LD_VEC_K = 1, LD_VEC_MN = 2 };

struct GemmArgs {
    int64_t M, N, K;
    const float *A; int64_t sa_b, sa_m, sa_k;
    const float *B; int64_t sb_b, sb_k, sb_n;
    float *C; int64_t sc_b, sc_m, sc_n;
    int a_mode, b_mode, c_vec;
    float beta;
    int64_t k_per_split;  // reduction slice handled by one blockIdx.y-split
    int splits;
    float *ws;            // split-K partials [splits][batch][M][N] or null
    EpiStages epi;
};

struct ConvArgs {
    int64_t M, N, K;       // M = CO, N = HO*WO, K = C*R*S
    int64_t C, H, W, R, S, HO, WO;
    int64_t stride_h, stride_w, pad_h, pad_w, dil_h, dil_w;
    float fill;
    const float *x; int64_t sx0, sx1, sx2, sx3;
    const float *w; int64_t sw0, sw1, sw2, sw3;
    float *o; int64_t so0, so1, so2, so3;
    int a_mode;            // LD_VEC_K when filters are (c,r,s)-contiguous
    float beta;
    int64_t k_per_split;   // split-K over the (c, r, s) taps (grid y = co tiles * splits)
    int splits;
    float *ws;             // partials [splits][img][co][pixel] or null
    EpiStages epi;
};

// ---------------------------------------------------------------------------
// loaders: global -> registers (prefetch), registers -> shared (transpose)
// A smem tile: As[BK][BM + 4]  (k-major; +4 pad breaks transposed-store conflicts)
// B smem tile: Bs[BK][BN]
// ---------------------------------------------------------------------------

template <int BM>
struct GemmLoader {
    static constexpr int kAPer = BM * kBK / kThreads;   // A elements per thread (4 or 2)
    float ra[4];
    float rb[4];

    __device__ __forceinline__ void load(const GemmArgs &p, int64_t bz, int64_t m0, int64_t n0,
                                         int64_t k0, int64_t kend) {
        const int t = threadIdx.x;
        const float *A = p.A + bz * p.sa_b;
        const float *B = p.B + bz * p.sb_b;
        // ---- A tile (BM x BK)
        if (p.a_mode == LD_VEC_K) {
            // float4 along k: (m, kq..kq+3)
            if (t < BM * 2) {
                int64_t m = m0 + (t >> 1);
                int64_t k = k0 + (t & 1) * 4;
                if (m < p.M && k < kend) {
                    float4 v = __ldg(reinterpret_cast<const float4 *>(A + m * p.sa_m + k));
                    ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
                } else {
                    ra[0] = ra[1] = ra[2] = ra[3] = 0.0f;
                }
            }
        } else if (p.a_mode == LD_VEC_MN) {
            // float4 along m: (mq..mq+3, k)
            if (t < BM * 2) {
                int64_t k = k0 + t / (BM / 4);
                int64_t m = m0 + (t % (BM / 4)) * 4;
                if (m < p.M && k < kend) {
                    float4 v = __ldg(reinterpret_cast<const float4 *>(A + m + k * p.sa_k));
                    ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
                } else {
                    ra[0] = ra[1] = ra[2] = ra[3] = 0.0f;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < kAPer; j++) {
                int e = t + j * kThreads;
                int64_t m = m0 + e % BM;
                int64_t k = k0 + e / BM;
                ra[j] = (m < p.M && k < kend) ? __ldg(A + m * p.sa_m + k * p.sa_k) : 0.0f;
            }
        }
        // ---- B tile (BK x BN)
        if (p.b_mode == LD_VEC_MN) {
            int64_t k = k0 + (t >> 5);
            int64_t n = n0 + (t & 31) * 4;
            if (n < p.N && k < kend) {
                float4 v = __ldg(reinterpret_cast<const float4 *>(B + k * p.sb_k + n));
                rb[0] = v.x; rb[1] = v.y; rb[2] = v.z; rb[3] = v.w;
            } else {
                rb[0] = rb[1] = rb[2] = rb[3] = 0.0f;
            }
        } else if (p.b_mode == LD_VEC_K) {
            int64_t n = n0 + (t >> 1);
            int64_t k = k0 + (t & 1) * 4;
            if (n < p.N && k < kend) {
                float4 v = __ldg(reinterpret_cast<const float4 *>(B + n * p.sb_n + k));
                rb[0] = v.x; rb[1] = v.y; rb[2] = v.z; rb[3] = v.w;
            } else {
                rb[0] = rb[1] = rb[2] = rb[3] = 0.0f;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                int e = t + j * kThreads;
                int64_t n = n0 + e % kBN;
                int64_t k = k0 + e / kBN;
                rb[j] = (n < p.N && k < kend) ? __ldg(B + k * p.sb_k + n * p.sb_n) : 0.0f;
            }
        }
    }

    __device__ __forceinline__ void store(const GemmArgs &p, float (*As)[BM + 4],
                                          float (*Bs)[kBN]) {
        const int t = threadIdx.x;
        if (p.a_mode == LD_VEC_K) {
            if (t < BM * 2) {
                int m = t >> 1, kq = (t & 1) * 4;
#pragma unroll
                for (int j = 0; j < 4; j++) As[kq + j][m] = ra[j];
            }
        } else if (p.a_mode == LD_VEC_MN) {
            if (t < BM * 2) {
                int k = t / (BM / 4), m = (t % (BM / 4)) * 4;
                *reinterpret_cast<float4 *>(&As[k][m]) = make_float4(ra[0], ra[1], ra[2], ra[3]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < kAPer; j++) {
                int e = t + j * kThreads;
                As[e / BM][e % BM] = ra[j];
            }
        }
        if (p.b_mode == LD_VEC_MN) {
            *reinterpret_cast<float4 *>(&Bs[t >> 5][(t & 31) * 4]) =
                make_float4(rb[0], rb[1], rb[2], rb[3]);
        } else if (p.b_mode == LD_VEC_K) {
            int n = t >> 1, kq = (t & 1) * 4;
#pragma unroll
            for (int j = 0; j < 4; j++) Bs[kq + j][n] = rb[j];
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                int e = t + j * kThreads;
                Bs[e / kBN][e % kBN] = rb[j];
            }
        }
    }
};

// Implicit-GEMM conv loader.  B(k, p) = x[n, ci, ho*sh + r*dh - ph, wo*sw + s*dw - pw]
// with (ci, r, s) = k and (ho, wo) = p; per-k offsets come from a smem table
// built once per CTA so the gather costs two compares and one add per tap.
struct ConvLoader {
    float ra[4];
    float rb[4];
    int64_t pix_off[4];   // n*sx0 + hbase*sx2 + wbase*sx3 for my 4 pixels
    int hb[4], wb[4];     // ho*sh - ph, wo*sw - pw (or a huge value if the pixel is out of range)

    __device__ __forceinline__ void init(const ConvArgs &p, int64_t img, int64_t n0) {
        const int t = threadIdx.x;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int64_t pix = n0 + (t & 31) * 4 + j;
            if (pix < p.N) {
                int64_t ho = pix / p.WO, wo = pix % p.WO;
                hb[j] = (int)(ho * p.stride_h - p.pad_h);
                wb[j] = (int)(wo * p.stride_w - p.pad_w);
                pix_off[j] = img * p.sx0 + (int64_t)hb[j] * p.sx2 + (int64_t)wb[j] * p.sx3;
            } else {
                hb[j] = -(1 << 30);
                wb[j] = -(1 << 30);
                pix_off[j] = 0;
            }
        }
    }

    template <int BM>
    __device__ __forceinline__ void load(const ConvArgs &p, const int64_t *koff, const int2 *krs,
                                         int64_t m0, int64_t k0, int64_t kend) {
        const int t = threadIdx.x;
        // ---- A = filters (co, k)
        if (p.a_mode == LD_VEC_K) {
            if (t < BM * 2) {
                int64_t m = m0 + (t >> 1);
                int64_t k = k0 + (t & 1) * 4;
                if (m < p.M && k < kend) {
                    float4 v = __ldg(reinterpret_cast<const float4 *>(p.w + m * p.sw0 + k));
                    ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
                } else {
                    ra[0] = ra[1] = ra[2] = ra[3] = 0.0f;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < BM * kBK / kThreads; j++) {
                int e = t + j * kThreads;
                int64_t m = m0 + e % BM;
                int64_t k = k0 + e / BM;
                float v = 0.0f;
                if (m < p.M && k < kend) {
                    int64_t rs = p.R * p.S;
                    int64_t ci = k / rs, r = (k % rs) / p.S, s = k % p.S;
                    v = __ldg(p.w + m * p.sw0 + ci * p.sw1 + r * p.sw2 + s * p.sw3);
                }
                ra[j] = v;
            }
        }
        // ---- B = im2col gather (k, pixel)
        int64_t k = k0 + (t >> 5);
        if (k < kend) {
            int64_t ko = koff[k];
            int2 rs = krs[k];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                int hi = hb[j] + rs.x, wi = wb[j] + rs.y;
                bool ok = (unsigned)hi < (unsigned)p.H && (unsigned)wi < (unsigned)p.W;
                rb[j] = ok ? __ldg(p.x + pix_off[j] + ko) : p.fill;
            }
        } else {
            rb[0] = rb[1] = rb[2] = rb[3] = 0.0f;
        }
    }

    template <int BM>
    __device__ __forceinline__ void store(const ConvArgs &p, float (*As)[BM + 4], float (*Bs)[kBN]) {
        const int t = threadIdx.x;
        if (p.a_mode == LD_VEC_K) {
            if (t < BM * 2) {
                int m = t >> 1, kq = (t & 1) * 4;
#pragma unroll
                for (int j = 0; j < 4; j++) As[kq + j][m] = ra[j];
            }
        } else {
#pragma unroll
            for (int j = 0; j < BM * kBK / kThreads; j++) {
                int e = t + j * kThreads;
                As[e / BM][e % BM] = ra[j];
            }
        }
        *reinterpret_cast<float4 *>(&Bs[t >> 5][(t & 31) * 4]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
    }
};

// the register-blocked micro-kernel
// ---------------------------------------------------------------------------

template <int TM>
struct Frag {
    float a[TM];
    float b[8];
};

template <int OPC, int OPR, bool BETA, int TM>
struct Micro {
    // acc[i][jp] holds outputs (row i, cols 2jp, 2jp+1) of the thread's TM x 8 block
    float2 acc[TM][4];

    static constexpr bool kFFMA2 = OPC == LSB_OP_MUL && OPR == LSB_OP_ADD && !BETA;
    static constexpr bool kMAX3 = OPC == LSB_OP_ADD && (OPR == LSB_OP_MAX || OPR == LSB_OP_MIN) && !BETA;

    __device__ __forceinline__ void init() {
        const float id = Op<OPR>::identity();
#pragma unroll
        for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) acc[i][j] = make_float2(id, id);
    }

    __device__ __forceinline__ static void frag(const float *As_k, const float *Bs_k, int ty, int tx,
                                                Frag<TM> &f) {
        float4 a0 = *reinterpret_cast<const float4 *>(As_k + ty * 4);
        f.a[0] = a0.x; f.a[1] = a0.y; f.a[2] = a0.z; f.a[3] = a0.w;
        if constexpr (TM == 8) {
            float4 a1 = *reinterpret_cast<const float4 *>(As_k + 64 + ty * 4);
            f.a[4] = a1.x; f.a[5] = a1.y; f.a[6] = a1.z; f.a[7] = a1.w;
        }
        float4 b0 = *reinterpret_cast<const float4 *>(Bs_k + tx * 4);
        float4 b1 = *reinterpret_cast<const float4 *>(Bs_k + 64 + tx * 4);
        f.b[0] = b0.x; f.b[1] = b0.y; f.b[2] = b0.z; f.b[3] = b0.w;
        f.b[4] = b1.x; f.b[5] = b1.y; f.b[6] = b1.z; f.b[7] = b1.w;
    }

    // one k step
    __device__ __forceinline__ void step1(const Frag<TM> &f, float beta) {
#pragma unroll
        for (int i = 0; i < TM; i++) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float2 bb = make_float2(f.b[2 * j], f.b[2 * j + 1]);
                if constexpr (kFFMA2) {
                    acc[i][j] = __ffma2_rn(make_float2(f.a[i], f.a[i]), bb, acc[i][j]);
                } else if constexpr (kMAX3) {
                    float2 s = __fadd2_rn(make_float2(f.a[i], f.a[i]), bb);
                    acc[i][j].x = Op<OPR>::apply(acc[i][j].x, s.x);
                    acc[i][j].y = Op<OPR>::apply(acc[i][j].y, s.y);
                } else {
                    float s0 = Op<OPC>::apply(f.a[i], bb.x);
                    float s1 = Op<OPC>::apply(f.a[i], bb.y);
                    if constexpr (BETA) { s0 = __fmul_rn(beta, s0); s1 = __fmul_rn(beta, s1); }
                    acc[i][j].x = Op<OPR>::apply(acc[i][j].x, s0);
                    acc[i][j].y = Op<OPR>::apply(acc[i][j].y, s1);
                }
            }
        }
    }

    // two k steps folded into one 3-input max/min (FADD2 + FMNMX3)
    __device__ __forceinline__ void step2(const Frag<TM> &f0, const Frag<TM> &f1) {
#pragma unroll
        for (int i = 0; i < TM; i++) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                float2 s = __fadd2_rn(make_float2(f0.a[i], f0.a[i]), make_float2(f0.b[2 * j], f0.b[2 * j + 1]));
                float2 u = __fadd2_rn(make_float2(f1.a[i], f1.a[i]), make_float2(f1.b[2 * j], f1.b[2 * j + 1]));
                acc[i][j].x = Op<OPR>::apply(acc[i][j].x, Op<OPR>::apply(s.x, u.x));
                acc[i][j].y = Op<OPR>::apply(acc[i][j].y, Op<OPR>::apply(s.y, u.y));
            }
        }
    }

    // a full BK slice.  Single-step operator pairs keep the next k's fragment
    // in flight while the current one computes; the fragment for k = 0 of the
    // next slice is loaded by the caller-provided hook after the slice barrier.
    template <int BM, class Boundary>
    __device__ __forceinline__ void full_slice(float (*As)[BM + 4], float (*Bs)[kBN], int ty, int tx,
                                               float beta, Frag<TM> (&f)[2], Boundary &&boundary) {
        if constexpr (kMAX3) {
#pragma unroll
            for (int kk = 0; kk < kBK; kk += 2) {
                Frag<TM> f1;
                if (kk > 0) frag(As[kk], Bs[kk], ty, tx, f[0]);
                frag(As[kk + 1], Bs[kk + 1], ty, tx, f1);
                step2(f[0], f1);
                // after the last pair: barrier + next slice's k = 0 into f[0]
                // (three live fragments would not fit 128 registers)
                if (kk == kBK - 2) boundary(f[0]);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < kBK; kk++) {
                if (kk < kBK - 1) frag(As[kk + 1], Bs[kk + 1], ty, tx, f[(kk + 1) & 1]);
                else boundary(f[(kk + 1) & 1]);
                step1(f[kk & 1], beta);
            }
        }
    }

    template <int BM>
    __device__ __forceinline__ void tail_slice(float (*As)[BM + 4], float (*Bs)[kBN], int kcount,
                                               int ty, int tx, float beta) {
#pragma unroll 1
        for (int kk = 0; kk < kcount; kk++) {
            Frag<TM> f0;
            frag(As[kk], Bs[kk], ty, tx, f0);
            step1(f0, beta);
        }
    }

    __device__ __forceinline__ float get(int i, int j) const {
        return (j & 1) ? acc[i][j >> 1].y : acc[i][j >> 1].x;
    }

    // two-level accumulation: add the chunk into the CTA-private smem total
    // (each thread owns its slots, no barrier) and restart the chunk.
    __device__ __forceinline__ void fold(float2 *tot) {
        const float id = Op<OPR>::identity();
#pragma unroll
        for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) {
                float2 *t = tot + (i * 4 + j) * kThreads + threadIdx.x;
                float2 v = *t;
                v.x = Op<OPR>::apply(v.x, acc[i][j].x);
                v.y = Op<OPR>::apply(v.y, acc[i][j].y);
                *t = v;
                acc[i][j] = make_float2(id, id);
            }
    }
    __device__ __forceinline__ void unfold(const float2 *tot) {
#pragma unroll
        for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float2 v = tot[(i * 4 + j) * kThreads + threadIdx.x];
                acc[i][j].x = Op<OPR>::apply(v.x, acc[i][j].x);
                acc[i][j].y = Op<OPR>::apply(v.y, acc[i][j].y);
            }
    }
};

// row / column of the thread's (i, j) output inside the CTA tile
template <int TM>
__device__ __forceinline__ int row_of(int ty, int i) { return (i < 4 ? 0 : 64) + ty * 4 + (i & 3); }
__device__ __forceinline__ int col_of(int tx, int j) { return (j < 4 ? 0 : 64) + tx * 4 + (j & 3); }

// dynamic shared memory of the GEMM kernel: the two-level chunk totals /
// epilogue staging area, TM*8 floats per thread
template <int BM>
constexpr size_t gemm_dyn_smem() { return (size_t)(BM / 16) * 8 * kThreads * sizeof(float); }

// ---------------------------------------------------------------------------
// GEMM kernel
// grid: x = n tiles, y = m tiles * splits, z = batch
// ---------------------------------------------------------------------------

// reduction over [kbeg, kend) of one output tile into mk (smem double buffer
// As/Bs; stage2 holds the two-level totals when TWO)
template <int BM, bool TWO, class MK>
__device__ __forceinline__ void mainloop(const GemmArgs &p, int64_t bz, int64_t m0, int64_t n0, int64_t kbeg,
                                         int64_t kend, MK &mk, float (*As)[kBK][BM + 4], float (*Bs)[kBK][kBN],
                                         float2 *stage2, int tx, int ty) {
    constexpr int TM = BM / 16;
    if (kbeg >= kend) return;
    GemmLoader<BM> ld;
    ld.load(p, bz, m0, n0, kbeg, kend);
    ld.store(p, As[0], Bs[0]);
    __syncthreads();
    Frag<TM> f[2];
    MK::frag(As[0][0], Bs[0][0], ty, tx, f[0]);
    int buf = 0;
    int chunk = 0;
    for (int64_t k0 = kbeg; k0 < kend; k0 += kBK) {
        const bool more = k0 + kBK < kend;
        if (more) ld.load(p, bz, m0, n0, k0 + kBK, kend);
        if (k0 + kBK <= kend) {
            // barrier + next slice's first fragment, issued before the
            // last k step of this slice so its latency overlaps the math
            auto boundary = [&](Frag<TM> &nf) {
                if (more) ld.store(p, As[buf ^ 1], Bs[buf ^ 1]);
                __syncthreads();
                if (more) MK::frag(As[buf ^ 1][0], Bs[buf ^ 1][0], ty, tx, nf);
            };
            mk.template full_slice<BM>(As[buf], Bs[buf], ty, tx, p.beta, f, boundary);
        } else {
            mk.template tail_slice<BM>(As[buf], Bs[buf], (int)(kend - k0), ty, tx, p.beta);
        }
        if constexpr (TWO) {
            if (++chunk == kChunkSlices) {
                mk.fold(stage2);
                chunk = 0;
            }
        }
        buf ^= 1;
    }
}

// order-preserving float max/min through integer atomics (exact, so the
// result does not depend on the order partial tiles arrive in)
// A NaN partial must win (np.max propagates it): for max it is stored as
// 0x7fffffff (above +inf as int, below every negative float as unsigned),
// for min as 0xffffffff (below every positive float as int, above every
// negative float as unsigned), so no later partial can displace it.
__device__ __forceinline__ void atomic_max_f32(float *a, float v) {
    if (v != v) atomicMax(reinterpret_cast<int *>(a), 0x7fffffff);
    else if (v >= 0.0f) atomicMax(reinterpret_cast<int *>(a), __float_as_int(v));
    else atomicMin(reinterpret_cast<unsigned *>(a), __float_as_uint(v));
}
__device__ __forceinline__ void atomic_min_f32(float *a, float v) {
    if (v != v) atomicMax(reinterpret_cast<unsigned *>(a), 0xffffffffu);
    else if (v >= 0.0f) atomicMin(reinterpret_cast<int *>(a), __float_as_int(v));
    else atomicMax(reinterpret_cast<unsigned *>(a), __float_as_uint(v));
}

// Stream-K for (add, max|min) without epilogue: the tiles x k-slices work is
// cut into gridDim.x equal contiguous ranges, so every SM slot gets the same
// work however few tiles there are (C2: 64 tiles on 296 slots); partial tiles
// merge with exact atomic max/min into C, pre-filled with the identity.
template <int OPC, int OPR, int BM>
__global__ void __launch_bounds__(kThreads, 2) semiring_streamk_kernel(const GemmArgs p) {
    constexpr int TM = BM / 16;
    __shared__ __align__(16) float As[2][kBK][BM + 4];
    __shared__ __align__(16) float Bs[2][kBK][kBN];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t m_tiles = (p.M + BM - 1) / BM, n_tiles = (p.N + kBN - 1) / kBN;
    const int64_t kslices = (p.K + kBK - 1) / kBK;
    const int64_t units = m_tiles * n_tiles * kslices;
    const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    using MK = Micro<OPC, OPR, false, TM>;
    for (int64_t u = u0; u < u1;) {
        const int64_t tile = u / kslices, ks = u % kslices;
        const int64_t seg_end = min(u1, (tile + 1) * kslices);
        const int64_t kbeg = ks * kBK, kend = min(p.K, (seg_end - tile * kslices) * kBK);
        const int64_t m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * kBN;
        MK mk;
        mk.init();
        __syncthreads();   // previous segment's readers are done with As/Bs
        mainloop<BM, false>(p, 0, m0, n0, kbeg, kend, mk, As, Bs, nullptr, tx, ty);
#pragma unroll
        for (int i = 0; i < TM; i++) {
            const int64_t m = m0 + row_of<TM>(ty, i);
            if (m >= p.M) continue;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int64_t n = n0 + col_of(tx, j);
                if (n >= p.N) continue;
                float *dst = p.C + m * p.sc_m + n * p.sc_n;
                if constexpr (OPR == LSB_OP_MAX) atomic_max_f32(dst, mk.get(i, j));
                else atomic_min_f32(dst, mk.get(i, j));
            }
        }
        u = seg_end;
    }
}

template <int kUnused = 0>
__global__ void fill_kernel(float *C, int64_t M, int64_t N, int64_t sc_m, int64_t sc_n, float v) {
    const int64_t total = M * N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x)
        C[(e / N) * sc_m + (e % N) * sc_n] = v;
}

template <int OPC, int OPR, bool BETA, int BM, bool TWO = false>
__global__ void __launch_bounds__(kThreads, 2) semiring_gemm_kernel(const GemmArgs p) {
    constexpr int TM = BM / 16;
    __shared__ __align__(16) float As[2][kBK][BM + 4];
    __shared__ __align__(16) float Bs[2][kBK][kBN];
    extern __shared__ __align__(16) float2 stage2[];   // [TM*4][kThreads] float2

    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t m_tiles = (p.M + BM - 1) / BM;
    const int64_t split = blockIdx.y / m_tiles;
    const int64_t m0 = (blockIdx.y % m_tiles) * BM;
    const int64_t n0 = (int64_t)blockIdx.x * kBN;
    const int64_t bz = blockIdx.z;
    const int64_t kbeg = split * p.k_per_split;
    const int64_t kend = min(p.K, kbeg + p.k_per_split);

    using MK = Micro<OPC, OPR, BETA, TM>;
    MK mk;
    mk.init();
    if constexpr (TWO) {
        const float id = Op<OPR>::identity();
        for (int e = threadIdx.x; e < TM * 4 * kThreads; e += kThreads) stage2[e] = make_float2(id, id);
    }
    mainloop<BM, TWO>(p, bz, m0, n0, kbeg, kend, mk, As, Bs, stage2, tx, ty);
    if constexpr (TWO) mk.unfold(stage2);

    // ---- epilogue
    if (p.ws != nullptr) {
        // split-K partial: raw accumulators, folded by splitk_epilogue_kernel
        float *W = p.ws + ((split * gridDim.z + bz) * p.M) * p.N;
#pragma unroll
        for (int i = 0; i < TM; i++) {
            int64_t m = m0 + row_of<TM>(ty, i);
            if (m >= p.M) continue;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                int64_t n = n0 + col_of(tx, j);
                if (n < p.N) W[m * p.N + n] = mk.get(i, j);
            }
        }
        return;
    }
    float *C = p.C + bz * p.sc_b;
    if (p.epi.n == 0) {
#pragma unroll
        for (int i = 0; i < TM; i++) {
            int64_t m = m0 + row_of<TM>(ty, i);
            if (m >= p.M) continue;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                int64_t nq = n0 + h * 64 + tx * 4;
                if (p.c_vec && nq + 3 < p.N) {
                    *reinterpret_cast<float4 *>(C + m * p.sc_m + nq) =
                        make_float4(mk.get(i, h * 4), mk.get(i, h * 4 + 1), mk.get(i, h * 4 + 2), mk.get(i, h * 4 + 3));
                } else {
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (nq + q < p.N) C[m * p.sc_m + (nq + q) * p.sc_n] = mk.get(i, h * 4 + q);
                }
            }
        }
        return;
    }
    // fused epilogue: stage the accumulators through shared memory so the
    // epilogue code is instantiated once (a rolled loop), not TM*8 times
    float *stage = reinterpret_cast<float *>(stage2);
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) stage[(i * 8 + j) * kThreads + threadIdx.x] = mk.get(i, j);
#pragma unroll 1
    for (int e = 0; e < TM * 2; e++) {
        const int i = e >> 1, h = e & 1;
        const int64_t m = m0 + row_of<TM>(ty, i);
        if (m >= p.M) continue;
        const int64_t nq = n0 + h * 64 + tx * 4;
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) v[q] = stage[(i * 8 + h * 4 + q) * kThreads + threadIdx.x];
        if (nq + 3 < p.N) {
            apply_epilogue4(p.epi, v, bz, m, nq, 0);
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (nq + q < p.N) v[q] = apply_epilogue(p.epi, v[q], bz, m, nq + q, 0);
        }
        if (p.c_vec && nq + 3 < p.N) {
            *reinterpret_cast<float4 *>(C + m * p.sc_m + nq) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (nq + q < p.N) C[m * p.sc_m + (nq + q) * p.sc_n] = v[q];
        }
    }
}

// fold split-K partials in split order (deterministic), then the epilogue
template <int OPR>
__global__ void splitk_epilogue_kernel(const GemmArgs p, int64_t batch) {
    const int64_t total = batch * p.M * p.N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        // partial loads batched 8 at a time (independent L2 round trips in
        // flight), folded strictly in split order
        float x = __ldcg(p.ws + e);
        int s = 1;
        for (; s + 8 <= p.splits; s += 8) {
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; q++) v[q] = __ldcg(p.ws + (s + q) * total + e);
#pragma unroll
            for (int q = 0; q < 8; q++) x = Op<OPR>::apply(x, v[q]);
        }
        for (; s < p.splits; s++) x = Op<OPR>::apply(x, __ldcg(p.ws + s * total + e));
        int64_t n = e % p.N, m = (e / p.N) % p.M, bz = e / (p.N * p.M);
        if (p.epi.n) x = apply_epilogue(p.epi, x, bz, m, n, 0);
        p.C[bz * p.sc_b + m * p.sc_m + n * p.sc_n] = x;
    }
}

// ---------------------------------------------------------------------------
// conv kernel: grid x = pixel tiles, y = co tiles, z = images
// ---------------------------------------------------------------------------

constexpr int kConvTableMax = 8192;   // K = C*R*S entries cached in smem

template <int OPC, int OPR, bool BETA, int BM>
__global__ void __launch_bounds__(kThreads, 2) conv_igemm_kernel(const ConvArgs p) {
    constexpr int TM = BM / 16;
    __shared__ __align__(16) float As[2][kBK][BM + 4];
    __shared__ __align__(16) float Bs[2][kBK][kBN];
    extern __shared__ __align__(16) unsigned char dyn[];
    int64_t *koff = reinterpret_cast<int64_t *>(dyn);
    int2 *krs = reinterpret_cast<int2 *>(dyn + sizeof(int64_t) * p.K);

    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t m_tiles = (p.M + BM - 1) / BM;
    const int64_t split = blockIdx.y / m_tiles;
    const int64_t m0 = (blockIdx.y % m_tiles) * BM;
    const int64_t n0 = (int64_t)blockIdx.x * kBN;
    const int64_t img = blockIdx.z;
    const int64_t kbeg = split * p.k_per_split;
    const int64_t kend = min(p.K, kbeg + p.k_per_split);
    const int64_t rs = p.R * p.S;
    for (int64_t k = threadIdx.x; k < p.K; k += kThreads) {
        int64_t ci = k / rs, r = (k % rs) / p.S, s = k % p.S;
        int rr = (int)(r * p.dil_h), ss = (int)(s * p.dil_w);
        koff[k] = ci * p.sx1 + (int64_t)rr * p.sx2 + (int64_t)ss * p.sx3;
        krs[k] = make_int2(rr, ss);
    }
    ConvLoader ld;
    ld.init(p, img, n0);
    __syncthreads();

    using MK = Micro<OPC, OPR, BETA, TM>;
    MK mk;
    mk.init();
    ld.load<BM>(p, koff, krs, m0, kbeg, kend);
    ld.store<BM>(p, As[0], Bs[0]);
    __syncthreads();
    Frag<TM> f[2];
    MK::frag(As[0][0], Bs[0][0], ty, tx, f[0]);
    int buf = 0;
    for (int64_t k0 = kbeg; k0 < kend; k0 += kBK) {
        const bool more = k0 + kBK < kend;
        if (more) ld.load<BM>(p, koff, krs, m0, k0 + kBK, kend);
        if (k0 + kBK <= kend) {
            auto boundary = [&](Frag<TM> &nf) {
                if (more) ld.store<BM>(p, As[buf ^ 1], Bs[buf ^ 1]);
                __syncthreads();
                if (more) MK::frag(As[buf ^ 1][0], Bs[buf ^ 1][0], ty, tx, nf);
            };
            mk.template full_slice<BM>(As[buf], Bs[buf], ty, tx, p.beta, f, boundary);
        } else {
            mk.template tail_slice<BM>(As[buf], Bs[buf], (int)(kend - k0), ty, tx, p.beta);
        }
        buf ^= 1;
    }

    if (p.ws != nullptr) {
        // split-K partial, folded (in split order) by conv_splitk_fold_kernel
        float *W = p.ws + ((split * gridDim.z + img) * p.M) * p.N;
#pragma unroll
        for (int i = 0; i < TM; i++) {
            const int64_t co = m0 + row_of<TM>(ty, i);
            if (co >= p.M) continue;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int64_t pq = n0 + h * 64 + tx * 4;
                if (pq + 3 < p.N && (p.N & 3) == 0) {
                    *reinterpret_cast<float4 *>(W + co * p.N + pq) =
                        make_float4(mk.get(i, h * 4), mk.get(i, h * 4 + 1), mk.get(i, h * 4 + 2), mk.get(i, h * 4 + 3));
                } else {
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (pq + q < p.N) W[co * p.N + pq + q] = mk.get(i, h * 4 + q);
                }
            }
        }
        return;
    }

#pragma unroll
    for (int i = 0; i < TM; i++) {
        int64_t co = m0 + row_of<TM>(ty, i);
        if (co >= p.M) continue;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            int64_t pix = n0 + col_of(tx, j);
            if (pix >= p.N) continue;
            int64_t ho = pix / p.WO, wo = pix % p.WO;
            float x = mk.get(i, j);
            if (p.epi.n) x = apply_epilogue(p.epi, x, img, co, ho, wo);
            p.o[img * p.so0 + co * p.so1 + ho * p.so2 + wo * p.so3] = x;
        }
    }
}

// fold the conv split-K partials (split order, deterministic) + epilogue
template <int kUnused = 0>
__global__ void conv_splitk_fold_kernel(const ConvArgs p, int64_t n_img) {
    const int64_t total = n_img * p.M * p.N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        float x = __ldcg(p.ws + e);
        int s = 1;
        for (; s + 8 <= p.splits; s += 8) {
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; q++) v[q] = __ldcg(p.ws + (s + q) * total + e);
#pragma unroll
            for (int q = 0; q < 8; q++) x += v[q];
        }
        for (; s < p.splits; s++) x += __ldcg(p.ws + s * total + e);
        const int64_t pix = e % p.N, co = (e / p.N) % p.M, img = e / (p.N * p.M);
        const int64_t ho = pix / p.WO, wo = pix % p.WO;
        if (p.epi.n) x = apply_epilogue(p.epi, x, img, co, ho, wo);
        p.o[img * p.so0 + co * p.so1 + ho * p.so2 + wo * p.so3] = x;
    }
}

}  // namespace lsb
