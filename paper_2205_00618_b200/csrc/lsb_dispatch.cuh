// lsb_dispatch.cuh -- launcher tables shared by the API TU (lsb_api.cu) and
// the kernel-instantiation TUs (kern_*.cu, compiled in parallel).
#pragma once

#include "affine_nest.cuh"
#include "semiring_gemm.cuh"

namespace lsb {

using GemmFn = void (*)(const GemmArgs &, dim3, cudaStream_t);
using ConvFn = void (*)(const ConvArgs &, dim3, size_t, cudaStream_t);
using SplitFn = void (*)(const GemmArgs &, int64_t, cudaStream_t);
using NestFn = void (*)(const NestArgs &, cudaStream_t);

int device_sms();                               // lsb_api.cu
int report_error(int code, const char *msg);    // lsb_api.cu: sets lsb_last_error

// Environment knobs, read once -- at the first use or on
// lsb_reload_env() -- never on the launch path.  Defaults are the measured best.
constexpr int kAlgoTf32x3Nhwc = 3;     // LSB_GEMM_ALGO=tf32x3_nhwc (convs: the NHWC-copy kernel)
constexpr int kAlgoTf32x3Planar = 4;   // LSB_GEMM_ALGO=tf32x3_planar (convs: the planar kernel)
struct Knobs {
    int gemm_algo;        // LSB_GEMM_ALGO: LSB_ALGO_AUTO | LSB_ALGO_SIMT | LSB_ALGO_TF32X3 | kAlgoTf32x3Nhwc
    int tc_chunk_k;       // LSB_TC_CHUNK_K: TMEM accumulation chunk depth (0 = auto)
    int tc_cfg;           // LSB_TC_CFG: -1 auto, 0 = 16x128, 1 = 32x128, 2 = 16x256
    int mp_mode;          // LSB_MP_MODE: 0 duo (default), 1 cluster, 2 streamk, 3 fixup (two CTAs per SM)
    int fixup_ctas, mp_cluster, streamk_ctas, conv_splits;   // 0 = model's choice
    int duo_bk;           // LSB_DUO_BK: slice depth of the duo max-plus kernel (8 | 16)
    int cp_dbg;           // LSB_CP_DBG: planar conv timing experiments (conv_planar.cuh)
    int cp_ctas;          // LSB_CP_CTAS: planar conv grid size (0 = one CTA per SM)
    int cp_nt;            // LSB_CP_NT: planar conv pixel tile (128 / 192 / 256; 0 = by tile count)
    bool scalar_split, no_pair, no_tail_split, no_persist, no_fast_epi, no_ilv;
    bool no_nest_fast;    // LSB_NO_NEST_FAST: every nest through affine_nest_kernel
    bool no_small, no_streamk, no_mp_fast, no_mp_cluster, no_conv_split;
    char gemm_trace[256], conv_trace[256];   // "" = off
};
const Knobs &knobs();
void reload_knobs();
// optional timing of the dominant kernel of a call (lsb_profile): which = 0
// before its launch, 1 after; no-op unless profiling is enabled
void prof_mark(int which, cudaStream_t s);

// the 32-bit row-walking / tiled-transpose nest kernels (nest_fast.cuh):
// returns 0 when the nest does not qualify (caller runs affine_nest_kernel),
// 1 = nest_rows_kernel, 2 = nest_transpose_kernel, 3 = nest_vec4_kernel, 4 = nest_pool_kernel, 5 = nest_transpose4_kernel launched
int launch_nest_fast(const lsb_nest_desc &d, const EpiStages &epi, cudaStream_t s);

GemmFn fast_gemm(int combine, int reduce, int bm, bool two_level);   // kern_fast.cu (nullptr if untuned)
void launch_conv_fast(const ConvArgs &a, dim3 grid, size_t dyn, cudaStream_t s);
void launch_conv_fold(const ConvArgs &a, int64_t n_img, cudaStream_t s);
void launch_streamk(int reduce, const GemmArgs &a, int ctas, cudaStream_t s);   // 2 launches
void launch_streamk_fast(int reduce, const GemmArgs &a, int ctas, cudaStream_t s);   // 2 launches
int launch_small_gemm(int combine, int reduce, const GemmArgs &a, int64_t batch, cudaStream_t s);   // -1: no kernel
int maxplus_fixup_ctas(int64_t units);   // co-resident CTA budget (cooperative launch)
int maxplus_duo_ctas(int64_t units, int bk);   // one 512-thread CTA per SM (maxplus_duo_kernel), bk = 8 | 16
int launch_maxplus_duo(int reduce, const GemmArgs &a, int bk, int ctas, float4 *part, int *flags, int epoch,
                       cudaStream_t s);
int launch_maxplus_fixup(int reduce, const GemmArgs &a, int ctas, float4 *part, int *flags, int epoch,
                         cudaStream_t s);   // 1 launch
int launch_maxplus_cluster(int reduce, const GemmArgs &a, int splits, cudaStream_t s);   // 1 launch
extern const GemmFn kGemmGeneric[4][4];          // kern_generic.cu
extern const SplitFn kSplit[4];                  // kern_generic.cu
extern const NestFn kNest[4][4];                 // kern_nest.cu

// 3xTF32 tcgen05 path (kern_tf32.cu)
bool tf32x3_supported(int64_t M, int64_t N, int64_t K);
int tf32x3_gemm(int64_t M, int64_t N, int64_t K, const float *A, int64_t sa_m, int64_t sa_k, const float *B,
                int64_t sb_k, int64_t sb_n, float *C, int64_t sc_m, int64_t sc_n, int c_vec, const EpiStages &epi,
                bool b_unchanged, int tile_n, cudaStream_t s, int *aux_launches, char *err, size_t errlen);
int tf32x3_gemm_blocked(const lsb_gemm_desc *d, const EpiStages &epi, int c_vec, cudaStream_t s, int *aux_launches,
                        char *err, size_t errlen);
bool tf32x3_conv_nhwc_ok(const ConvArgs &c, int64_t n_img);
int tf32x3_conv_nhwc(const ConvArgs &c, int64_t n_img, cudaStream_t s, int *aux_launches, char *err,
                     size_t errlen);
bool conv_planar_ok(const ConvArgs &c, int64_t n_img);
int conv_planar_nt(const ConvArgs &c, int64_t n_img);   // its pixel tile (0: not eligible)
int conv_planar(const ConvArgs &c, int64_t n_img, cudaStream_t s, int *aux_launches, char *err, size_t errlen);

template <int C, int R, bool B, int BM, bool TWO = false>
void launch_gemm(const GemmArgs &a, dim3 grid, cudaStream_t s) {
    constexpr size_t dyn = gemm_dyn_smem<BM>();
    static bool attr = false;   // > 48 KiB dynamic smem needs an opt-in, once per kernel
    if (!attr) {
        cudaFuncSetAttribute(semiring_gemm_kernel<C, R, B, BM, TWO>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        attr = true;
    }
    semiring_gemm_kernel<C, R, B, BM, TWO><<<grid, kThreads, dyn, s>>>(a);
}

}  // namespace lsb
