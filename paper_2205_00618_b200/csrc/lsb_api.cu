// lsb_api.cu -- the C ABI (include/lsb.h): argument checking, kernel
// selection and launch.  Built with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared
// into paper_2205_00618_b200/liblsb.so (see paper_2205_00618_b200/build.py).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/lsb.h"
#include "lsb_dispatch.cuh"

namespace {

thread_local char g_err[512] = "";
std::atomic<int64_t> g_launches{0};

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define LSB_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(LSB_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),       \
                        __FILE__, __LINE__);                                               \
    } while (0)

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(LSB_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return LSB_OK;
}

int g_sm_count = 0;
int sm_count();
std::atomic<int> g_device{-1};   // the device lsb_init bound this process to

// compute entry points run on the bound device only (the caller's current
// device must be it)
int check_device() {
    const int bound = g_device.load(std::memory_order_relaxed);
    if (bound < 0) return fail(LSB_ERR_INVALID, "lsb_init was not called");
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != bound)
        return fail(LSB_ERR_UNSUPPORTED, "current device %d is not the device %d liblsb is bound to", cur, bound);
    return LSB_OK;
}

}  // namespace

int lsb::device_sms() { return sm_count(); }

int lsb::report_error(int code, const char *msg) { return fail(code, "%s", msg); }

namespace {
lsb::Knobs g_knobs;
std::once_flag g_knobs_once;
std::mutex g_knobs_mu;

void read_knobs(lsb::Knobs &k) {
    memset(&k, 0, sizeof(k));
    auto on = [](const char *n) { return getenv(n) != nullptr; };
    auto num = [](const char *n) { const char *e = getenv(n); return e ? atoi(e) : 0; };
    auto str = [](const char *n, char *dst) {
        const char *e = getenv(n);
        snprintf(dst, 256, "%s", e ? e : "");
    };
    k.gemm_algo = LSB_ALGO_AUTO;
    if (const char *e = getenv("LSB_GEMM_ALGO")) {
        if (!strcmp(e, "simt")) k.gemm_algo = LSB_ALGO_SIMT;
        else if (!strcmp(e, "tf32x3")) k.gemm_algo = LSB_ALGO_TF32X3;
        else if (!strcmp(e, "tf32x3_nhwc")) k.gemm_algo = lsb::kAlgoTf32x3Nhwc;
        else if (!strcmp(e, "tf32x3_planar")) k.gemm_algo = lsb::kAlgoTf32x3Planar;
    }
    k.tc_cfg = -1;
    if (const char *e = getenv("LSB_TC_CFG")) {
        if (!strcmp(e, "16x128")) k.tc_cfg = 0;
        else if (!strcmp(e, "32x128")) k.tc_cfg = 1;
        else if (!strcmp(e, "16x256")) k.tc_cfg = 2;
    }
    if (const char *e = getenv("LSB_MP_MODE")) k.mp_mode = !strcmp(e, "cluster") ? 1 : !strcmp(e, "streamk") ? 2 : !strcmp(e, "fixup") ? 3 : 0;
    k.fixup_ctas = num("LSB_FIXUP_CTAS");
    k.tc_chunk_k = num("LSB_TC_CHUNK_K");
    k.duo_bk = num("LSB_DUO_BK") == 8 ? 8 : num("LSB_DUO_BK") == 16 ? 16 : 32;
    k.mp_cluster = num("LSB_MP_CLUSTER");
    k.streamk_ctas = num("LSB_STREAMK_CTAS");
    k.conv_splits = num("LSB_CONV_SPLITS");
    k.cp_dbg = num("LSB_CP_DBG");
    k.cp_ctas = num("LSB_CP_CTAS");
    k.cp_nt = num("LSB_CP_NT");
    k.scalar_split = on("LSB_SCALAR_SPLIT");
    k.no_pair = on("LSB_NO_PAIR");
    k.no_tail_split = on("LSB_NO_TAIL_SPLIT");
    k.no_persist = on("LSB_NO_PERSIST");
    k.no_fast_epi = on("LSB_NO_FAST_EPI");
    k.no_ilv = on("LSB_NO_ILV");
    k.no_nest_fast = on("LSB_NO_NEST_FAST");
    k.no_small = on("LSB_NO_SMALL");
    k.no_streamk = on("LSB_NO_STREAMK");
    k.no_mp_fast = on("LSB_NO_MP_FAST");
    k.no_mp_cluster = on("LSB_NO_MP_CLUSTER");
    k.no_conv_split = on("LSB_NO_CONV_SPLIT");
    str("LSB_GEMM_TRACE", k.gemm_trace);
    str("LSB_CONV_TRACE", k.conv_trace);
}
}  // namespace

const lsb::Knobs &lsb::knobs() {
    std::call_once(g_knobs_once, [] { read_knobs(g_knobs); });
    return g_knobs;
}

void lsb::reload_knobs() {
    knobs();
    std::lock_guard<std::mutex> lk(g_knobs_mu);
    read_knobs(g_knobs);
}

namespace {
bool g_prof = false;
cudaEvent_t g_prof_ev[2] = {nullptr, nullptr};
}  // namespace

void lsb::prof_mark(int which, cudaStream_t s) {
    if (g_prof && g_prof_ev[which]) cudaEventRecord(g_prof_ev[which], s);
}

namespace {

int sm_count() {
    if (g_sm_count == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (g_sm_count <= 0) g_sm_count = 148;
    }
    return g_sm_count;
}

// split-K workspace (one per process, grown on demand; stream-ordered use)
std::mutex g_ws_mu;
float *g_ws = nullptr;
size_t g_ws_bytes = 0;

int workspace(size_t bytes, float **out) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (bytes > g_ws_bytes) {
        if (g_ws) {
            cudaDeviceSynchronize();
            cudaFree(g_ws);
            g_ws = nullptr;
            g_ws_bytes = 0;
        }
        LSB_CUDA(cudaMalloc(&g_ws, bytes));
        g_ws_bytes = bytes;
    }
    *out = g_ws;
    return LSB_OK;
}

// stream-K fixup buffers (maxplus_fixup_kernel): per-CTA partial tiles and
// epoch-stamped ready flags, zeroed once -- each launch stamps a new epoch,
// so flags never need a reset launch.  Stream-ordered use, like the split-K
// workspace: concurrent fixup launches on different streams would share them.
std::mutex g_fx_mu;
float4 *g_fx_part = nullptr;
int *g_fx_flags = nullptr;
int g_fx_ctas = 0, g_fx_epoch = 0;

int fixup_buffers(int ctas, float4 **part, int **flags, int *epoch) {
    std::lock_guard<std::mutex> lk(g_fx_mu);
    if (ctas > g_fx_ctas || g_fx_epoch >= 0x7ffffff0) {
        cudaDeviceSynchronize();
        cudaFree(g_fx_part);
        cudaFree(g_fx_flags);
        g_fx_part = nullptr;
        g_fx_flags = nullptr;
        g_fx_ctas = 0;
        LSB_CUDA(cudaMalloc(&g_fx_part, sizeof(float4) * 16 * lsb::kThreads * (size_t)ctas));
        LSB_CUDA(cudaMalloc(&g_fx_flags, sizeof(int) * (size_t)ctas));
        LSB_CUDA(cudaMemset(g_fx_flags, 0, sizeof(int) * (size_t)ctas));
        g_fx_ctas = ctas;
        g_fx_epoch = 0;
    }
    *part = g_fx_part;
    *flags = g_fx_flags;
    *epoch = ++g_fx_epoch;
    return LSB_OK;
}

bool valid_op(int op) { return op >= LSB_OP_ADD && op <= LSB_OP_MIN; }
bool valid_ew(int ew) { return ew >= LSB_EW_IDENTITY && ew <= LSB_EW_SIGMOID; }

int check_epi(int n, const lsb_epi_stage *s) {
    if (n < 0 || n > LSB_MAX_EPI) return fail(LSB_ERR_INVALID, "n_epi %d out of range", n);
    for (int i = 0; i < n; i++) {
        if (s[i].combine != -1 && !valid_op(s[i].combine))
            return fail(LSB_ERR_INVALID, "epi[%d].combine %d invalid", i, s[i].combine);
        if (s[i].combine != -1 && s[i].operand == nullptr)
            return fail(LSB_ERR_INVALID, "epi[%d] combine without operand", i);
        if (s[i].alpha != 0.0f && s[i].c_in == nullptr)
            return fail(LSB_ERR_INVALID, "epi[%d] alpha without c_in", i);
        if (!valid_op(s[i].reduce) || !valid_ew(s[i].pre) || !valid_ew(s[i].post))
            return fail(LSB_ERR_INVALID, "epi[%d] invalid op codes", i);
    }
    return LSB_OK;
}

// stages that leave x unchanged (no operand, beta 1, alpha 0, identity post)
// are dropped so plain contractions take the epilogue-free store path
lsb::EpiStages pack_epi(int n, const lsb_epi_stage *s) {
    lsb::EpiStages e;
    memset(&e, 0, sizeof(e));
    for (int i = 0; i < n; i++) {
        const bool noop = s[i].combine < 0 && s[i].beta == 1.0f && s[i].alpha == 0.0f &&
                          s[i].post == LSB_EW_IDENTITY;
        if (!noop) e.s[e.n++] = s[i];
    }
    return e;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------- dispatch
// kernel instantiations live in kern_*.cu so they compile in parallel
using lsb::GemmFn;
using lsb::ConvFn;
using lsb::SplitFn;
using lsb::NestFn;
using lsb::fast_gemm;
using lsb::kGemmGeneric;
using lsb::kNest;
using lsb::kSplit;

int pick_mode_a(const lsb_gemm_desc *d, int64_t sa_m, int64_t sa_k) {
    if (!aligned16(d->A) || (d->batch > 1 && d->sa_b % 4)) return lsb::LD_GENERIC;
    if (sa_k == 1 && sa_m % 4 == 0 && d->K % 4 == 0) return lsb::LD_VEC_K;
    if (sa_m == 1 && sa_k % 4 == 0 && d->M % 4 == 0) return lsb::LD_VEC_MN;
    return lsb::LD_GENERIC;
}
int pick_mode_b(const lsb_gemm_desc *d) {
    if (!aligned16(d->B) || (d->batch > 1 && d->sb_b % 4)) return lsb::LD_GENERIC;
    if (d->sb_n == 1 && d->sb_k % 4 == 0 && d->N % 4 == 0) return lsb::LD_VEC_MN;
    if (d->sb_k == 1 && d->sb_n % 4 == 0 && d->K % 4 == 0) return lsb::LD_VEC_K;
    return lsb::LD_GENERIC;
}

// GEMM algorithm the launcher uses for this descriptor (M = rows actually
// computed); -1 when an explicit request cannot be honoured
int select_algo(const lsb_gemm_desc *d, int64_t M) {
    int algo = d->algo;
    const int forced = lsb::knobs().gemm_algo;
    if (forced == LSB_ALGO_SIMT || forced == LSB_ALGO_TF32X3) algo = forced;
    const bool tc_ok = d->combine == LSB_OP_MUL && d->reduce == LSB_OP_ADD && !d->beta_in_loop &&
                       d->batch == 1 && d->K > 0;
    if (algo == LSB_ALGO_TF32X3) return tc_ok ? algo : -1;
    if (algo == LSB_ALGO_AUTO && tc_ok && M >= 128 && d->N >= 128 && d->K >= 256 &&
        (double)M * d->N * d->K >= (double)(1ll << 30) && lsb::tf32x3_supported(M, d->N, d->K))
        return LSB_ALGO_TF32X3;
    return LSB_ALGO_SIMT;
}

}  // namespace

extern "C" {

int lsb_gemm_algo(const lsb_gemm_desc *d) {
    if (!d) return fail(LSB_ERR_INVALID, "null desc");
    const int64_t m_begin = std::max<int64_t>(0, d->m_begin);
    const int64_t m_end = d->m_end > 0 ? std::min(d->m_end, d->M) : d->M;
    return select_algo(d, m_end - m_begin);
}

int lsb_abi_version(void) { return LSB_ABI_VERSION; }

int lsb_reload_env(void) {
    lsb::reload_knobs();
    return LSB_OK;
}

int lsb_last_error(char *buf, size_t len) {
    if (buf && len) {
        strncpy(buf, g_err, len - 1);
        buf[len - 1] = 0;
    }
    return LSB_OK;
}

int lsb_init(int device) {
    int n = 0;
    LSB_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return fail(LSB_ERR_INVALID, "device %d of %d", device, n);
    // one device per process: the workspaces, tensor-map entry point and
    // kernel smem attributes are process-wide (one process per GPU)
    int bound = -1;
    if (!g_device.compare_exchange_strong(bound, device) && bound != device)
        return fail(LSB_ERR_UNSUPPORTED, "liblsb is bound to device %d in this process; device %d needs its own process",
                    bound, device);
    LSB_CUDA(cudaSetDevice(device));
    int major = 0;
    LSB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) return fail(LSB_ERR_UNSUPPORTED, "device %d is sm_%d x, this build targets sm_100a", device, major);
    LSB_CUDA(cudaFree(nullptr));
    g_sm_count = 0;
    sm_count();
    return LSB_OK;
}

int lsb_device_info(int device, int *sms, int *cc_major, int *cc_minor, int *clock_khz) {
    if (sms) LSB_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device));
    if (cc_major) LSB_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
    if (cc_minor) LSB_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
    if (clock_khz) LSB_CUDA(cudaDeviceGetAttribute(clock_khz, cudaDevAttrClockRate, device));
    return LSB_OK;
}

int lsb_device_alloc(void **ptr, size_t bytes) {
    if (!ptr) return fail(LSB_ERR_INVALID, "null ptr");
    cudaError_t e = cudaMalloc(ptr, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) return fail(LSB_ERR_NOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    return LSB_OK;
}
int lsb_device_free(void *ptr) {
    LSB_CUDA(cudaFree(ptr));
    return LSB_OK;
}
int lsb_host_alloc(void **ptr, size_t bytes) {
    if (!ptr) return fail(LSB_ERR_INVALID, "null ptr");
    cudaError_t e = cudaHostAlloc(ptr, std::max<size_t>(bytes, 16), cudaHostAllocDefault);
    if (e != cudaSuccess) return fail(LSB_ERR_NOMEM, "cudaHostAlloc(%zu): %s", bytes, cudaGetErrorString(e));
    return LSB_OK;
}
int lsb_host_free(void *ptr) {
    LSB_CUDA(cudaFreeHost(ptr));
    return LSB_OK;
}
int lsb_memcpy_h2d(void *dst, const void *src, size_t bytes, void *stream) {
    LSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    return LSB_OK;
}
int lsb_memcpy_d2h(void *dst, const void *src, size_t bytes, void *stream) {
    LSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    return LSB_OK;
}
int lsb_memcpy_h2d_2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height,
                      void *stream) {
    LSB_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice,
                               (cudaStream_t)stream));
    return LSB_OK;
}

int lsb_memcpy_d2h_2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height,
                      void *stream) {
    LSB_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost,
                               (cudaStream_t)stream));
    return LSB_OK;
}

int lsb_memcpy_d2d(void *dst, const void *src, size_t bytes, void *stream) {
    LSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return LSB_OK;
}
int lsb_stream_sync(void *stream) {
    LSB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return LSB_OK;
}
int lsb_stream_create(void **stream) {
    if (!stream) return fail(LSB_ERR_INVALID, "null out");
    LSB_CUDA(cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t *>(stream), cudaStreamNonBlocking));
    return LSB_OK;
}
int lsb_stream_destroy(void *stream) {
    LSB_CUDA(cudaStreamDestroy((cudaStream_t)stream));
    return LSB_OK;
}
int lsb_event_create(void **event) {
    if (!event) return fail(LSB_ERR_INVALID, "null out");
    LSB_CUDA(cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t *>(event), cudaEventDisableTiming));
    return LSB_OK;
}
int lsb_event_destroy(void *event) {
    LSB_CUDA(cudaEventDestroy((cudaEvent_t)event));
    return LSB_OK;
}
int lsb_event_record(void *event, void *stream) {
    LSB_CUDA(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream));
    return LSB_OK;
}
int lsb_stream_wait_event(void *stream, void *event) {
    LSB_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0));
    return LSB_OK;
}

int lsb_profile(int enable) {
    if (enable && !g_prof_ev[0]) {
        LSB_CUDA(cudaEventCreate(&g_prof_ev[0]));
        LSB_CUDA(cudaEventCreate(&g_prof_ev[1]));
    }
    g_prof = enable != 0;
    return LSB_OK;
}

int lsb_last_kernel_ms(float *ms) {
    if (!ms) return fail(LSB_ERR_INVALID, "null out");
    if (!g_prof_ev[0]) return fail(LSB_ERR_INVALID, "profiling was never enabled");
    LSB_CUDA(cudaEventSynchronize(g_prof_ev[1]));
    LSB_CUDA(cudaEventElapsedTime(ms, g_prof_ev[0], g_prof_ev[1]));
    return LSB_OK;
}

int64_t lsb_sizeof(int which) {
    switch (which) {
    case 0: return (int64_t)sizeof(lsb_gemm_desc);
    case 1: return (int64_t)sizeof(lsb_conv_desc);
    case 2: return (int64_t)sizeof(lsb_nest_desc);
    case 3: return (int64_t)sizeof(lsb_epi_stage);
    default: return -1;
    }
}

int64_t lsb_launch_count(int reset) {
    return reset ? g_launches.exchange(0) : g_launches.load();
}

int lsb_semiring_gemm(const lsb_gemm_desc *d, void *stream) {
    if (!d) return fail(LSB_ERR_INVALID, "null desc");
    if (d->M < 0 || d->N < 0 || d->K < 0 || d->batch < 1)
        return fail(LSB_ERR_INVALID, "bad extents M=%lld N=%lld K=%lld batch=%lld",
                    (long long)d->M, (long long)d->N, (long long)d->K, (long long)d->batch);
    if (!valid_op(d->combine) || !valid_op(d->reduce))
        return fail(LSB_ERR_INVALID, "bad operator pair (%d, %d)", d->combine, d->reduce);
    if (!d->A || !d->B || !d->C) return fail(LSB_ERR_INVALID, "null operand");
    int rc = check_epi(d->n_epi, d->epi);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if ((rc = check_device())) return rc;

    if (d->flags & (LSB_GEMM_PREP_A | LSB_GEMM_PREP_B | LSB_GEMM_PRESPLIT)) {
        // blocked 3xTF32 sequence step: global coordinates throughout
        if (d->combine != LSB_OP_MUL || d->reduce != LSB_OP_ADD || d->batch != 1 || d->beta_in_loop ||
            d->beta != 1.0f || d->K == 0)
            return fail(LSB_ERR_UNSUPPORTED, "blocked tf32x3 steps cover batch-1 (mul, add) contractions");
        lsb::EpiStages epi = pack_epi(d->n_epi, d->epi);
        const int c_vec = (d->sc_n == 1 && aligned16(d->C) && d->sc_m % 4 == 0)
                              ? ((reinterpret_cast<uintptr_t>(d->C) % 32 == 0 && d->sc_m % 8 == 0) ? 2 : 1)
                              : 0;
        char err[256] = "";
        int aux = 0;
        rc = lsb::tf32x3_gemm_blocked(d, epi, c_vec, s, &aux, err, sizeof(err));
        if (rc) return fail(rc, "%s", err);
        rc = check_launch("tf32x3_gemm_blocked");
        if (rc) return rc;
        g_launches.fetch_add(aux + ((d->flags & LSB_GEMM_PRESPLIT) ? 1 : 0), std::memory_order_relaxed);
        return LSB_OK;
    }

    int64_t m_begin = std::max<int64_t>(0, d->m_begin);
    int64_t m_end = d->m_end > 0 ? std::min(d->m_end, d->M) : d->M;
    int64_t M = m_end - m_begin;
    if (M <= 0 || d->N == 0) return LSB_OK;

    lsb::GemmArgs a;
    memset(&a, 0, sizeof(a));
    a.M = M; a.N = d->N; a.K = d->K;
    a.A = d->A + m_begin * d->sa_m; a.sa_b = d->sa_b; a.sa_m = d->sa_m; a.sa_k = d->sa_k;
    a.B = d->B; a.sb_b = d->sb_b; a.sb_k = d->sb_k; a.sb_n = d->sb_n;
    a.C = d->C + m_begin * d->sc_m; a.sc_b = d->sc_b; a.sc_m = d->sc_m; a.sc_n = d->sc_n;
    a.beta = d->beta;
    a.epi = pack_epi(d->n_epi, d->epi);
    // row-sharded epilogue operands keep global coordinates: shift their bases
    for (int i = 0; i < a.epi.n; i++) {
        if (a.epi.s[i].operand) a.epi.s[i].operand += m_begin * a.epi.s[i].so[1];
        if (a.epi.s[i].c_in) a.epi.s[i].c_in += m_begin * a.epi.s[i].sc[1];
    }
    lsb_gemm_desc dd = *d;
    dd.A = a.A; dd.M = M;
    a.a_mode = pick_mode_a(&dd, d->sa_m, d->sa_k);
    a.b_mode = pick_mode_b(&dd);
    a.c_vec = (d->sc_n == 1 && aligned16(a.C) && d->sc_m % 4 == 0 && (d->batch == 1 || d->sc_b % 4 == 0)) ? 1 : 0;
    // 32-B aligned rows take 256-bit stores in the tensor-core GEMM's persistent epilogue
    if (a.c_vec && reinterpret_cast<uintptr_t>(a.C) % 32 == 0 && d->sc_m % 8 == 0 && (d->batch == 1 || d->sc_b % 8 == 0))
        a.c_vec = 2;

    // ---- algorithm: 3xTF32 tensor cores for large fp32 (mul, add) contractions
    const int algo = select_algo(d, M);
    if (algo < 0) return fail(LSB_ERR_UNSUPPORTED, "tf32x3 covers batch-1 (mul, add) contractions");
    if (algo == LSB_ALGO_TF32X3) {
        char err[256] = "";
        int aux = 0;
        rc = lsb::tf32x3_gemm(M, d->N, d->K, a.A, d->sa_m, d->sa_k, d->B, d->sb_k, d->sb_n, a.C, d->sc_m,
                              d->sc_n, a.c_vec, a.epi, (d->flags & LSB_GEMM_B_UNCHANGED) != 0, d->tile_n, s, &aux,
                              err, sizeof(err));
        if (rc) return fail(rc, "%s", err);
        rc = check_launch("tf32x3_gemm");
        if (rc) return rc;
        g_launches.fetch_add(aux, std::memory_order_relaxed);   // + the split prepasses
        return LSB_OK;
    }

    if (d->K == 0) {
        // empty reduction: every output is the reduce identity, then the epilogue
        return fail(LSB_ERR_UNSUPPORTED, "K == 0 contraction");
    }

    // latency-bound sizes: one launch, K split across each CTA's warps
    // (small_gemm.cuh; C1 256^3)
    if (!d->beta_in_loop && d->beta == 1.0f && d->split_k == 0 && d->K >= 4 &&
        d->K <= 1024 && d->K % 4 == 0 && d->N % 4 == 0 && (double)M * d->N * d->K * d->batch <= (double)(1 << 26) &&
        d->sa_k == 1 && d->sa_m % 4 == 0 && aligned16(a.A) && d->sb_n == 1 && d->sb_k % 4 == 0 &&
        aligned16(d->B) && (d->batch == 1 || (d->sa_b % 4 == 0 && d->sb_b % 4 == 0)) && d->batch <= 65535 &&
        !lsb::knobs().no_small) {
        lsb::prof_mark(0, s);
        const int lrc = lsb::launch_small_gemm(d->combine, d->reduce, a, d->batch, s);
        lsb::prof_mark(1, s);
        if (lrc == 0) return check_launch("small_gemm");
    }

    GemmFn fn = nullptr;
    int bm = 128;
    if (!d->beta_in_loop) {
        // 64-row tiles when the rows would leave half a 128-row tile idle, and
        // for tiny problems (C1 256^3: latency-bound, more and shorter CTAs win;
        // tools/small_gemm_sweep.py: 20.4 -> 14.2 us with 64-row tiles + 16 splits)
        const bool tiny = (double)M * d->N * d->K * d->batch <= (double)(1 << 26);
        bm = (d->tile_m == 64 || (d->tile_m == 0 && (M <= 64 || tiny))) ? 64 : 128;
        // two-level accumulation for long fp32 sums (K split into 256-chunks)
        const bool two = d->reduce == LSB_OP_ADD && d->K > 1024;
        fn = fast_gemm(d->combine, d->reduce, bm, two);
    }
    if (!fn) {
        bm = 128;
        fn = kGemmGeneric[d->combine][d->reduce];
        if (!d->beta_in_loop && d->beta != 1.0f)
            return fail(LSB_ERR_INVALID, "beta outside the loop needs a tuned operator pair");
    }
    const int64_t m_tiles = (M + bm - 1) / bm;
    const int64_t n_tiles = (d->N + lsb::kBN - 1) / lsb::kBN;
    const int64_t tiles = m_tiles * n_tiles * d->batch;

    // (add, max|min) with no epilogue on a grid that would not fill a few
    // waves: stream-K, exact atomic max/min merge (C2)
    {
        const int64_t slots = (int64_t)sm_count() * 2;
        const int64_t t128 = ((M + 127) / 128) * n_tiles;
        if (d->combine == LSB_OP_ADD && (d->reduce == LSB_OP_MAX || d->reduce == LSB_OP_MIN) &&
            !d->beta_in_loop && d->beta == 1.0f && a.epi.n == 0 && d->batch == 1 && d->split_k == 0 &&
            t128 < 3 * slots && d->K >= 64 * lsb::kBK && !lsb::knobs().no_streamk) {
            // row-major 16-B aligned operands with K % 16 == 0 (C2): the
            // cp.async kernel with 16-deep slices (maxplus_fast.cuh)
            const bool fast = d->sa_k == 1 && d->sa_m % 4 == 0 && aligned16(a.A) && d->sb_n == 1 &&
                              d->sb_k % 4 == 0 && aligned16(d->B) && d->N % 4 == 0 && d->K % 16 == 0 &&
                              !lsb::knobs().no_mp_fast;
            // split-K over a cluster with a DSMEM reduction: one launch, no
            // fill, no atomics; cluster size S from the slot-wave cost model
            // (C2: 64 tiles x 4 = 256 CTAs: 78.6 us vs 87 us stream-K)
            // default: stream-K with the in-kernel fixup (every SM the same
            // slice count); LSB_MP_MODE=cluster|streamk selects the others
            const int mode = lsb::knobs().mp_mode;
            if (fast && mode == 0) {
                // one 512-thread CTA per SM, two groups sharing each segment's
                // slices dynamically (C2: 0.078 -> see DESIGN 3.2b)
                const int bk = (lsb::knobs().duo_bk == 32 && d->K % 32) ? 16 : lsb::knobs().duo_bk;
                const int64_t units = t128 * (d->K / bk);
                int ctas = lsb::maxplus_duo_ctas(units, bk);
                if (lsb::knobs().fixup_ctas > 0) ctas = std::max(1, std::min(ctas, lsb::knobs().fixup_ctas));
                if (ctas >= 1) {
                    float4 *part = nullptr;
                    int *flags = nullptr, epoch = 0;
                    rc = fixup_buffers(ctas, &part, &flags, &epoch);
                    if (rc) return rc;
                    lsb::prof_mark(0, s);
                    const int lrc = lsb::launch_maxplus_duo(d->reduce, a, bk, ctas, part, flags, epoch, s);
                    lsb::prof_mark(1, s);
                    if (lrc) return fail(LSB_ERR_CUDA, "maxplus_duo launch (%d CTAs): %s", ctas,
                                         cudaGetErrorString(cudaGetLastError()));
                    return check_launch("maxplus_duo");
                }
            }
            if (fast && mode == 3) {
                const int64_t units = t128 * (d->K / 16);
                int ctas = lsb::maxplus_fixup_ctas(units);
                if (lsb::knobs().fixup_ctas > 0) ctas = std::max(1, std::min(ctas, lsb::knobs().fixup_ctas));
                if (ctas >= 1) {
                    float4 *part = nullptr;
                    int *flags = nullptr, epoch = 0;
                    rc = fixup_buffers(ctas, &part, &flags, &epoch);
                    if (rc) return rc;
                    lsb::prof_mark(0, s);
                    const int lrc = lsb::launch_maxplus_fixup(d->reduce, a, ctas, part, flags, epoch, s);
                    lsb::prof_mark(1, s);
                    if (lrc) return fail(LSB_ERR_CUDA, "maxplus_fixup launch (%d CTAs): %s", ctas,
                                         cudaGetErrorString(cudaGetLastError()));
                    return check_launch("maxplus_fixup");
                }
            }
            if (fast && !lsb::knobs().no_mp_cluster && mode != 2) {
                int best_s = 0;
                double best = 1e30;
                // powers of two only: 3-, 5-, 6-, 7- and 9-CTA clusters measured
                // 20-30 % slower on C2 (tools/dbg/c2ab.sh), 4 the best
                for (int sp = 2; sp <= 8; sp *= 2) {
                    if (d->K / 16 < sp * 4) break;   // >= 4 slices per CTA
                    const double cost = (double)((t128 * sp + slots - 1) / slots) / sp + 0.002 * sp;
                    if (cost < best - 1e-12) { best = cost; best_s = sp; }
                }
                if (lsb::knobs().mp_cluster > 0) best_s = lsb::knobs().mp_cluster;
                if (best_s >= 2) {
                    lsb::prof_mark(0, s);
                    const int lrc = lsb::launch_maxplus_cluster(d->reduce, a, best_s, s);
                    lsb::prof_mark(1, s);
                    if (lrc) return fail(LSB_ERR_CUDA, "maxplus_cluster launch (cluster %d): %s", best_s,
                                         cudaGetErrorString(cudaGetLastError()));
                    return check_launch("maxplus_cluster");
                }
            }
            const int64_t units = t128 * (fast ? d->K / 16 : (d->K + lsb::kBK - 1) / lsb::kBK);
            int ctas = (int)std::min<int64_t>(slots, std::max<int64_t>(1, units / (fast ? 8 : 16)));
            if (lsb::knobs().streamk_ctas > 0) ctas = lsb::knobs().streamk_ctas;
            lsb::prof_mark(0, s);
            if (fast) lsb::launch_streamk_fast(d->reduce, a, ctas, s);
            else lsb::launch_streamk(d->reduce, a, ctas, s);
            lsb::prof_mark(1, s);
            rc = check_launch("semiring_streamk");
            if (rc) return rc;
            g_launches.fetch_add(1, std::memory_order_relaxed);   // + the identity fill
            return LSB_OK;
        }
    }

    int splits = d->split_k;
    if (splits <= 0) {
        splits = 1;
        const int64_t slots = (int64_t)sm_count() * 2;
        const int64_t k_slices = (d->K + lsb::kBK - 1) / lsb::kBK;
        // split K when the tiles alone underfill the 2-CTA/SM slots: pick the
        // split count minimising (waves / splits) + 0.05 * splits, the last term
        // standing for the partial-sum traffic of the fold kernel
        if (tiles < slots && k_slices >= 8) {
            double best = 1e30;
            for (int s = 1; s <= 16 && s <= k_slices / 2; s++) {
                const int64_t waves = (tiles * s + slots - 1) / slots;
                const double cost = (double)waves / s + 0.05 * s;
                if (cost < best - 1e-9) { best = cost; splits = s; }
            }
            // tiny problems are latency-bound: as many splits as fit one wave
            // (>= 2 k-slices each), the fold is cheap at this size
            if ((double)M * d->N * d->K * d->batch <= (double)(1 << 26))
                splits = (int)std::max<int64_t>(1, std::min<int64_t>({16, k_slices / 2, slots / std::max<int64_t>(1, tiles)}));
        }
    }
    int64_t kps = (d->K + splits - 1) / splits;
    kps = ((kps + lsb::kBK - 1) / lsb::kBK) * lsb::kBK;
    splits = (int)((d->K + kps - 1) / kps);
    a.k_per_split = kps;
    a.splits = splits;
    if (m_tiles * splits > 65535 || d->batch > 65535 || n_tiles > 2147483647)
        return fail(LSB_ERR_UNSUPPORTED, "grid too large");

    if (splits > 1) {
        rc = workspace(sizeof(float) * (size_t)splits * d->batch * M * d->N, &a.ws);
        if (rc) return rc;
    }
    dim3 grid((unsigned)n_tiles, (unsigned)(m_tiles * splits), (unsigned)d->batch);
    lsb::prof_mark(0, s);
    fn(a, grid, s);
    lsb::prof_mark(1, s);
    rc = check_launch("semiring_gemm");
    if (rc) return rc;
    if (splits > 1) {
        kSplit[d->reduce](a, d->batch, s);
        rc = check_launch("splitk_epilogue");
        if (rc) return rc;
    }
    return LSB_OK;
}

static int g_last_conv_kind = 0, g_last_conv_nt = 0;   // lsb_last_conv_kernel (diagnostics)

int lsb_last_conv_kernel(int *kind, int *nt) {
    if (kind) *kind = g_last_conv_kind;
    if (nt) *nt = g_last_conv_nt;
    return LSB_OK;
}

int lsb_conv2d_nchw(const lsb_conv_desc *d, void *stream) {
    if (!d) return fail(LSB_ERR_INVALID, "null desc");
    if (!d->x || !d->w || !d->o) return fail(LSB_ERR_INVALID, "null operand");
    if (d->N < 1 || d->C < 1 || d->CO < 1 || d->R < 1 || d->S < 1 || d->HO < 1 || d->WO < 1 ||
        d->stride_h < 1 || d->stride_w < 1 || d->dil_h < 1 || d->dil_w < 1)
        return fail(LSB_ERR_INVALID, "bad conv extents");
    if (!(d->combine == LSB_OP_MUL && d->reduce == LSB_OP_ADD) || d->beta_in_loop)
        return fail(LSB_ERR_UNSUPPORTED, "conv kernel covers (mul, add) only");
    int rc = check_epi(d->n_epi, d->epi);
    if (rc) return rc;
    const int64_t K = d->C * d->R * d->S;
    if (K > lsb::kConvTableMax) return fail(LSB_ERR_UNSUPPORTED, "conv K=%lld too large", (long long)K);
    if (d->N > 65535) return fail(LSB_ERR_UNSUPPORTED, "too many images");
    if ((rc = check_device())) return rc;

    lsb::ConvArgs a;
    memset(&a, 0, sizeof(a));
    a.M = d->CO; a.N = d->HO * d->WO; a.K = K;
    a.C = d->C; a.H = d->H; a.W = d->W; a.R = d->R; a.S = d->S; a.HO = d->HO; a.WO = d->WO;
    a.stride_h = d->stride_h; a.stride_w = d->stride_w; a.pad_h = d->pad_h; a.pad_w = d->pad_w;
    a.dil_h = d->dil_h; a.dil_w = d->dil_w; a.fill = d->fill;
    a.x = d->x; a.sx0 = d->sx[0]; a.sx1 = d->sx[1]; a.sx2 = d->sx[2]; a.sx3 = d->sx[3];
    a.w = d->w; a.sw0 = d->sw[0]; a.sw1 = d->sw[1]; a.sw2 = d->sw[2]; a.sw3 = d->sw[3];
    a.o = d->o; a.so0 = d->so[0]; a.so1 = d->so[1]; a.so2 = d->so[2]; a.so3 = d->so[3];
    a.beta = d->beta;
    a.epi = pack_epi(d->n_epi, d->epi);
    const bool wcontig = d->sw[3] == 1 && d->sw[2] == d->S && d->sw[1] == d->R * d->S;
    a.a_mode = (wcontig && aligned16(d->w) && d->sw[0] % 4 == 0 && K % 4 == 0) ? lsb::LD_VEC_K : lsb::LD_GENERIC;

    // tensor cores (split TF32) for real work: the planar kernel
    // (conv_planar.cuh: stride 1, zero fill, TMA-able X strides; raw X boxes
    // converted in shared memory, no X copy), else the NHWC-copy kernel
    // (tf32x3_conv_nhwc.cuh: zero fill, strides <= 8); SIMT otherwise
    // (nonzero fill, tiny convs).  LSB_GEMM_ALGO=simt|tf32x3|tf32x3_nhwc|tf32x3_planar.
    // Measured on C3 (tools/c3_probe.py, back-to-back launches):
    // planar 21.6 us per call (filter prepass + conv), NHWC-copy 23.1 us.
    const bool big = 2.0 * a.M * a.N * d->N * K >= (double)(1ll << 28) && a.M >= 16;
    const bool planar_ok = lsb::conv_planar_ok(a, d->N), nhwc_ok = lsb::tf32x3_conv_nhwc_ok(a, d->N);
    int tc_mode = !big ? 0 : planar_ok ? 5 : nhwc_ok ? 4 : 0;
    switch (lsb::knobs().gemm_algo) {
    case LSB_ALGO_SIMT: tc_mode = 0; break;
    case LSB_ALGO_TF32X3: tc_mode = planar_ok ? 5 : nhwc_ok ? 4 : 0; break;
    case lsb::kAlgoTf32x3Nhwc: tc_mode = nhwc_ok ? 4 : planar_ok ? 5 : 0; break;
    case lsb::kAlgoTf32x3Planar: tc_mode = planar_ok ? 5 : nhwc_ok ? 4 : 0; break;
    default: break;
    }
    g_last_conv_kind = tc_mode == 5 ? 2 : tc_mode == 4 ? 1 : 0;
    g_last_conv_nt = tc_mode == 5 ? lsb::conv_planar_nt(a, d->N) : 0;
    if (tc_mode) {
        char err[256] = "";
        int aux = 0;
        cudaStream_t st = (cudaStream_t)stream;
        rc = tc_mode == 5 ? lsb::conv_planar(a, d->N, st, &aux, err, sizeof(err))
                          : lsb::tf32x3_conv_nhwc(a, d->N, st, &aux, err, sizeof(err));
        if (rc) return fail(rc, "%s", err);
        rc = check_launch(tc_mode == 5 ? "conv_planar" : "tf32x3_conv_nhwc");
        if (rc) return rc;
        g_launches.fetch_add(aux, std::memory_order_relaxed);
        return LSB_OK;
    }
    const int bm = 64;
    const int64_t m_tiles = (a.M + bm - 1) / bm;
    const int64_t tiles = ((a.N + lsb::kBN - 1) / lsb::kBN) * m_tiles * d->N;
    // split the (c, r, s) taps when the tiles underfill the 2-CTA/SM slots
    // (C3: 200 tiles for 296 slots); same wave cost model as the GEMM split-K
    int splits = 1;
    {
        const int64_t slots = (int64_t)sm_count() * 2;
        const int64_t k_slices = (K + lsb::kBK - 1) / lsb::kBK;
        if (tiles < 2 * slots && k_slices >= 16 && !lsb::knobs().no_conv_split) {
            // cost = the busiest SM's CTA count x work per CTA (+ fold traffic)
            const int64_t sms = sm_count();
            double best = 1e30;
            for (int s = 1; s <= 8 && s <= k_slices / 8; s++) {
                const int64_t per_sm = (tiles * s + sms - 1) / sms;
                const double cost = (double)per_sm / s + 0.05 * (s > 1 ? s : 0);
                if (cost < best - 1e-9) { best = cost; splits = s; }
            }
        }
        if (lsb::knobs().conv_splits > 0) splits = lsb::knobs().conv_splits;
    }
    int64_t kps = (K + splits - 1) / splits;
    kps = (kps + lsb::kBK - 1) / lsb::kBK * lsb::kBK;
    splits = (int)((K + kps - 1) / kps);
    a.k_per_split = kps;
    a.splits = splits;
    if (splits > 1) {
        rc = workspace(sizeof(float) * (size_t)splits * d->N * a.M * a.N, &a.ws);
        if (rc) return rc;
    }
    dim3 grid((unsigned)((a.N + lsb::kBN - 1) / lsb::kBN), (unsigned)(m_tiles * splits), (unsigned)d->N);
    size_t dyn = (size_t)K * (sizeof(int64_t) + sizeof(int2));
    lsb::prof_mark(0, (cudaStream_t)stream);
    lsb::launch_conv_fast(a, grid, dyn, (cudaStream_t)stream);
    lsb::prof_mark(1, (cudaStream_t)stream);
    rc = check_launch("conv_igemm");
    if (rc || splits == 1) return rc;
    lsb::launch_conv_fold(a, d->N, (cudaStream_t)stream);
    return check_launch("conv_splitk_fold");
}

static int g_last_nest_kind = 0;   // lsb_last_nest_kernel (diagnostics)

int lsb_affine_nest(const lsb_nest_desc *d, void *stream) {
    if (!d) return fail(LSB_ERR_INVALID, "null desc");
    if (d->n_out < 0 || d->n_red < 0 || d->n_out + d->n_red > LSB_MAX_NEST_DIMS)
        return fail(LSB_ERR_INVALID, "bad dim counts %d + %d", d->n_out, d->n_red);
    if (d->n_operands < 1 || d->n_operands > LSB_MAX_NEST_OPERANDS)
        return fail(LSB_ERR_INVALID, "bad operand count %d", d->n_operands);
    if (!valid_op(d->combine) || !valid_op(d->reduce))
        return fail(LSB_ERR_INVALID, "bad operator pair");
    if (!d->out) return fail(LSB_ERR_INVALID, "null output");
    int rc = check_epi(d->n_epi, d->epi);
    if (rc) return rc;
    lsb::NestArgs a;
    memset(&a, 0, sizeof(a));
    a.n_out = d->n_out; a.n_red = d->n_red; a.n_ops = d->n_operands;
    a.n_points = 1;
    for (int i = 0; i < d->n_out + d->n_red; i++) {
        if (d->extent[i] < 1) return fail(LSB_ERR_INVALID, "extent[%d] = %lld", i, (long long)d->extent[i]);
        a.extent[i] = d->extent[i];
        if (i < d->n_out) a.n_points *= d->extent[i];
    }
    for (int o = 0; o < d->n_operands; o++) {
        if (!d->operand[o].ptr) return fail(LSB_ERR_INVALID, "operand %d null", o);
        if (d->operand[o].n_guards < 0 || d->operand[o].n_guards > LSB_MAX_GUARDS)
            return fail(LSB_ERR_INVALID, "operand %d guards", o);
        a.op[o] = d->operand[o];
    }
    a.out = d->out; a.out_addr = d->out_addr; a.beta = d->beta;
    a.epi = pack_epi(d->n_epi, d->epi);
    if ((rc = check_device())) return rc;
    g_last_nest_kind = lsb::knobs().no_nest_fast ? 0 : lsb::launch_nest_fast(*d, a.epi, (cudaStream_t)stream);
    if (g_last_nest_kind == 0) kNest[d->combine][d->reduce](a, (cudaStream_t)stream);
    return check_launch("affine_nest");
}

int lsb_last_nest_kernel(int *kind) {
    if (kind) *kind = g_last_nest_kind;
    return LSB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- NCCL row gather
// (resolved at run time so liblsb.so has no link-time NCCL dependency; with
// torch imported first, dlopen returns the libnccl.so.2 torch already mapped)
namespace {
struct NcclApi {
    bool tried = false;
    void *h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

int nccl_load() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl.tried) {
        g_nccl.tried = true;
        g_nccl.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (g_nccl.h) {
            g_nccl.get_unique_id = (decltype(g_nccl.get_unique_id))dlsym(g_nccl.h, "ncclGetUniqueId");
            g_nccl.comm_init_rank = (decltype(g_nccl.comm_init_rank))dlsym(g_nccl.h, "ncclCommInitRank");
            g_nccl.comm_destroy = (decltype(g_nccl.comm_destroy))dlsym(g_nccl.h, "ncclCommDestroy");
            g_nccl.all_gather = (decltype(g_nccl.all_gather))dlsym(g_nccl.h, "ncclAllGather");
            g_nccl.error_string = (decltype(g_nccl.error_string))dlsym(g_nccl.h, "ncclGetErrorString");
        }
    }
    if (!g_nccl.get_unique_id || !g_nccl.comm_init_rank || !g_nccl.comm_destroy || !g_nccl.all_gather)
        return fail(LSB_ERR_UNSUPPORTED, "libnccl.so.2 not loadable: %s", g_nccl.h ? "missing symbols" : dlerror());
    return LSB_OK;
}

int nccl_fail(ncclResult_t r, const char *what) {
    return fail(LSB_ERR_CUDA, "%s: %s", what, g_nccl.error_string ? g_nccl.error_string(r) : "NCCL error");
}
}  // namespace

extern "C" {

int lsb_nccl_unique_id(unsigned char *id) {
    if (!id) return fail(LSB_ERR_INVALID, "null id");
    static_assert(sizeof(ncclUniqueId) == LSB_NCCL_ID_BYTES, "ncclUniqueId size");
    int rc = nccl_load();
    if (rc) return rc;
    ncclUniqueId u;
    ncclResult_t r = g_nccl.get_unique_id(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id, &u, sizeof(u));
    return LSB_OK;
}

int lsb_nccl_init(int rank, int nranks, const unsigned char *id, void **comm) {
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(LSB_ERR_INVALID, "bad communicator arguments (rank %d of %d)", rank, nranks);
    int rc = nccl_load();
    if (rc) return rc;
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    ncclComm_t c = nullptr;
    ncclResult_t r = g_nccl.comm_init_rank(&c, nranks, u, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return LSB_OK;
}

int lsb_nccl_destroy(void *comm) {
    if (!comm) return LSB_OK;
    int rc = nccl_load();
    if (rc) return rc;
    ncclResult_t r = g_nccl.comm_destroy((ncclComm_t)comm);
    return r == ncclSuccess ? LSB_OK : nccl_fail(r, "ncclCommDestroy");
}

int lsb_allgather_rows(void *comm, const float *send, float *recv, int64_t count, void *stream) {
    if (!comm || count < 0 || (count > 0 && (!send || !recv))) return fail(LSB_ERR_INVALID, "bad gather arguments");
    int rc = nccl_load();
    if (rc) return rc;
    ncclResult_t r = g_nccl.all_gather(send, recv, (size_t)count, ncclFloat32, (ncclComm_t)comm, (cudaStream_t)stream);
    return r == ncclSuccess ? LSB_OK : nccl_fail(r, "ncclAllGather");
}

}  // extern "C"
