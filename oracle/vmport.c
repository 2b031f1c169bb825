/*
 * vmport.c -- TEST/BASELINE INFRASTRUCTURE ONLY (never linked into the product).
 *
 * A C restatement of the arithmetic the reference's kernel VM performs for
 * the hot-path contractions, used (1) as the CPU baseline timed beside the
 * GPU numbers (bench.py cpu_baseline, kind "port", and `bench.py --impl
 * reference`, because the numba VM itself cannot travel to the GPU box) and
 * (2) as a bit-exact cross-check of the reference VM on the golden fixtures.
 *
 * What is restated (reference pkg/src/loopsmith/...):
 *   vm.py:112-129   vop.{add,mul,max,min}: one f32 op per lane
 *   vm.py:130-136   vfma: dst + s1*s2 evaluated UNFUSED in f32 (the product
 *                   is rounded before the add) -- built with -ffp-contract=off
 *   vm.py:214-228   post relu = max(x, 0); sigmoid evaluated in f64 then
 *                   rounded (x >= 0: 1/(1+exp(-x)), else e/(1+e))
 *   backend.py:938-968  register-blocked region: accumulators start at the
 *                   reduce identity (ir.py:182), the reduction loop runs in
 *                   order, one store at region exit.
 * For the SURVEY §8(d) schedules the reduction order per output point is the
 * plain sequential order of the flattened reduction index, so this port is
 * bit-identical to the VM on those schedules (pinned in tests/test_oracle.py).
 *
 * Parallelism: output rows are split across pthreads; each output point is
 * still reduced sequentially, so results do not depend on the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OP_ADD = 0, OP_MUL = 1, OP_MAX = 2, OP_MIN = 3 };
enum { EW_ID = 0, EW_RELU = 1, EW_SIGMOID = 2 };

static inline float vm_op(int op, float x, float y) {
    switch (op) {
    case OP_ADD: return x + y;
    case OP_MUL: return x * y;
    case OP_MAX: return x > y ? x : y;   /* numba max(): first arg on ties */
    default:     return x < y ? x : y;
    }
}

static inline float identity_of(int op) {
    switch (op) {
    case OP_ADD: return 0.0f;
    case OP_MUL: return 1.0f;
    case OP_MAX: return -INFINITY;
    default:     return INFINITY;
    }
}

static inline float vm_post(int ew, float x) {
    if (ew == EW_RELU) return x > 0.0f ? x : 0.0f;
    if (ew == EW_SIGMOID) {
        double d = (double)x;
        if (d >= 0.0) return (float)(1.0 / (1.0 + exp(-d)));
        double e = exp(d);
        return (float)(e / (1.0 + e));
    }
    return x;
}

/* ------------------------------------------------------------------ GEMM */

typedef struct {
    int64_t M, N, K;
    const float *A; int64_t sam, sak;
    const float *B; int64_t sbk, sbn;
    float *C; int64_t scm, scn;
    int comb, red;
    const float *bias; int64_t sbias;   /* optional y = post(h + bias[n]) */
    int post;
    int64_t r0, r1;
} gemm_job;

#define BM 4
#define BN 64

static void gemm_block(const gemm_job *j, int64_t i0, int64_t ni, int64_t j0, int64_t nj) {
    float acc[BM][BN];
    float id = identity_of(j->red);
    for (int i = 0; i < BM; i++)
        for (int q = 0; q < BN; q++) acc[i][q] = id;
    for (int64_t k = 0; k < j->K; k++) {
        const float *brow = j->B + k * j->sbk + j0 * j->sbn;
        for (int i = 0; i < ni; i++) {
            float a = j->A[(i0 + i) * j->sam + k * j->sak];
            float *ac = acc[i];
            if (j->comb == OP_MUL && j->red == OP_ADD) {
                if (j->sbn == 1) {
                    for (int q = 0; q < nj; q++) { float p = a * brow[q]; ac[q] = ac[q] + p; }
                } else {
                    for (int q = 0; q < nj; q++) { float p = a * brow[q * j->sbn]; ac[q] = ac[q] + p; }
                }
            } else if (j->comb == OP_ADD && j->red == OP_MAX) {
                for (int q = 0; q < nj; q++) {
                    float s = a + brow[q * j->sbn];
                    ac[q] = ac[q] > s ? ac[q] : s;
                }
            } else {
                for (int q = 0; q < nj; q++)
                    ac[q] = vm_op(j->red, ac[q], vm_op(j->comb, a, brow[q * j->sbn]));
            }
        }
    }
    for (int i = 0; i < ni; i++)
        for (int q = 0; q < nj; q++) {
            float h = acc[i][q];
            if (j->bias) h = h + j->bias[(j0 + q) * j->sbias];
            j->C[(i0 + i) * j->scm + (j0 + q) * j->scn] = vm_post(j->post, h);
        }
}

static void *gemm_worker(void *arg) {
    const gemm_job *j = (const gemm_job *)arg;
    for (int64_t i0 = j->r0; i0 < j->r1; i0 += BM) {
        int64_t ni = j->r1 - i0 < BM ? j->r1 - i0 : BM;
        for (int64_t j0 = 0; j0 < j->N; j0 += BN) {
            int64_t nj = j->N - j0 < BN ? j->N - j0 : BN;
            gemm_block(j, i0, ni, j0, nj);
        }
    }
    return NULL;
}

/* C[r0:r1, :] = post(reduce_k comb(A[m,k], B[k,n]) (+ bias[n]))  */
int vmp_gemm(int64_t M, int64_t N, int64_t K,
             const float *A, int64_t sam, int64_t sak,
             const float *B, int64_t sbk, int64_t sbn,
             float *C, int64_t scm, int64_t scn,
             int comb, int red, const float *bias, int64_t sbias, int post,
             int64_t r0, int64_t r1, int threads) {
    if (r1 > M) r1 = M;
    if (r0 < 0 || r0 >= r1) return 0;
    if (threads < 1) threads = 1;
    int64_t rows = r1 - r0;
    int64_t blocks = (rows + BM - 1) / BM;
    if (threads > blocks) threads = (int)blocks;
    gemm_job *jobs = (gemm_job *)calloc((size_t)threads, sizeof(gemm_job));
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    int64_t per = (blocks + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        gemm_job *j = &jobs[t];
        *j = (gemm_job){M, N, K, A, sam, sak, B, sbk, sbn, C, scm, scn, comb, red,
                        bias, sbias, post, 0, 0};
        j->r0 = r0 + (int64_t)t * per * BM;
        j->r1 = j->r0 + per * BM;
        if (j->r1 > r1) j->r1 = r1;
        if (j->r0 > r1) j->r0 = r1;
        if (t > 0) pthread_create(&tid[t], NULL, gemm_worker, j);
    }
    gemm_worker(&jobs[0]);
    for (int t = 1; t < threads; t++) pthread_join(tid[t], NULL);
    free(jobs);
    free(tid);
    return 0;
}

/* ------------------------------------------------------------------ conv */

typedef struct {
    int64_t N, C, H, W, CO, R, S, HO, WO, stride, pad;
    const float *x, *w; float *o;
    int64_t n0, n1;   /* (n, co) pairs [n0, n1) */
} conv_job;

static void *conv_worker(void *arg) {
    const conv_job *j = (const conv_job *)arg;
    float *acc = (float *)malloc((size_t)j->WO * sizeof(float));
    for (int64_t p = j->n0; p < j->n1; p++) {
        int64_t n = p / j->CO, co = p % j->CO;
        for (int64_t h = 0; h < j->HO; h++) {
            for (int64_t q = 0; q < j->WO; q++) acc[q] = 0.0f;
            for (int64_t ci = 0; ci < j->C; ci++)
                for (int64_t r = 0; r < j->R; r++) {
                    int64_t hi = h * j->stride + r - j->pad;
                    const float *xrow = j->x + ((n * j->C + ci) * j->H + hi) * j->W;
                    for (int64_t s = 0; s < j->S; s++) {
                        float wv = j->w[((co * j->C + ci) * j->R + r) * j->S + s];
                        for (int64_t q = 0; q < j->WO; q++) {
                            int64_t wi = q * j->stride + s - j->pad;
                            float xv = (hi >= 0 && hi < j->H && wi >= 0 && wi < j->W) ? xrow[wi] : 0.0f;
                            float prod = xv * wv;
                            acc[q] = acc[q] + prod;
                        }
                    }
                }
            float *orow = j->o + ((n * j->CO + co) * j->HO + h) * j->WO;
            memcpy(orow, acc, (size_t)j->WO * sizeof(float));
        }
    }
    free(acc);
    return NULL;
}

/* o[n,co,h,w] = sum_{ci,r,s} x[n,ci,h*st+r-pad, w*st+s-pad] * w[co,ci,r,s]
 * over images [img0, img1). */
int vmp_conv2d(int64_t N, int64_t C, int64_t H, int64_t W, int64_t CO, int64_t R, int64_t S,
               int64_t stride, int64_t pad, const float *x, const float *w, float *o,
               int64_t img0, int64_t img1, int threads) {
    int64_t HO = (H + 2 * pad - R) / stride + 1, WO = (W + 2 * pad - S) / stride + 1;
    if (img1 > N) img1 = N;
    int64_t pairs = (img1 - img0) * CO;
    if (pairs <= 0) return 0;
    if (threads < 1) threads = 1;
    if (threads > pairs) threads = (int)pairs;
    conv_job *jobs = (conv_job *)calloc((size_t)threads, sizeof(conv_job));
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    int64_t per = (pairs + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        conv_job *j = &jobs[t];
        *j = (conv_job){N, C, H, W, CO, R, S, HO, WO, stride, pad, x, w, o, 0, 0};
        j->n0 = img0 * CO + (int64_t)t * per;
        j->n1 = j->n0 + per;
        if (j->n1 > img1 * CO) j->n1 = img1 * CO;
        if (j->n0 > j->n1) j->n0 = j->n1;
        if (t > 0) pthread_create(&tid[t], NULL, conv_worker, j);
    }
    conv_worker(&jobs[0]);
    for (int t = 1; t < threads; t++) pthread_join(tid[t], NULL);
    free(jobs);
    free(tid);
    return 0;
}
