/*
 * lsb.h -- C ABI of the B200 loop-nest backend (liblsb.so).
 *
 * This is the drop-in boundary under the reference's backend surface.  The
 * reference (loopsmith) compiles a LoopTree into a VM program and interprets
 * it on the CPU:
 *
 *     compile_tree(tree, target)   reference pkg/src/loopsmith/backend.py:1427-1454
 *     execute(kernel, buffers)     reference pkg/src/loopsmith/backend.py:121-161
 *       -> vm.run / vm._run        reference pkg/src/loopsmith/vm.py:20-257
 *
 * The B200 backend keeps that Python surface (paper_2205_00618_b200.backend)
 * and replaces encode_program + vm.run with launches of hand-written sm_100a
 * kernels through the entry points below.  Each launch entry point takes one
 * plain-C descriptor (pointers, sizes, element strides, operator codes) and a
 * cudaStream_t passed as void*; nothing here uses torch or C++ types.
 *
 * Conventions
 *   - every function returns int: LSB_OK (0) on success, a negative
 *     LSB_ERR_* on failure; lsb_last_error() copies a message for the last
 *     failure on the calling thread.
 *   - all data is f32; strides are in ELEMENTS (may be 0 for broadcast).
 *   - device buffers are owned by the caller (lsb_device_alloc or any CUDA
 *     allocation, e.g. torch tensors); launches are asynchronous on `stream`.
 *   - operator codes equal the reference's program.KIND_CODE / EW_CODE
 *     (program.py:182-183) so plans carry them verbatim.
 *   - thread-compatible, not thread-safe per stream (like the reference's
 *     CompiledKernel).
 *   - library workspaces (split-K partials, the tensor-core split copies, the
 *     max-plus fixup slots and flags) are per process and stream-ordered:
 *     contractions enqueued on two different streams at once must not both
 *     need them (run them on one stream, or synchronise in between).
 */
#ifndef LSB_H_
#define LSB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSB_ABI_VERSION 3

/* reduce / combine operators: program.py:182 KIND_CODE */
enum { LSB_OP_ADD = 0, LSB_OP_MUL = 1, LSB_OP_MAX = 2, LSB_OP_MIN = 3 };
/* elementwise pre/post: program.py:183 EW_CODE (ir.py:179 ELEMENTWISE_OPS) */
enum { LSB_EW_IDENTITY = 0, LSB_EW_RELU = 1, LSB_EW_SIGMOID = 2 };
/* GEMM algorithm selector */
/* LSB_ALGO_TF32X3 names the fp32-accurate tensor-core path (the name is kept
 * for ABI stability): GEMMs split power-of-two-scaled operands into fp16 hi/lo
 * parts and run three fp16 tcgen05 MMAs per product (hi.hi, hi.lo, lo.hi),
 * convs a tf32 + bf16-correction mix; within 1e-5 + 1e-4|ref| per element. */
enum { LSB_ALGO_AUTO = 0, LSB_ALGO_SIMT = 1, LSB_ALGO_TF32X3 = 2 };

enum {
    LSB_OK = 0,
    LSB_ERR_INVALID = -1,      /* bad descriptor / argument */
    LSB_ERR_CUDA = -2,         /* CUDA runtime error */
    LSB_ERR_UNSUPPORTED = -3,  /* shape / operator combination not covered */
    LSB_ERR_NOMEM = -4
};

#define LSB_MAX_EPI 4
#define LSB_MAX_NEST_DIMS 8
#define LSB_MAX_NEST_OPERANDS 4
#define LSB_MAX_GUARDS 4

/*
 * One fused elementwise stage of a contraction epilogue, the per-output-point
 * part of the reference Arith semantics (ir.py:194-222, feedback.py:144-170):
 *
 *     t = operand ? combine(x, operand[idx]) : x
 *     t = beta * t                              (skipped when beta == 1)
 *     t = alpha != 0 ? reduce(alpha * pre(c_in[idx]), t) : t
 *     x = post(t)
 *
 * Stage 0 is the contraction node itself (operand NULL; its beta is the
 * post-reduction scale when the plan moved beta out of the loop); later
 * stages are the elementwise Arith nodes that follow it (bias add, ReLU, ...).
 * idx = Σ s[d] * coord[d] over the kernel's output coordinates:
 *   GEMM (batch, m, n, -), conv (n, co, h, w).
 */
typedef struct {
    int32_t combine;           /* LSB_OP_* with operand, or -1 for none */
    int32_t reduce;            /* op folding alpha*pre(c_in) into x      */
    int32_t pre, post;         /* LSB_EW_*                                */
    float beta, alpha;
    const float *operand; int64_t so[4];
    const float *c_in;    int64_t sc[4];
} lsb_epi_stage;

/*
 * Semiring contraction  C[b,m,n] = epi( reduce_k  combine(A[b,m,k], B[b,k,n]) )
 * Replaces the register-blocked region of backend.py:593-971 executed by
 * vm.py:112-161 (vop / vfma / vreduce) for 2-operand contractions.
 */
typedef struct {
    int64_t M, N, K, batch;
    const float *A; int64_t sa_b, sa_m, sa_k;
    const float *B; int64_t sb_b, sb_k, sb_n;
    float *C;       int64_t sc_b, sc_m, sc_n;
    int32_t combine, reduce;
    float beta;                /* scale of every combine term             */
    int32_t beta_in_loop;      /* 1: apply beta per term (exact);
                                  0: caller moved it to epi[0]             */
    int32_t n_epi;
    lsb_epi_stage epi[LSB_MAX_EPI];
    int32_t algo;              /* LSB_ALGO_*                               */
    int32_t split_k;           /* 0 = auto; > 0: SIMT split-K slices (the
                                  schedule's outermost reduction loop)    */
    int32_t tile_m, tile_n;    /* 0 = auto; tile_m 64: 64-row SIMT tiles;
                                  tile_n 128 / 256: 3xTF32 tile width (the
                                  schedule's register block, schedule.py) */
    int64_t m_begin, m_end;    /* compute output rows [m_begin, m_end); m_end <= 0 -> M
                                  (row sharding across GPUs) */
    int32_t flags;             /* LSB_GEMM_* bits                          */
    int32_t gen;               /* PREP/PRESPLIT sequences: the caller's nonzero
                                  generation stamp for non-finite row flags  */
    int64_t n_begin, n_end;    /* PRESPLIT: output columns [n_begin, n_end)  */
} lsb_gemm_desc;

/* lsb_gemm_desc.flags: B (pointer, extents, strides and contents) is the same
 * as in the previous lsb_semiring_gemm call on this device -- the 3xTF32 path
 * then reuses its hi/lo split of B (row-block streaming of one contraction) */
#define LSB_GEMM_B_UNCHANGED 1
/* Blocked 3xTF32 sequences (execute() overlapping PCIe with compute): split
 * rows [m_begin, m_end) of A / columns [n_begin, n_end) of B into the
 * library's full-size split workspace without computing, then compute an
 * output rectangle from what is already split.  Rectangle corners must be
 * multiples of the tile (128 rows, 256 columns).  tf32x3 (mul, add) only.
 * A sequence owns the device's split workspace from its first PREP to its
 * last PRESPLIT: other tf32x3 calls on the device in between invalidate it. */
#define LSB_GEMM_PREP_A 2
#define LSB_GEMM_PREP_B 4
#define LSB_GEMM_PRESPLIT 8
/* with PRESPLIT: the output region is the L [0, m_end) x [0, n_end) minus
 * [0, m_begin) x [0, n_begin) -- what becomes computable when the split
 * pieces grow from (m_begin, n_begin) to (m_end, n_end); one launch */
#define LSB_GEMM_GROW 16

/*
 * Direct 2-D convolution over NCHW-indexed tensors (any element strides),
 * implicit GEMM: M = CO, N = pixels, K = C*R*S.  Out-of-range taps read
 * `fill` (a guarded View's oob, ir.py:238-245; 0 for zero padding).
 * Replaces the guarded-load + FMA loops of backend.py:357-395 / vm.py:86-188.
 */
typedef struct {
    int64_t N, C, H, W;        /* input extent  */
    int64_t CO, R, S;          /* filter extent */
    int64_t HO, WO;            /* output extent */
    int64_t stride_h, stride_w, pad_h, pad_w, dil_h, dil_w;
    float fill;
    const float *x; int64_t sx[4];   /* n, c, h, w  */
    const float *w; int64_t sw[4];   /* co, c, r, s */
    float *o;       int64_t so[4];   /* n, co, h, w */
    int32_t combine, reduce;
    float beta; int32_t beta_in_loop;
    int32_t n_epi;
    lsb_epi_stage epi[LSB_MAX_EPI];
} lsb_conv_desc;

/*
 * General affine loop nest (one Arith node): for every output point,
 *   acc = identity(reduce); for every reduction point:
 *       acc = reduce(acc, beta * combine_i operand_i[addr_i])
 * with addr_i = base_i + Σ coeff_i[d] * iter[d], guarded coordinates reading
 * `fill_i`, then the epilogue stages (coords = the first 4 output dims).
 * Covers every graph the frontend can build (views, windows, concat,
 * transposes, broadcasts, pooling) -- the coverage path for trees the tuned
 * kernels do not match.
 */
typedef struct {
    int64_t base;
    int64_t coeff[LSB_MAX_NEST_DIMS];
} lsb_affine;

typedef struct {
    const float *ptr;
    lsb_affine addr;
    int32_t n_guards;
    lsb_affine guard[LSB_MAX_GUARDS];   /* value must lie in [0, guard_size) */
    int64_t guard_size[LSB_MAX_GUARDS];
    float fill;
} lsb_nest_operand;

typedef struct {
    int32_t n_out, n_red;                 /* dims: out first, then reduction */
    int64_t extent[LSB_MAX_NEST_DIMS];
    int32_t n_operands;
    lsb_nest_operand operand[LSB_MAX_NEST_OPERANDS];
    float *out; lsb_affine out_addr;
    int32_t combine, reduce;
    float beta;
    int32_t n_epi;
    lsb_epi_stage epi[LSB_MAX_EPI];       /* so/sc index the first 4 out dims */
} lsb_nest_desc;

/* ---- lifecycle / errors --------------------------------------------------- */
int lsb_abi_version(void);
/* Binds the process to `device` (cudaSetDevice) and checks it is sm_100.
 * One device per process: a second lsb_init with another device fails with
 * LSB_ERR_UNSUPPORTED, and the compute calls fail unless the caller's
 * current device is the bound one (workspaces and kernel attributes are
 * process-wide; the multi-GPU path runs one process per GPU). */
int lsb_init(int device);
int lsb_last_error(char *buf, size_t len);
/* Re-read the LSB_* environment knobs.  The library reads
 * them once, at first use; nothing on the launch path calls getenv. */
int lsb_reload_env(void);
int lsb_device_info(int device, int *sm_count, int *cc_major, int *cc_minor,
                    int *clock_khz);

/* ---- memory (caller-owned; thin wrappers so the ABI needs no CUDA headers) */
int lsb_device_alloc(void **ptr, size_t bytes);
int lsb_device_free(void *ptr);
int lsb_host_alloc(void **ptr, size_t bytes);       /* pinned */
int lsb_host_free(void *ptr);
int lsb_memcpy_h2d(void *dst, const void *src, size_t bytes, void *stream);
int lsb_memcpy_d2h(void *dst, const void *src, size_t bytes, void *stream);
int lsb_memcpy_d2d(void *dst, const void *src, size_t bytes, void *stream);
/* pitched host->device copy of `height` rows of `width` bytes (a column
 * block of a row-major matrix): lets execute() start on B's first column
 * block while the rest is still crossing PCIe */
int lsb_memcpy_h2d_2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height,
                      void *stream);
int lsb_memcpy_d2h_2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height,
                      void *stream);
int lsb_stream_sync(void *stream);
/* streams / events for overlapping copies with kernels (row-block streaming) */
int lsb_stream_create(void **stream);
int lsb_stream_destroy(void *stream);
int lsb_event_create(void **event);
int lsb_event_destroy(void *event);
int lsb_event_record(void *event, void *stream);
int lsb_stream_wait_event(void *stream, void *event);

/* Copies between ordinary (pageable) host memory and the device through
 * page-locked staging slots filled and drained by a pool of host threads
 * (csrc/lsb_stage.cu): the DMAs run at pinned speed and overlap the host
 * copies.  h2d returns once `src` has been read (the DMAs are enqueued on
 * `stream`); d2h enqueues the DMAs and returns -- `dst` is complete after
 * lsb_stage_wait().  One calling thread at a time. */
int lsb_stage_h2d_2d(void *dst, size_t dpitch, const void *src, size_t spitch,
                     size_t width, size_t height, void *stream);
int lsb_stage_d2h_2d(void *dst, size_t dpitch, const void *src, size_t spitch,
                     size_t width, size_t height, void *stream);
int lsb_stage_wait(void);
/* *pinned = 1 when `p` is page-locked (cudaHostAlloc'd or registered). */
int lsb_host_is_pinned(const void *p, int *pinned);
/* Geometry of the last tensor-core GEMM launch on this process: tile width (128 /
 * 256), grid size, persistent units (0 = one tile per CTA), 2-CTA clusters.
 * Diagnostics for tests and tools. */
int lsb_last_gemm_launch(int *bn, int *ctas, int *units, int *pair);
/* Kernel of the last lsb_conv2d_nchw on this process: 0 SIMT implicit GEMM,
 * 1 NHWC-copy tensor-core kernel, 2 planar tensor-core kernel (*nt = its
 * pixel tile, 0 otherwise).  Diagnostics for tests and tools. */
int lsb_last_conv_kernel(int *kind, int *nt);

/* ---- kernels ---------------------------------------------------------------- */
int lsb_semiring_gemm(const lsb_gemm_desc *desc, void *stream);
/* the LSB_ALGO_* lsb_semiring_gemm will use for `desc` (AUTO resolved:
 * the split-precision tensor-core path for large batch-1 (mul, add)
 * contractions, else the
 * SIMT semiring kernel); < 0 if an explicit request cannot be honoured */
int lsb_gemm_algo(const lsb_gemm_desc *desc);
int lsb_conv2d_nchw(const lsb_conv_desc *desc, void *stream);
int lsb_affine_nest(const lsb_nest_desc *desc, void *stream);
/* diagnostics: which kernel the last lsb_affine_nest call launched --
 * 0 affine_nest_kernel (general), 1 nest_rows_kernel, 2 nest_transpose_kernel,
 * 3 nest_vec4_kernel, 4 nest_pool_kernel, 5 nest_transpose4_kernel */
int lsb_last_nest_kernel(int *kind);

/* per-kernel timing for rooflines: when enabled, the dominant kernel of each
 * lsb_semiring_gemm call (the contraction, not its prepass / fold) is
 * bracketed by CUDA events on the call's stream; lsb_last_kernel_ms waits for
 * and returns the most recent one.  Not for use inside graph capture. */
int lsb_profile(int enable);
int lsb_last_kernel_ms(float *ms);

/* ---- optional all-gather of row shards -----------------------
 * Rank r of P holds rows [r*R, (r+1)*R) of a row-major matrix; the gather
 * leaves all P*R rows on every rank.  NCCL over NVLink / NVSwitch, loaded at
 * run time (dlopen libnccl.so.2: the copy torch already loaded when present).
 * unique id: 128 opaque bytes made on one rank and shared out of band. */
#define LSB_NCCL_ID_BYTES 128
int lsb_nccl_unique_id(unsigned char *id /* LSB_NCCL_ID_BYTES */);
int lsb_nccl_init(int rank, int nranks, const unsigned char *id, void **comm);
int lsb_nccl_destroy(void *comm);
/* send: this rank's count floats; recv: nranks*count floats, rank r's block
 * at recv + r*count; asynchronous on stream */
int lsb_allgather_rows(void *comm, const float *send, float *recv, int64_t count, void *stream);

/* sizeof of the descriptor structs (which: 0 gemm, 1 conv, 2 nest, 3 epi
 * stage) so bindings can verify their layout without a GPU */
int64_t lsb_sizeof(int which);

/* number of kernel launches issued since the last reset (launch accounting
 * for bench.py's "gpu_launches") */
int64_t lsb_launch_count(int reset);

#ifdef __cplusplus
}
#endif
#endif /* LSB_H_ */
