/*
 * plssvm.h -- C ABI of the B200-native PLSSVM hot path (LS-SVM training by CG on the
 * reduced kernel system Q~, and prediction).  extern "C", plain pointers and sizes only.
 *
 * Citations: P:L = PAPER.md line L (arXiv 2202.12674, Van Craen/Breyer/Pflüger),
 *            S:L = SPEC.md line L.  DESIGN.md lists every reading of the paper used here.
 *
 * What is computed (one call of plssvm_train*):
 *   full LS-SVM system  [[Q, 1],[1^T, 0]] [alpha; b] = [y; 0],  Q_ij = k(x_i,x_j) + delta_ij/C
 *                                                                  (Eq. 11)
 *   reduced system      Q~ a~ = y_bar - y_m 1                       (Eq. 14)
 *   Q~_ij = k(x_i,x_j) + delta_ij/C - k(x_m,x_j) - k(x_i,x_m) + k(x_m,x_m) + 1/C
 *                                                                  (Eq. 16)
 *   x_m = the LAST point (index m-1); CG = Shewchuk's algorithm, x0 = 0,
 *   stop when ||r|| <= eps ||r0|| on the recurrence residual (R-5)
 *   b = y_m + Q_mm <1, a~> - <q, a~>  (Eq. 15),  alpha = (a~, -sum a~)
 * Kernels: 0 linear <x,z>; 1 polynomial (gamma <x,z> + coef0)^degree;
 *                      2 radial exp(-gamma ||x - z||^2).
 * Decision function (Eq. 10, labels absorbed into alpha, R-2):
 *   f(z) = sum_i alpha_i k(x_i, z) + b ; label = +1 if f >= 0 else -1 (sgn(0) -> +1).
 *
 * Memory / ownership: unless options.device_pointers != 0, every pointer is a HOST pointer
 * owned by the caller; the library copies what it needs to the device, never retains a
 * pointer after return and never returns memory the caller must free.  With
 * device_pointers != 0, X, y, alpha, b, Z, decision, labels, p, out are DEVICE pointers on
 * options.device (e.g. torch tensors' data_ptr()), and all work is ordered on
 * options.stream (cudaStream_t; cudaStreamLegacy = the legacy default stream; NULL = the
 * library's own non-blocking stream, one per host thread and device, NOT ordered after other
 * streams' work); the call still returns only after the results are written (it synchronises
 * that stream).
 * Layout: X is point-major (row i = point i), m x d, C-contiguous (numpy/torch default);
 * Z is n x d, same layout.  The device transposes to the paper's feature-major layout
 * itself.
 * Validation: scalar arguments on the host; X, Z, alpha, p (finite) and y (every y_i in
 * {-1, +1}, both present) on the device right after they are staged, for host and device
 * pointers alike (one small read-back; no host-side scan of the caller's arrays).
 * Errors: every entry point returns a plssvm_status_t; on any error the outputs are left
 * untouched (except PLSSVM_W_NOT_CONVERGED, which fills alpha and b) and
 * plssvm_last_error() returns a thread-local message valid until the next call on the thread.
 * There is no CPU fallback: without a usable CUDA device every compute call returns
 * PLSSVM_E_CUDA.
 * Thread safety: concurrent calls must use different devices or different streams.
 * Multi-GPU: either one process per GPU with a communicator (options.comm, plssvm_comm_init) or one
 * call driving options.num_gpus devices itself (a host thread per device, NCCL or peer transport).
 */
#ifndef PLSSVM_B200_H
#define PLSSVM_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PLSSVM_API __attribute__((visibility("default")))
#else
#define PLSSVM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { PLSSVM_LINEAR = 0, PLSSVM_POLYNOMIAL = 1, PLSSVM_RBF = 2 } plssvm_kernel_t;

typedef enum {
    PLSSVM_OK = 0,
    PLSSVM_E_INVALID_ARG = 1,  /* m < 2, d < 1, C <= 0, gamma <= 0 (poly/rbf), degree < 1,
                                  eps <= 0, unknown kernel, non-finite X/Z/alpha/p, NULL pointer */
    PLSSVM_E_LABELS = 2,       /* a y_i not in {-1,+1}, or only one class present */
    PLSSVM_E_OOM = 3,          /* device allocation failed */
    PLSSVM_E_CUDA = 4,         /* CUDA runtime error / no device */
    PLSSVM_E_NCCL = 5,         /* NCCL error in row-sharded mode */
    PLSSVM_E_NUMERICAL = 6,    /* CG breakdown: p.Q~p <= 0 or non-finite */
    PLSSVM_W_NOT_CONVERGED = 7, /* max_iter reached (or the stagnation guard fired, stats.stop_reason)
                                   before ||r|| <= eps ||r0||; alpha, b filled */
    PLSSVM_E_IO = 8            /* file open / read / write failure or malformed file (message names the line) */
} plssvm_status_t;

typedef enum { PLSSVM_F64 = 0, PLSSVM_F32 = 1 } plssvm_dtype_t;
/* LOWRANK (linear kernel only): Q~p = B^T (X (X^T (B p))) + (p + 1 sum p)/C with B = [I; -1^T]
 * (Q~ = B^T Q B, Eq. 13), two O(m d) streams over X per product instead of O(m^2 d) -- a
 * different cost model from the paper's implicit entries; never picked by AUTO. */
typedef enum { PLSSVM_MODE_AUTO = 0, PLSSVM_MODE_IMPLICIT = 1, PLSSVM_MODE_CACHED = 2, PLSSVM_MODE_LOWRANK = 3 } plssvm_mode_t;

/* Options for the _ex entry points.  plssvm_default_options() fills the defaults given in
 * brackets.  All-zero is NOT the default (stream/comm NULL are fine, but mode 0 = AUTO). */
typedef struct {
    int32_t mode;            /* plssvm_mode_t [AUTO: cached when Q~ fits in free HBM, §8(a3')] */
    int32_t x0;              /* CG start: 0 = zeros [0], 1 = ones (reproduces paper Fig. 3) */
    int64_t max_iter;        /* CG iteration cap; <= 0 means m-1 [0] */
    int64_t replace_every;   /* explicit residual r = rhs - Q~x every R iterations; 0 = off [0] */
    int64_t fixed_iter;      /* > 0: run exactly this many CG iterations, ignore eps (throughput
                                benchmarking); the returned model is the state after them [0] */
    int32_t device;          /* CUDA device ordinal [0] */
    int32_t device_pointers; /* 1: X,y,alpha,b,Z,... are device pointers on `device` [0] */
    void *stream;            /* cudaStream_t to order work on; NULL = library stream [NULL] */
    void *comm;              /* plssvm_comm_t from plssvm_comm_init (row-sharded multi-GPU,
                                one process per GPU); NULL = single GPU [NULL] */
    int64_t cache_budget_bytes; /* AUTO/CACHED: max bytes for the cached Q~ band;
                                   <= 0 means 90 % of free HBM after the other buffers [0] */
    int32_t fp32_engine;     /* plssvm_fp32_engine_t: fp32 contraction of the implicit Q~p, the cached
                                precompute and predict [AUTO] */
    int32_t linear_w;        /* predict with the linear kernel through w = sum_i alpha_i x_i (Eq. 15,
                                O((m+n)d)) [1]; 0 = evaluate the kernel matrix like the other kernels */
    int32_t fp64_engine;     /* plssvm_fp64_engine_t: fp64 pairwise contraction of the implicit Q~p, the
                                cached precompute and predict [AUTO] */
    int32_t cg_loop;         /* plssvm_cg_loop_t: how the CG iterations are issued [AUTO] */
    int32_t multi_gpu;       /* plssvm_multi_gpu_t: how `comm`'s ranks share the work [ROWS] */
    int32_t cg_variant;      /* plssvm_cg_variant_t [SHEWCHUK] */
    int32_t num_gpus;        /* single-process multi-GPU: this call drives num_gpus devices
                                [device, device+1, ...) (modulo the visible device count: ranks beyond it
                                share devices round-robin -- correct, not faster) with one host thread and
                                one row shard per device; <= 0 means the PLSSVM_NUM_GPUS environment
                                variable, else 1 [0].  Not with `comm` (that is the one-process-per-GPU
                                mode).  train: rank 0 (on `device`) writes alpha, b; predict: the test
                                points are split over the devices */
    int32_t transport;       /* plssvm_transport_t: collectives of the num_gpus mode [AUTO] */
    int32_t true_residual;   /* 1: after CG, one more product gives ||rhs - Q~x|| / ||r0|| in
                                stats.rel_residual_true (SURVEY §5 metrics) [0: not computed, stats -1] */
    int32_t reserved0;
    double *residual_trace;  /* HOST buffer (nullable) for the CG trace (SPEC CGTrace): on return
                                residual_trace[k] = ||r_k||, the recurrence residual norm after iteration k,
                                k = 0 .. min(iterations, residual_trace_len - 1) (entry 0: the initial
                                residual); entries beyond are untouched.  Shewchuk variant only; the CG
                                loop is then issued in batches (no CUDA graph) [NULL] */
    int64_t residual_trace_len;  /* entries available in residual_trace [0] */
} plssvm_options_t;

/* Collectives of the single-process multi-GPU mode (options.num_gpus > 1).
 *  NCCL: ncclCommInitAll over the devices (needs distinct devices); all-gather of p, all-reduces
 *        of the CG scalars, reduce-scatter of the circulant partial products over NVLink.
 *  PEER: the library's own transport over peer memory (NVLink P2P): the p update kernel stores its
 *        band straight into every rank's p buffer (the all-gather fused into the CG update,
 *        SURVEY §8(f) NEXT-1), scalars and partial products are pulled with peer copies and summed
 *        in rank order by every rank (deterministic, identical on all ranks); cross-device order
 *        comes from CUDA events, no host round trip per collective beyond an enqueue barrier.
 *        Works with ranks sharing a device.
 *  AUTO: NCCL when every rank has its own device, else PEER. */
typedef enum { PLSSVM_TRANSPORT_AUTO = 0, PLSSVM_TRANSPORT_NCCL = 1, PLSSVM_TRANSPORT_PEER = 2 } plssvm_transport_t;

/* CG formulation.  SHEWCHUK: the paper's loop (two inner products per iteration, each
 * its own reduction / all-reduce).  SINGLE_REDUCTION: Chronopoulos-Gear CG:
 * the product is taken of r, s = Q~p is carried by recurrence, and gamma = r.r, delta = (Q~r).r
 * share ONE reduction point (one all-reduce of a scalar pair per iteration on several GPUs, three
 * kernels per iteration instead of four).  Same iterates in exact arithmetic, same stopping rule
 * (||r|| <= eps ||r0||); one extra product at exit.  Not with replace_every > 0. */
typedef enum { PLSSVM_CG_SHEWCHUK = 0, PLSSVM_CG_SINGLE_REDUCTION = 1 } plssvm_cg_variant_t;

/* CG loop issue.  The convergence test always runs on the device
 * (Shewchuk's loop condition, evaluated by the last block of the p update).
 *  BATCHED: the host enqueues iterations in batches of 8 and reads the control block once per
 *           batch; per-product CUDA events give stats.t_matvec.
 *  GRAPH:   one CUDA graph whose device-side WHILE conditional node runs the iteration body
 *           until the device sets the condition to 0 -- a single launch, no host round trip;
 *           stats.t_matvec stays 0 (no events inside conditional bodies).  Single GPU only, and
 *           not with replace_every > 0 (its period is a host-side branch).
 *  AUTO:    GRAPH when it applies and one product is latency-sized (cached / low-rank products,
 *           or m <= 8192), else BATCHED (launch overhead < 0.1 % of a multi-ms product). */
typedef enum { PLSSVM_CG_AUTO = 0, PLSSVM_CG_BATCHED = 1, PLSSVM_CG_GRAPH = 2 } plssvm_cg_loop_t;

/* Multi-GPU work split when options.comm has P > 1 ranks.
 *  ROWS:     Q~ rows are sharded (cached: row bands; implicit: circulant symmetric tile pairs +
 *            reduce-scatter), all kernels; p all-gathered, CG scalars all-reduced.
 *  FEATURES: the paper's own multi-GPU scheme (§III-C5): every rank holds all points
 *            but only its feature slice [f0, f1) (plssvm_feature_partition), computes the
 *            partial Q~^(g) p of Eq. 16 restricted to those features (the 1/C terms on rank 0
 *            only), and the partial products are summed by one all-reduce of the m-1 vector per
 *            iteration; the CG vectors are replicated.  Valid for the LINEAR kernel only (the
 *            kernel must be a sum over features), fp64, implicit products (mode AUTO or
 *            IMPLICIT); needs d >= P.  Otherwise PLSSVM_E_INVALID_ARG. */
typedef enum { PLSSVM_MULTI_GPU_ROWS = 0, PLSSVM_MULTI_GPU_FEATURES = 1 } plssvm_multi_gpu_t;

/* fp32 contraction engines.
 *  TCGEN05: tcgen05 kind::tf32 tensor cores, 3xTF32 hi/lo split (21 + 21 bits per operand).
 *  FFMA:    CUDA-core fp32 FMA tiles.
 *  OZAKI:   int8 tensor cores (tcgen05 kind::i8, 2-SM UMMA) on a 3-digit balanced base-256 split of
 *           every point, rounded to 22 bits below its row maximum (6 digit pairs, exact int32 sums,
 *           one TMEM pass): |s~ - s| <= u32 |s| + 40.2 d u32 ||x_i||_inf ||x_j||_inf, u32 = 2^-24.
 *           d <= 16384.
 *  AUTO:    OZAKI when 40.2 rho^2 <= d (rho as for fp64: the bound is then no larger than an fp32
 *           dot product's in Cauchy-Schwarz form) and d <= 16384, else TCGEN05. */
typedef enum { PLSSVM_FP32_TCGEN05 = 0, PLSSVM_FP32_FFMA = 1, PLSSVM_FP32_OZAKI = 2, PLSSVM_FP32_AUTO = 3 } plssvm_fp32_engine_t;

/* fp64 contraction engines.
 *  OZAKI: int8 tensor cores (tcgen05 kind::i8, 2-SM UMMA).  Every point is rounded to the fixed-point
 *         grid 2^(E_i-54) of its row maximum (2^(E_i-1) <= max_k |x_ik| < 2^E_i; features within a
 *         factor 4 of the maximum are exact) and written as 7 balanced base-256 int8 digits; the 28
 *         digit-pair products of levels a+b <= 6 are summed exactly in int32 and combined with one fp64
 *         rounding.  Error of s = x_i.x_j:
 *             |s~ - s| <= u |s| + 13.04 d u ||x_i||_inf ||x_j||_inf,   u = 2^-53
 *         i.e. an fp64-GEMM-type bound weighted by the row maxima, not the componentwise
 *         d u sum_k |x_ik x_jk| of an fp64 dot.  Needs d <= 16384 (int32 level sums).
 *  DMMA:  fp64 tensor cores (mma.sync f64, error <~ d u sum_k |x_ik||x_jk|).
 *  AUTO:  OZAKI when its bound is no larger than the fp64 dot product's in Cauchy-Schwarz form
 *         (d u ||x_i||_2 ||x_j||_2): 13.04 rho^2 <= d with rho = max over points of
 *         max_k |x_ik| / rms_k(x_ik) (N(0,1)-like data: rho ~ 5, so d >= ~330); else DMMA.  Also DMMA
 *         for d > 16384 and for tiny problems (at most 384 padded points, where the persistent
 *         kernel's fixed cost dominates). */
typedef enum { PLSSVM_FP64_AUTO = 0, PLSSVM_FP64_OZAKI = 1, PLSSVM_FP64_DMMA = 2 } plssvm_fp64_engine_t;

/* Statistics of one training call (all times are device-event seconds). */
typedef struct {
    int64_t iterations;              /* CG iterations performed */
    int64_t matvecs;                 /* Q~ products performed (incl. initial / replacement) */
    double rel_residual;             /* ||r|| / ||r0|| of the recurrence at exit */
    int32_t mode_used;               /* PLSSVM_MODE_IMPLICIT, _CACHED or _LOWRANK */
    int32_t num_ranks;               /* 1, or the communicator size */
    double t_h2d, t_transform, t_q;
    double t_alloc;                  /* device work-buffer allocation (stream-ordered pool) */
    double t_precompute, t_cg, t_bias_d2h, t_total;
    double t_matvec;                 /* summed duration of the Q~p kernels (CUDA events) */
    double t_matvec_min;             /* shortest single Q~p kernel duration */
    int64_t bytes_per_gpu;           /* device bytes allocated by this call on this GPU */
    int64_t gpu_launches;            /* kernels launched by this call (this rank) */
    int64_t launches_in_cg;          /* of which inside the CG loop */
    int32_t fp64_engine_used;        /* PLSSVM_FP64_OZAKI or _DMMA for fp64 calls, 0 for fp32 */
    int32_t cg_loop_used;            /* PLSSVM_CG_BATCHED or PLSSVM_CG_GRAPH */
    int32_t fp32_engine_used;        /* fp32 calls: PLSSVM_FP32_OZAKI, _TCGEN05 or _FFMA; 0 for fp64 */
    int32_t allgather_fused;         /* 1: the all-gather of p was part of the p update kernel (NCCL device
                                        API stores into the ranks' symmetric windows, or the PEER
                                        transport's peer stores); 0: a separate collective or one GPU */
    double t_comm;                   /* summed duration of the CG loop's collectives (all-gather of p,
                                        scalar all-reduces, reduce-scatter of the partial products;
                                        CUDA events, batched loop; 0 on one GPU) -- inside t_matvec for
                                        the reduce-scatter, which is part of the product */
    double rel_residual_true;        /* ||rhs - Q~x|| / ||r0|| from one extra product after CG
                                        (options.true_residual = 1), else -1 */
    int32_t stop_reason;             /* plssvm_stop_t: why the CG loop ended */
    int32_t transport_used;          /* num_gpus mode: PLSSVM_TRANSPORT_NCCL or _PEER; 0 otherwise */
} plssvm_stats_t;

/* Why the CG loop stopped (stats.stop_reason). */
typedef enum {
    PLSSVM_STOP_CONVERGED = 0,   /* ||r|| <= eps ||r0|| (recurrence residual) */
    PLSSVM_STOP_MAX_ITER = 1,    /* options.max_iter (or m-1) iterations -> PLSSVM_W_NOT_CONVERGED */
    PLSSVM_STOP_FIXED = 2,       /* options.fixed_iter iterations done */
    PLSSVM_STOP_STAGNATED = 3,   /* stagnation guard (replace_every > 0, R-20): no 4x drop of
                                    r.r within 2 max(R, 50) iterations -> PLSSVM_W_NOT_CONVERGED */
    PLSSVM_STOP_BREAKDOWN = 4    /* p.Q~p <= 0 or non-finite -> PLSSVM_E_NUMERICAL */
} plssvm_stop_t;

PLSSVM_API void plssvm_default_options(plssvm_options_t *opts);

/* ---- training (Eq. 11-16 + CG) ------------------------------------------------------
 * X [m*d] point-major, y [m] entries +1/-1.  alpha [m] out, b [1] out.
 * gamma is used by poly/rbf (must be > 0 there); degree (>= 1) and coef0 by poly only. */
PLSSVM_API int plssvm_train(const double *X, const double *y, int64_t m, int64_t d, int kernel, double gamma,
                 int degree, double coef0, double C, double eps, double *alpha, double *b);
PLSSVM_API int plssvm_train_f32(const float *X, const float *y, int64_t m, int64_t d, int kernel, float gamma,
                     int degree, float coef0, float C, float eps, float *alpha, float *b);
/* dtype selects double (X, y, alpha, b are double*) or float (float*).  opts/stats nullable. */
PLSSVM_API int plssvm_train_ex(const void *X, const void *y, int64_t m, int64_t d, int dtype, int kernel,
                    double gamma, int degree, double coef0, double C, double eps,
                    const plssvm_options_t *opts, void *alpha, void *b, plssvm_stats_t *stats);

/* ---- prediction (Eq. 10) -------------------------------------------------------------
 * X [m*d] training points, alpha [m], b: the model.  Z [n*d] points to classify.
 * decision [n] (nullable) receives f(z); labels [n] (nullable) receives +1/-1. */
PLSSVM_API int plssvm_predict(const double *X, const double *alpha, double b, int64_t m, int64_t d, int kernel,
                   double gamma, int degree, double coef0, const double *Z, int64_t n,
                   double *decision, int32_t *labels);
PLSSVM_API int plssvm_predict_f32(const float *X, const float *alpha, float b, int64_t m, int64_t d, int kernel,
                       float gamma, int degree, float coef0, const float *Z, int64_t n,
                       float *decision, int32_t *labels);
PLSSVM_API int plssvm_predict_ex(const void *X, const void *alpha, double b, int64_t m, int64_t d, int dtype,
                      int kernel, double gamma, int degree, double coef0, const void *Z, int64_t n,
                      const plssvm_options_t *opts, void *decision, int32_t *labels, double *t_kernel);
/* t_kernel (nullable, 2 doubles): [0] duration (s) of the predict tile kernel, [1] number of
 * kernels this call launched. */

/* ---- the hot product alone (diagnostics, parity tests, roofline) ----------------------
 * out[m-1] = Q~ p for p [m-1] (Eq. 16), computed `repeats` times (>= 1) with the mode in
 * opts (IMPLICIT: recompute tiles; CACHED: precompute Q~ once then stream it).
 * t_kernel (nullable, 3 doubles) receives: mean, min duration (s) of one Q~p product, and
 * the one-time precompute duration (cached mode, else 0). */
PLSSVM_API int plssvm_qtilde_matvec(const void *X, const void *p, int64_t m, int64_t d, int dtype, int kernel,
                         double gamma, int degree, double coef0, double C, int32_t repeats,
                         const plssvm_options_t *opts, void *out, double *t_kernel);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) -----------------------------------
 * Vectors are row-sharded (rank r owns rows [r*m_pad/P, (r+1)*m_pad/P)).  Cached mode: each
 * rank stores and streams its rows of Q~.  Implicit mode: the symmetric tile pairs are dealt
 * out circulantly (tile row I computes pairs (I, I+j mod T), j = 0..T/2), so every rank does
 * ~1/P of the symmetric work; the partial products are combined by a reduce-scatter.
 * plssvm_comm_unique_id writes an opaque 128-byte NCCL id (rank 0 creates it, the caller
 * broadcasts it, e.g. with torch.distributed); every rank then calls plssvm_comm_init.
 * The communicator is bound to `device`.  Destroy with plssvm_comm_destroy. */
typedef void *plssvm_comm_t;
PLSSVM_API int plssvm_comm_unique_id(void *id128);
PLSSVM_API int plssvm_comm_init(const void *id128, int32_t nranks, int32_t rank, int32_t device, plssvm_comm_t *comm);
PLSSVM_API int plssvm_comm_destroy(plssvm_comm_t comm);

/* Caller-supplied transport (e.g. MPI, or a host-staged gloo exchange in tests): the same
 * row-sharded driver, with the two collectives it needs delegated to these callbacks.  Both
 * operate IN PLACE on DEVICE memory of `device`, must be complete (or ordered on `stream`)
 * when they return, and return 0 on success (anything else aborts the call with
 * PLSSVM_E_NCCL).  The struct is copied; ctx is passed through untouched. */
typedef struct {
    void *ctx;
    /* buf[0..count) <- sum over ranks of buf[0..count)   (doubles) */
    int (*allreduce_sum_f64)(void *ctx, double *buf, int64_t count, void *stream);
    /* rank r's count_per_rank elements live at buf + r * count_per_rank; afterwards every rank
     * holds all nranks * count_per_rank elements.  dtype: PLSSVM_F64 / PLSSVM_F32. */
    int (*allgather)(void *ctx, void *buf, int64_t count_per_rank, int32_t dtype, void *stream);
    /* optional (NULL: implicit mode falls back to row bands): recv[0..count_per_rank) <- this
     * rank's block of the element-wise sum over ranks of send[0..nranks*count_per_rank). */
    int (*reduce_scatter_sum)(void *ctx, const void *send, void *recv, int64_t count_per_rank, int32_t dtype,
                              void *stream);
} plssvm_comm_callbacks_t;
PLSSVM_API int plssvm_comm_init_callbacks(const plssvm_comm_callbacks_t *cb, int32_t nranks, int32_t rank,
                                          int32_t device, plssvm_comm_t *comm);

/* Host-side partition rule (no GPU needed): rows [row_begin, row_end) of the padded
 * (m-1)-system owned by `rank` of `nranks`, and the padded length m_pad (a multiple of
 * 128 * nranks).  Rows >= m-1 are padding (masked). */
PLSSVM_API int plssvm_partition(int64_t m, int32_t nranks, int32_t rank, int64_t *row_begin, int64_t *row_end,
                     int64_t *m_pad);

/* Host-side feature split of PLSSVM_MULTI_GPU_FEATURES (no GPU needed): rank `rank` of `nranks`
 * owns features [f_begin, f_end) = [rank*d/nranks, (rank+1)*d/nranks) (integer division, so the
 * slices differ by at most one feature).  d >= nranks >= 1. */
PLSSVM_API int plssvm_feature_partition(int64_t d, int32_t nranks, int32_t rank, int64_t *f_begin, int64_t *f_end);

/* ---- LIBSVM files and scaling -----------------------------------
 * The read / write steps around the hot path (the paper's runtime components, Fig. 2,
 * P:624-632) and the LIBSVM drop-in formats.  Host-only, no GPU needed; native
 * C++ (io.cpp), multi-threaded parse.  Paths are NUL-terminated file names.  Numbers are
 * parsed correctly rounded and written as %.17g, so files round-trip bit-exactly.
 *
 * plssvm_libsvm_read: data file, one point per line "<label> <index>:<value> ...", 1-based
 *   strictly ascending indices, blank / '#' lines skipped, LF or CRLF.  Sparse
 *   input becomes dense (absent features are 0).  Outputs: m points, d = the
 *   largest index, labels[0..nlabels) = the distinct label values in first-seen order
 *   (nlabels 1 or 2; a third label -> PLSSVM_E_LABELS).  Query mode: X or y NULL -> only m, d,
 *   labels, nlabels are written.  Otherwise needs cap_m >= m, cap_d >= max(d, 1): X[i*cap_d + k]
 *   (row stride cap_d, features >= d set to 0) and y[i] = the RAW label of point i (map it to
 *   +1 / -1 yourself, e.g. labels[0] -> +1 as the CLI does). */
PLSSVM_API int plssvm_libsvm_read(const char *path, double *X, double *y, int64_t cap_m, int64_t cap_d, int64_t *m,
                                  int64_t *d, double *labels /* [2] */, int32_t *nlabels);
/* X [m*d] point-major, y [m] labels: "<y_i> <k+1>:<x_ik> ..." per point, zero features omitted. */
PLSSVM_API int plssvm_libsvm_write(const char *path, const double *X, const double *y, int64_t m, int64_t d);
/* LIBSVM c_svc model file of a trained LS-SVM: header svm_type c_svc, kernel_type,
 * degree (poly) / gamma (poly, rbf) / coef0 (poly), nr_class 2, total_sv m, rho = -b, label
 * labels[0] labels[1] (the original labels of y = +1 and y = -1), nr_sv n+ n-, SV; then one line
 * per training point "<alpha_i> <k>:<x_ik> ..." -- every LS-SVM point is a support vector, the
 * y = +1 points first (LIBSVM's class grouping), each group in input order.  y [m] = +1 / -1. */
PLSSVM_API int plssvm_model_write(const char *path, int kernel, double gamma, int degree, double coef0,
                                  const double *X, const double *alpha, double b, int64_t m, int64_t d,
                                  const double *y, const double *labels /* [2] */);
/* Reads a model written by plssvm_model_write or an equivalent LIBSVM c_svc model:
 * unknown kernel_type, nr_class != 2, or a missing mandatory field -> PLSSVM_E_IO with the field
 * named.  b = -rho; labels[0] is predicted for f >= 0.  Query mode: X or alpha NULL.  Otherwise
 * cap_m >= m, cap_d >= max(d, 1), X row stride cap_d. */
PLSSVM_API int plssvm_model_read(const char *path, int32_t *kernel, double *gamma, int32_t *degree, double *coef0,
                                 double *X, double *alpha, double *b, int64_t cap_m, int64_t cap_d, int64_t *m,
                                 int64_t *d, double *labels /* [2] */);
/* svm-scale: per-feature ranges over all m points (zeros included) ... */
PLSSVM_API int plssvm_scale_fit(const double *X, int64_t m, int64_t d, double *fmin /* [d] */, double *fmax /* [d] */);
/* ... and the affine map x -> lo + (hi - lo) (x - min) / (max - min), constant features -> lo, no
 * clamping (values outside the fitted range map outside [lo, hi]).  In place.  lo < hi. */
PLSSVM_API int plssvm_scale_apply(double *X, int64_t m, int64_t d, const double *fmin, const double *fmax, double lo,
                                  double hi);

/* ---- misc ------------------------------------------------------------------------------ */
PLSSVM_API const char *plssvm_last_error(void); /* thread-local; "" when the last call succeeded */
PLSSVM_API const char *plssvm_version(void);    /* build string: version, sm arch, CUDA and NCCL versions */
PLSSVM_API int plssvm_device_count(void);       /* visible CUDA devices (0 when none / no driver) */

#ifdef __cplusplus
}
#endif
#endif /* PLSSVM_B200_H */
