// capi.cu -- the extern "C" boundary declared in include/plssvm.h: validation, error
// conventions (status codes + thread-local message), dispatch to the device driver.
// Validation rules (plssvm.h): m >= 2, d >= 1; y_i in {-1,+1}
// with both classes present; C > 0; gamma > 0 for poly/rbf and degree >= 1
// (P:248-249); eps > 0; kernel in {0,1,2}.  Finite X / Z / alpha / p and the labels are checked
// on the device after staging (driver.cu validate_inputs), for host and device pointers alike.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "../../include/plssvm.h"
#include "common.cuh"
#include "driver.h"
#include "io.h"

#ifndef PLSSVM_VERSION
#define PLSSVM_VERSION "0.1.0"
#endif

extern "C" int plssvm_comm_unique_id_impl(void *id128);
extern "C" int plssvm_comm_init_impl(const void *id128, int32_t nranks, int32_t rank, int32_t device, void **out);
extern "C" int plssvm_comm_destroy_impl(void *c);
extern "C" int plssvm_comm_init_callbacks_impl(const plssvm_comm_callbacks_t *cb, int32_t nranks, int32_t rank,
                                               int32_t device, void **out);

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

template <typename F>
int guarded(F f) {
    g_last_error.clear();
    try {
        return f();
    } catch (const plssvm::Error &e) {
        return fail(e.code, e.what());
    } catch (const std::exception &e) {
        return fail(PLSSVM_E_CUDA, e.what());
    }
}

int device_ok(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0)
        return fail(PLSSVM_E_CUDA, "no CUDA device available (the library has no CPU fallback)");
    if (device < 0 || device >= n) return fail(PLSSVM_E_INVALID_ARG, "options.device out of range");
    return PLSSVM_OK;
}

int check_params(int64_t m, int64_t d, int kernel, double gamma, int degree, double C) {
    if (m < 2) return fail(PLSSVM_E_INVALID_ARG, "m must be >= 2");
    if (d < 1) return fail(PLSSVM_E_INVALID_ARG, "d must be >= 1");
    if (kernel < 0 || kernel > 2) return fail(PLSSVM_E_INVALID_ARG, "kernel must be 0 (linear), 1 (polynomial) or 2 (rbf)");
    if (!(C > 0) || !std::isfinite(C)) return fail(PLSSVM_E_INVALID_ARG, "C must be > 0");
    if (kernel != 0 && (!(gamma > 0) || !std::isfinite(gamma))) return fail(PLSSVM_E_INVALID_ARG, "gamma must be > 0");
    if (kernel == 1 && degree < 1) return fail(PLSSVM_E_INVALID_ARG, "degree must be >= 1");
    return PLSSVM_OK;
}

plssvm_options_t defaults() {
    plssvm_options_t o;
    plssvm_default_options(&o);
    return o;
}

// Engine options (plssvm.h plssvm_fp64_engine_t / plssvm_fp32_engine_t).
int check_engines(const plssvm_options_t &o) {
    if (o.fp64_engine < PLSSVM_FP64_AUTO || o.fp64_engine > PLSSVM_FP64_DMMA)
        return fail(PLSSVM_E_INVALID_ARG, "options.fp64_engine must be 0 (AUTO), 1 (OZAKI) or 2 (DMMA)");
    if (o.fp32_engine < PLSSVM_FP32_TCGEN05 || o.fp32_engine > PLSSVM_FP32_AUTO)
        return fail(PLSSVM_E_INVALID_ARG, "options.fp32_engine must be 0 (TCGEN05), 1 (FFMA), 2 (OZAKI) or 3 (AUTO)");
    return PLSSVM_OK;
}

// PLSSVM_MULTI_GPU_FEATURES (paper §III-C5): linear kernel, fp64, implicit, d >= P.
int check_multi_gpu(const plssvm_options_t &o, int kernel, int dtype, int64_t d) {
    if (int s = check_engines(o)) return s;
    if (o.transport < PLSSVM_TRANSPORT_AUTO || o.transport > PLSSVM_TRANSPORT_PEER)
        return fail(PLSSVM_E_INVALID_ARG, "options.transport must be 0 (AUTO), 1 (NCCL) or 2 (PEER)");
    if (o.comm && plssvm::resolve_num_gpus(o) > 1)
        return fail(PLSSVM_E_INVALID_ARG, "options.num_gpus > 1 (one call drives several GPUs) cannot be combined "
                                          "with options.comm (one process per GPU)");
    if (o.comm && o.device != plssvm::comm_device(static_cast<plssvm::CommHandle *>(o.comm)))
        return fail(PLSSVM_E_INVALID_ARG, "options.device must be the device the communicator was created on");
    if (o.multi_gpu != PLSSVM_MULTI_GPU_ROWS && o.multi_gpu != PLSSVM_MULTI_GPU_FEATURES)
        return fail(PLSSVM_E_INVALID_ARG, "options.multi_gpu must be 0 (ROWS) or 1 (FEATURES)");
    if (o.multi_gpu != PLSSVM_MULTI_GPU_FEATURES) return PLSSVM_OK;
    if (kernel != PLSSVM_LINEAR)
        return fail(PLSSVM_E_INVALID_ARG, "multi_gpu FEATURES needs the linear kernel (P:421-425)");
    if (dtype != PLSSVM_F64) return fail(PLSSVM_E_INVALID_ARG, "multi_gpu FEATURES is fp64 only");
    if (o.mode != PLSSVM_MODE_AUTO && o.mode != PLSSVM_MODE_IMPLICIT)
        return fail(PLSSVM_E_INVALID_ARG, "multi_gpu FEATURES computes implicit products (mode AUTO or IMPLICIT)");
    if (o.comm && d < plssvm::comm_size(static_cast<plssvm::CommHandle *>(o.comm)))
        return fail(PLSSVM_E_INVALID_ARG, "multi_gpu FEATURES needs d >= number of ranks");
    return PLSSVM_OK;
}

}  // namespace

extern "C" {

void plssvm_default_options(plssvm_options_t *o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->mode = PLSSVM_MODE_AUTO;
    o->x0 = 0;
    o->max_iter = 0;
    o->replace_every = 0;
    o->fixed_iter = 0;
    o->device = 0;
    o->device_pointers = 0;
    o->stream = nullptr;
    o->comm = nullptr;
    o->cache_budget_bytes = 0;
    o->fp32_engine = PLSSVM_FP32_AUTO;
    o->linear_w = 1;
    o->fp64_engine = PLSSVM_FP64_AUTO;
    o->cg_loop = PLSSVM_CG_AUTO;
    o->multi_gpu = PLSSVM_MULTI_GPU_ROWS;
    o->cg_variant = PLSSVM_CG_SHEWCHUK;
    o->num_gpus = 0;  // PLSSVM_NUM_GPUS, else 1
    o->transport = PLSSVM_TRANSPORT_AUTO;
    o->true_residual = 0;
}

int plssvm_train_ex(const void *X, const void *y, int64_t m, int64_t d, int dtype, int kernel, double gamma, int degree,
                    double coef0, double C, double eps, const plssvm_options_t *opts, void *alpha, void *b,
                    plssvm_stats_t *stats) {
    g_last_error.clear();
    const plssvm_options_t o = opts ? *opts : defaults();
    if (!X || !y || !alpha || !b) return fail(PLSSVM_E_INVALID_ARG, "NULL pointer argument");
    if (dtype != PLSSVM_F64 && dtype != PLSSVM_F32) return fail(PLSSVM_E_INVALID_ARG, "dtype must be 0 (f64) or 1 (f32)");
    int s = check_params(m, d, kernel, gamma, degree, C);
    if (s) return s;
    if (!(eps > 0) || !std::isfinite(eps)) return fail(PLSSVM_E_INVALID_ARG, "eps must be > 0");
    if (o.mode < 0 || o.mode > 3) return fail(PLSSVM_E_INVALID_ARG, "options.mode must be 0, 1, 2 or 3");
    if (o.mode == PLSSVM_MODE_LOWRANK && kernel != PLSSVM_LINEAR)
        return fail(PLSSVM_E_INVALID_ARG, "options.mode LOWRANK needs the linear kernel");
    if (o.x0 != 0 && o.x0 != 1) return fail(PLSSVM_E_INVALID_ARG, "options.x0 must be 0 or 1");
    if (o.cg_loop < 0 || o.cg_loop > 2) return fail(PLSSVM_E_INVALID_ARG, "options.cg_loop must be 0, 1 or 2");
    if (o.cg_variant != PLSSVM_CG_SHEWCHUK && o.cg_variant != PLSSVM_CG_SINGLE_REDUCTION)
        return fail(PLSSVM_E_INVALID_ARG, "options.cg_variant must be 0 (SHEWCHUK) or 1 (SINGLE_REDUCTION)");
    if (o.cg_variant == PLSSVM_CG_SINGLE_REDUCTION && o.replace_every > 0)
        return fail(PLSSVM_E_INVALID_ARG, "cg_variant SINGLE_REDUCTION does not support replace_every");
    if ((s = check_multi_gpu(o, kernel, dtype, d))) return s;
    if ((s = device_ok(o.device))) return s;
    if (stats) std::memset(stats, 0, sizeof(*stats));
    plssvm::Problem pb{X, y, m, d, dtype, kernel, gamma, degree, coef0, C, eps};
    const int P = plssvm::resolve_num_gpus(o);
    if (P > 1) return guarded([&] { return plssvm::train_multi(pb, o, P, alpha, b, stats); });
    return guarded([&] { return plssvm::train(pb, o, alpha, b, stats); });
}

int plssvm_train(const double *X, const double *y, int64_t m, int64_t d, int kernel, double gamma, int degree,
                 double coef0, double C, double eps, double *alpha, double *b) {
    return plssvm_train_ex(X, y, m, d, PLSSVM_F64, kernel, gamma, degree, coef0, C, eps, nullptr, alpha, b, nullptr);
}

int plssvm_train_f32(const float *X, const float *y, int64_t m, int64_t d, int kernel, float gamma, int degree,
                     float coef0, float C, float eps, float *alpha, float *b) {
    return plssvm_train_ex(X, y, m, d, PLSSVM_F32, kernel, gamma, degree, coef0, C, eps, nullptr, alpha, b, nullptr);
}

int plssvm_predict_ex(const void *X, const void *alpha, double b, int64_t m, int64_t d, int dtype, int kernel,
                      double gamma, int degree, double coef0, const void *Z, int64_t n, const plssvm_options_t *opts,
                      void *decision, int32_t *labels, double *t_kernel) {
    g_last_error.clear();
    const plssvm_options_t o = opts ? *opts : defaults();
    if (!X || !alpha || !Z) return fail(PLSSVM_E_INVALID_ARG, "NULL pointer argument");
    if (dtype != PLSSVM_F64 && dtype != PLSSVM_F32) return fail(PLSSVM_E_INVALID_ARG, "dtype must be 0 (f64) or 1 (f32)");
    if (m < 1) return fail(PLSSVM_E_INVALID_ARG, "m must be >= 1");
    int s = check_params(m < 2 ? 2 : m, d, kernel, gamma, degree, 1.0);
    if (s) return s;
    if (n < 0) return fail(PLSSVM_E_INVALID_ARG, "n must be >= 0");
    if (n == 0) return PLSSVM_OK;
    if (!std::isfinite(b)) return fail(PLSSVM_E_INVALID_ARG, "b is not finite");
    if ((s = check_engines(o))) return s;
    if (o.transport < PLSSVM_TRANSPORT_AUTO || o.transport > PLSSVM_TRANSPORT_PEER)
        return fail(PLSSVM_E_INVALID_ARG, "options.transport must be 0 (AUTO), 1 (NCCL) or 2 (PEER)");
    if ((s = device_ok(o.device))) return s;
    plssvm::Problem pb{X, nullptr, m, d, dtype, kernel, gamma, degree, coef0, 1.0, 1.0};
    const int P = plssvm::resolve_num_gpus(o);
    if (P > 1) return guarded([&] { return plssvm::predict_multi(pb, alpha, b, Z, n, o, P, decision, labels, t_kernel); });
    return guarded([&] { return plssvm::predict(pb, alpha, b, Z, n, o, decision, labels, t_kernel); });
}

int plssvm_predict(const double *X, const double *alpha, double b, int64_t m, int64_t d, int kernel, double gamma,
                   int degree, double coef0, const double *Z, int64_t n, double *decision, int32_t *labels) {
    return plssvm_predict_ex(X, alpha, b, m, d, PLSSVM_F64, kernel, gamma, degree, coef0, Z, n, nullptr, decision, labels,
                             nullptr);
}

int plssvm_predict_f32(const float *X, const float *alpha, float b, int64_t m, int64_t d, int kernel, float gamma,
                       int degree, float coef0, const float *Z, int64_t n, float *decision, int32_t *labels) {
    return plssvm_predict_ex(X, alpha, b, m, d, PLSSVM_F32, kernel, gamma, degree, coef0, Z, n, nullptr, decision, labels,
                             nullptr);
}

int plssvm_qtilde_matvec(const void *X, const void *p, int64_t m, int64_t d, int dtype, int kernel, double gamma,
                         int degree, double coef0, double C, int32_t repeats, const plssvm_options_t *opts, void *out,
                         double *t_kernel) {
    g_last_error.clear();
    const plssvm_options_t o = opts ? *opts : defaults();
    if (!X || !p || !out) return fail(PLSSVM_E_INVALID_ARG, "NULL pointer argument");
    if (dtype != PLSSVM_F64 && dtype != PLSSVM_F32) return fail(PLSSVM_E_INVALID_ARG, "dtype must be 0 (f64) or 1 (f32)");
    int s = check_params(m, d, kernel, gamma, degree, C);
    if (s) return s;
    if ((s = device_ok(o.device))) return s;
    if (o.mode < 0 || o.mode > 3) return fail(PLSSVM_E_INVALID_ARG, "options.mode must be 0, 1, 2 or 3");
    if (o.mode == PLSSVM_MODE_LOWRANK && kernel != PLSSVM_LINEAR)
        return fail(PLSSVM_E_INVALID_ARG, "options.mode LOWRANK needs the linear kernel");
    if ((s = check_multi_gpu(o, kernel, dtype, d))) return s;
    plssvm::Problem pb{X, nullptr, m, d, dtype, kernel, gamma, degree, coef0, C, 1.0};
    return guarded([&] { return plssvm::qtilde_matvec(pb, p, repeats, o, out, t_kernel); });
}

int plssvm_comm_unique_id(void *id128) {
    g_last_error.clear();
    if (!id128) return fail(PLSSVM_E_INVALID_ARG, "NULL id buffer");
    int s = plssvm_comm_unique_id_impl(id128);
    return s ? fail(s, "ncclGetUniqueId failed") : PLSSVM_OK;
}

int plssvm_comm_init(const void *id128, int32_t nranks, int32_t rank, int32_t device, plssvm_comm_t *comm) {
    g_last_error.clear();
    if (!id128 || !comm) return fail(PLSSVM_E_INVALID_ARG, "NULL pointer argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PLSSVM_E_INVALID_ARG, "bad rank / nranks");
    int s = device_ok(device);
    if (s) return s;
    s = plssvm_comm_init_impl(id128, nranks, rank, device, comm);
    return s ? fail(s, "ncclCommInitRank failed") : PLSSVM_OK;
}

int plssvm_comm_init_callbacks(const plssvm_comm_callbacks_t *cb, int32_t nranks, int32_t rank, int32_t device,
                               plssvm_comm_t *comm) {
    g_last_error.clear();
    if (!cb || !comm || !cb->allreduce_sum_f64 || !cb->allgather) return fail(PLSSVM_E_INVALID_ARG, "NULL callback");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PLSSVM_E_INVALID_ARG, "bad rank / nranks");
    if (device < 0) return fail(PLSSVM_E_INVALID_ARG, "bad device");
    return plssvm_comm_init_callbacks_impl(cb, nranks, rank, device, comm);
}

int plssvm_comm_destroy(plssvm_comm_t comm) { return plssvm_comm_destroy_impl(comm); }

int plssvm_partition(int64_t m, int32_t nranks, int32_t rank, int64_t *row_begin, int64_t *row_end, int64_t *m_pad) {
    g_last_error.clear();
    if (m < 2 || nranks < 1 || rank < 0 || rank >= nranks || !row_begin || !row_end || !m_pad)
        return fail(PLSSVM_E_INVALID_ARG, "bad partition arguments");
    const int64_t mpad = plssvm::round_up(m, static_cast<int64_t>(plssvm::kTile) * nranks);
    const int64_t nb = mpad / nranks;
    *m_pad = mpad;
    *row_begin = static_cast<int64_t>(rank) * nb;
    *row_end = *row_begin + nb;
    return PLSSVM_OK;
}

int plssvm_feature_partition(int64_t d, int32_t nranks, int32_t rank, int64_t *f_begin, int64_t *f_end) {
    g_last_error.clear();
    if (d < 1 || nranks < 1 || d < nranks || rank < 0 || rank >= nranks || !f_begin || !f_end)
        return fail(PLSSVM_E_INVALID_ARG, "bad feature partition arguments");
    *f_begin = plssvm::feature_begin(d, nranks, rank);
    *f_end = plssvm::feature_begin(d, nranks, rank + 1);
    return PLSSVM_OK;
}

int plssvm_libsvm_read(const char *path, double *X, double *y, int64_t cap_m, int64_t cap_d, int64_t *m, int64_t *d,
                       double *labels, int32_t *nlabels) {
    return guarded([&] {
        plssvm::io::libsvm_read(path, X, y, cap_m, cap_d, m, d, labels, nlabels);
        return PLSSVM_OK;
    });
}

int plssvm_libsvm_write(const char *path, const double *X, const double *y, int64_t m, int64_t d) {
    if (!X || !y || m < 0 || d < 0) return fail(PLSSVM_E_INVALID_ARG, "bad libsvm_write arguments");
    return guarded([&] {
        plssvm::io::libsvm_write(path, X, y, m, d);
        return PLSSVM_OK;
    });
}

int plssvm_model_write(const char *path, int kernel, double gamma, int degree, double coef0, const double *X,
                       const double *alpha, double b, int64_t m, int64_t d, const double *y, const double *labels) {
    if (!X || !alpha || !y || !labels || m < 1 || d < 1) return fail(PLSSVM_E_INVALID_ARG, "bad model_write arguments");
    return guarded([&] {
        plssvm::io::model_write(path, kernel, gamma, degree, coef0, X, alpha, b, m, d, y, labels);
        return PLSSVM_OK;
    });
}

int plssvm_model_read(const char *path, int32_t *kernel, double *gamma, int32_t *degree, double *coef0, double *X,
                      double *alpha, double *b, int64_t cap_m, int64_t cap_d, int64_t *m, int64_t *d, double *labels) {
    return guarded([&] {
        plssvm::io::model_read(path, kernel, gamma, degree, coef0, X, alpha, b, cap_m, cap_d, m, d, labels);
        return PLSSVM_OK;
    });
}

int plssvm_scale_fit(const double *X, int64_t m, int64_t d, double *fmin, double *fmax) {
    g_last_error.clear();
    if (!X || !fmin || !fmax || m < 1 || d < 1) return fail(PLSSVM_E_INVALID_ARG, "bad scale_fit arguments");
    plssvm::io::scale_fit(X, m, d, fmin, fmax);
    return PLSSVM_OK;
}

int plssvm_scale_apply(double *X, int64_t m, int64_t d, const double *fmin, const double *fmax, double lo, double hi) {
    g_last_error.clear();
    if (!X || !fmin || !fmax || m < 0 || d < 1) return fail(PLSSVM_E_INVALID_ARG, "bad scale_apply arguments");
    if (!(lo < hi)) return fail(PLSSVM_E_INVALID_ARG, "scale_apply: lower bound must be < upper bound");
    plssvm::io::scale_apply(X, m, d, fmin, fmax, lo, hi);
    return PLSSVM_OK;
}

const char *plssvm_last_error(void) { return g_last_error.c_str(); }

#ifdef PLSSVM_OZ_EXPERIMENTS
// Experiment build only (not part of the product ABI): copy / reset the k_tile_ozaki cycle counters.
PLSSVM_API int plssvm_exp_oz_profile(unsigned long long *out /* 160 x 8 */, int reset) {
    return plssvm::exp_oz_profile(out, reset);
}
#endif

const char *plssvm_version(void) {
    static std::string v;
    if (v.empty()) {
        int rt = 0;
        cudaRuntimeGetVersion(&rt);
        v = std::string("plssvm-b200 ") + PLSSVM_VERSION + " sm_100a CUDA-runtime " + std::to_string(rt / 1000) + "." +
            std::to_string((rt % 1000) / 10) + " " + plssvm::nccl_version_string();
    }
    return v.c_str();
}

int plssvm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // extern "C"
