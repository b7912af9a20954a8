// io.h -- internal interface of io.cpp (LIBSVM files, model files, scaling; host only).
// Each function throws plssvm::Error(PLSSVM_E_IO / _E_LABELS / _E_INVALID_ARG, message).
#pragma once
#include <cstdint>

namespace plssvm {
namespace io {

void libsvm_read(const char *path, double *X, double *y, int64_t cap_m, int64_t cap_d, int64_t *m, int64_t *d,
                 double *labels, int32_t *nlabels);
void libsvm_write(const char *path, const double *X, const double *y, int64_t m, int64_t d);
void model_write(const char *path, int kernel, double gamma, int degree, double coef0, const double *X,
                 const double *alpha, double b, int64_t m, int64_t d, const double *y, const double *labels);
void model_read(const char *path, int32_t *kernel, double *gamma, int32_t *degree, double *coef0, double *X,
                double *alpha, double *b, int64_t cap_m, int64_t cap_d, int64_t *m, int64_t *d, double *labels);
void scale_fit(const double *X, int64_t m, int64_t d, double *fmin, double *fmax);
void scale_apply(double *X, int64_t m, int64_t d, const double *fmin, const double *fmax, double lo, double hi);

}  // namespace io
}  // namespace plssvm
