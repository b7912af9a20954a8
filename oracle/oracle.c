/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the PLSSVM LS-SVM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2202_12674_b200/) never includes, links or calls anything here, and this file
 * shares no code, header, table or helper with the CUDA path.
 *
 * Citations: P:L = /root/reference/PAPER.md line L; S:L = SPEC.md line L.
 * Every quantity is fp64 (the paper's precision).  fp32 configs feed this oracle the
 * fp32-rounded inputs upcast to fp64 (reading R-12).
 * Data layout: X is point-major, X[i*d + k] = feature k of point i (plain C array).
 * Summation order: the natural sequential loop order, no blocking, no reassociation.
 * OpenMP is used only to run independent rows (outer loops) in parallel; each row's sum
 * is sequential, so results are bitwise independent of the thread count.
 *
 * Pins (tests/test_oracle_pins.py): worked examples with exact rationals (S:230-291 and
 * DESIGN.md), dense LU solve of the full KKT system Eq. 11, Cholesky of Q~ (SPD),
 * Q~ = B^T Q B, ridge closed form for the linear kernel, CG special cases, invariants.
 * Parity unpinned: none of the functions below (each is pinned by at least one test).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define OR_LINEAR 0
#define OR_POLYNOMIAL 1
#define OR_RBF 2

#define OR_OK 0
#define OR_E_INVALID 1
#define OR_E_NUMERICAL 6
#define OR_W_NOT_CONVERGED 7

/* Kernel functions, P:244-250 (§II-E table):
 *   linear      <x_i, x_j>
 *   polynomial  (gamma <x_i, x_j> + r)^d      gamma > 0, d integer (repeated multiplication)
 *   radial      exp(-gamma ||x_i - x_j||^2)   gamma > 0 (squared distance summed directly)
 */
double oracle_kernel(const double *a, const double *b, int64_t d, int kernel, double gamma,
                     int degree, double coef0) {
    if (kernel == OR_LINEAR) {
        double s = 0.0;
        for (int64_t k = 0; k < d; ++k) s += a[k] * b[k];
        return s;
    } else if (kernel == OR_POLYNOMIAL) {
        double s = 0.0;
        for (int64_t k = 0; k < d; ++k) s += a[k] * b[k];
        double base = gamma * s + coef0, r = 1.0;
        for (int t = 0; t < degree; ++t) r *= base;
        return r;
    } else {
        double s = 0.0;
        for (int64_t k = 0; k < d; ++k) {
            double t = a[k] - b[k];
            s += t * t;
        }
        return exp(-gamma * s);
    }
}

/* q cache, P:391-395 (§III-C2) and Eq. 12: x_m is the LAST point (index m-1,
 * DESIGN.md reading R-4).  q_i = k(x_i, x_m) for i < m-1;  Q_mm = k(x_m, x_m) + 1/C. */
void oracle_q(const double *X, int64_t m, int64_t d, int kernel, double gamma, int degree,
              double coef0, double C, double *q, double *Qmm) {
    const double *xm = X + (m - 1) * d;
    for (int64_t i = 0; i < m - 1; ++i) q[i] = oracle_kernel(X + i * d, xm, d, kernel, gamma, degree, coef0);
    *Qmm = oracle_kernel(xm, xm, d, kernel, gamma, degree, coef0) + 1.0 / C;
}

/* One entry of the reduced matrix, Eq. 16:
 *   Q~_ij = k(x_i,x_j) + delta_ij/C - k(x_m,x_j) - k(x_i,x_m) + k(x_m,x_m) + 1/C
 * with the cached q and Q_mm = k(x_m,x_m) + 1/C (reading R-1: the trailing 1/C
 * belongs to Q_mm, Eq. 12/13 P:278-290). */
static double qtilde_entry(const double *X, int64_t d, int kernel, double gamma, int degree,
                           double coef0, double C, const double *q, double Qmm, int64_t i, int64_t j) {
    double kij = oracle_kernel(X + i * d, X + j * d, d, kernel, gamma, degree, coef0);
    double v = kij + (i == j ? 1.0 / C : 0.0) - q[j] - q[i] + Qmm;
    return v;
}

/* Explicit dense Q~ (m-1) x (m-1), row-major.  Eq. 13 entry-wise via Eq. 16. */
void oracle_qtilde(const double *X, int64_t m, int64_t d, int kernel, double gamma, int degree,
                   double coef0, double C, double *Qt) {
    int64_t n = m - 1;
    double *q = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double Qmm;
    oracle_q(X, m, d, kernel, gamma, degree, coef0, C, q, &Qmm);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j)
            Qt[i * n + j] = qtilde_entry(X, d, kernel, gamma, degree, coef0, C, q, Qmm, i, j);
    free(q);
}

/* Selected rows of Q~ (for sampled parity at full size without forming all of Q~). */
void oracle_qtilde_rows(const double *X, int64_t m, int64_t d, int kernel, double gamma, int degree,
                        double coef0, double C, const int64_t *rows, int64_t nrows, double *out) {
    int64_t n = m - 1;
    double *q = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double Qmm;
    oracle_q(X, m, d, kernel, gamma, degree, coef0, C, q, &Qmm);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < nrows; ++r)
        for (int64_t j = 0; j < n; ++j)
            out[r * n + j] = qtilde_entry(X, d, kernel, gamma, degree, coef0, C, q, Qmm, rows[r], j);
    free(q);
}

/* y = A p for a dense row-major n x n matrix (plain row-by-row dot products). */
void oracle_matvec(const double *A, int64_t n, const double *p, double *y) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += A[i * n + j] * p[j];
        y[i] = s;
    }
}

static double dot(const double *a, const double *b, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* Conjugate gradients on the reduced system, P:351-356 ("a variant of Shewchuk"), following
 * Shewchuk 1994 App. B2 in its order and notation (reading R-5):
 *   i=0; r=b-Ax; d=r; delta_new=r.r; delta_0=delta_new
 *   while i<imax and delta_new > eps^2 delta_0:
 *       q=Ad; alpha=delta_new/(d.q); x=x+alpha d
 *       if replace_every>0 and i>0 and i%replace_every==0: r=b-Ax  else: r=r-alpha q
 *       delta_old=delta_new; delta_new=r.r; beta=delta_new/delta_old; d=r+beta d; i++
 * x holds x0 on entry (ZERO by default).  d.q <= 0 or non-finite -> OR_E_NUMERICAL.
 * Stagnation guard (SURVEY.md §5 "failure detection" and App. A.7; reading R-20),
 * active only when replace_every = R > 0: delta_best starts at delta_0; after iteration i, a
 * delta_new < delta_best / 4 makes delta_best = delta_new and i_best = i; otherwise, once
 * i - i_best >= W = 2 max(R, 50), the loop stops with OR_W_NOT_CONVERGED (replacement makes the
 * recurrence oscillate instead of converging at high condition numbers, App. A.2/A.7).  SURVEY
 * states the window as 2R for Shewchuk's R = 50; the floor of 100 keeps small R from firing on
 * CG's ordinary plateaus (several iterations without a 4x drop are normal).
 * trace (nullable, length imax+1) receives sqrt(delta) per iteration. */
int oracle_cg(const double *A, int64_t n, const double *b, double *x, double eps, int64_t imax,
              int64_t replace_every, int64_t *iters_out, double *trace) {
    double *r = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *dd = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *qv = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int status = OR_OK;
    oracle_matvec(A, n, x, qv);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - qv[k];
    memcpy(dd, r, sizeof(double) * (size_t)n);
    double delta_new = dot(r, r, n), delta0 = delta_new;
    double delta_best = delta0;
    int64_t i = 0, i_best = 0;
    int stagnated = 0;
    if (trace) trace[0] = sqrt(delta_new);
    while (i < imax && delta_new > eps * eps * delta0) {
        oracle_matvec(A, n, dd, qv);
        double dq = dot(dd, qv, n);
        if (!(dq > 0.0) || !isfinite(dq)) { status = OR_E_NUMERICAL; break; }
        double alpha = delta_new / dq;
        for (int64_t k = 0; k < n; ++k) x[k] += alpha * dd[k];
        if (replace_every > 0 && i > 0 && i % replace_every == 0) {
            oracle_matvec(A, n, x, qv);
            for (int64_t k = 0; k < n; ++k) r[k] = b[k] - qv[k];
        } else {
            for (int64_t k = 0; k < n; ++k) r[k] -= alpha * qv[k];
        }
        double delta_old = delta_new;
        delta_new = dot(r, r, n);
        if (!isfinite(delta_new)) { status = OR_E_NUMERICAL; break; }
        double beta = delta_new / delta_old;
        for (int64_t k = 0; k < n; ++k) dd[k] = r[k] + beta * dd[k];
        ++i;
        if (trace) trace[i] = sqrt(delta_new);
        if (replace_every > 0) {
            if (delta_new < 0.25 * delta_best) {
                delta_best = delta_new;
                i_best = i;
            } else if (i - i_best >= 2 * (replace_every > 50 ? replace_every : 50) &&
                       delta_new > eps * eps * delta0) {
                stagnated = 1;
                break;
            }
        }
    }
    if (status == OR_OK && (stagnated || delta_new > eps * eps * delta0)) status = OR_W_NOT_CONVERGED;
    *iters_out = i;
    free(r); free(dd); free(qv);
    return status;
}

/* Full training: Eq. 14 rhs, CG on the explicit Q~, Eq. 15 bias, alpha assembly.
 *   rhs_i = y_i - y_m                                   (Eq. 14)
 *   b = y_m + Q_mm <1, a~> - <q, a~>                     (Eq. 15)
 *   alpha = (a~_0 .. a~_{m-2}, -sum a~)                  (last row of Eq. 11: 1^T alpha = 0)
 * x0_mode: 0 = zeros, 1 = ones.  imax <= 0 means m-1.
 * timings (nullable, 3 doubles): seconds for Q~ formation, CG, total (plain wall clock). */
static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int oracle_train(const double *X, const double *y, int64_t m, int64_t d, int kernel, double gamma,
                 int degree, double coef0, double C, double eps, int64_t imax, int x0_mode,
                 int64_t replace_every, double *alpha, double *b, int64_t *iters, double *timings) {
    if (m < 2 || d < 1 || !(C > 0)) return OR_E_INVALID;
    double t0 = now_s();
    int64_t n = m - 1;
    double *Qt = (double *)malloc(sizeof(double) * (size_t)n * (size_t)n);
    double *q = (double *)malloc(sizeof(double) * (size_t)n);
    double *rhs = (double *)malloc(sizeof(double) * (size_t)n);
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    if (!Qt || !q || !rhs || !x) { free(Qt); free(q); free(rhs); free(x); return OR_E_INVALID; }
    double Qmm;
    oracle_q(X, m, d, kernel, gamma, degree, coef0, C, q, &Qmm);
    oracle_qtilde(X, m, d, kernel, gamma, degree, coef0, C, Qt);
    double t1 = now_s();
    double ym = y[m - 1];
    for (int64_t i = 0; i < n; ++i) rhs[i] = y[i] - ym;
    for (int64_t i = 0; i < n; ++i) x[i] = (x0_mode == 1) ? 1.0 : 0.0;
    if (imax <= 0) imax = n;
    int st = oracle_cg(Qt, n, rhs, x, eps, imax, replace_every, iters, NULL);
    double t2 = now_s();
    double sx = 0.0, qx = 0.0;
    for (int64_t i = 0; i < n; ++i) sx += x[i];
    for (int64_t i = 0; i < n; ++i) qx += q[i] * x[i];
    *b = ym + Qmm * sx - qx;
    for (int64_t i = 0; i < n; ++i) alpha[i] = x[i];
    alpha[n] = -sx;
    if (timings) { timings[0] = t1 - t0; timings[1] = t2 - t1; timings[2] = now_s() - t0; }
    free(Qt); free(q); free(rhs); free(x);
    return st;
}

/* Decision function, Eq. 10 with labels absorbed into alpha (R-2):
 *   f(z) = sum_i alpha_i k(x_i, z) + b;   label = +1 if f >= 0 else -1 (sgn(0) -> +1, R-11). */
void oracle_predict(const double *X, const double *alpha, double b, int64_t m, int64_t d, int kernel,
                    double gamma, int degree, double coef0, const double *Z, int64_t n, double *f,
                    int32_t *labels) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t t = 0; t < n; ++t) {
        double s = 0.0;
        for (int64_t i = 0; i < m; ++i) s += alpha[i] * oracle_kernel(X + i * d, Z + t * d, d, kernel, gamma, degree, coef0);
        double v = s + b;
        if (f) f[t] = v;
        if (labels) labels[t] = (v >= 0.0) ? 1 : -1;
    }
}

/* Threads the OpenMP runtime will use (reported as cpu_baseline.cores). */
#ifdef _OPENMP
#include <omp.h>
#endif
int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
