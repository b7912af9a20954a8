// driver.h -- internal (C++) interface between the C ABI (capi.cu) and the device driver.
#pragma once
#include <nccl.h>

#include <cstdint>
#include <vector>
#include "../../include/plssvm.h"

struct ncclDevComm;  // nccl_device.h

namespace plssvm {

struct Problem {
    const void *X;
    const void *y;
    int64_t m, d;
    int dtype;
    int kernel;
    double gamma;
    int degree;
    double coef0;
    double C;
    double eps;
};

struct CommHandle;  // comm.cu

// Feature split of PLSSVM_MULTI_GPU_FEATURES: rank r owns features [feature_begin(r), feature_begin(r+1)).
inline int64_t feature_begin(int64_t d, int nranks, int rank) { return d * rank / nranks; }

// Each returns a plssvm_status_t and throws plssvm::Error for CUDA / NCCL failures.
int train(const Problem &pb, const plssvm_options_t &o, void *alpha, void *b, plssvm_stats_t *st);
int predict(const Problem &pb, const void *alpha, double b, const void *Z, int64_t n, const plssvm_options_t &o,
            void *decision, int32_t *labels, double *t_kernel);
int qtilde_matvec(const Problem &pb, const void *p, int32_t repeats, const plssvm_options_t &o, void *out,
                  double *t_kernel);

#ifdef PLSSVM_OZ_EXPERIMENTS
int exp_oz_profile(unsigned long long *out, int reset);
#endif

// multi.cu: the num_gpus mode (one host thread per device, NCCL or PEER transport)
int resolve_num_gpus(const plssvm_options_t &o);
int train_multi(const Problem &pb, const plssvm_options_t &o, int P, void *alpha, void *b, plssvm_stats_t *st);
int predict_multi(const Problem &pb, const void *alpha, double b, const void *Z, int64_t n, const plssvm_options_t &o,
                  int P, void *decision, int32_t *labels, double *t_kernel);

// comm.cu
int comm_rank(const CommHandle *c);
int comm_size(const CommHandle *c);
int comm_device(const CommHandle *c);
bool comm_is_peer(const CommHandle *c);
bool comm_peer_direct(const CommHandle *c);
void comm_peer_fence(CommHandle *c, void *stream);
std::vector<void *> comm_peer_exchange_ptr(CommHandle *c, void *ptr);
void comm_allreduce_sum_f64(CommHandle *c, const double *send, double *recv, int64_t count, void *stream);
void comm_allgather(CommHandle *c, void *buf, int64_t count_per_rank, int dtype, void *stream);
bool comm_has_reduce_scatter(const CommHandle *c);
void comm_reduce_scatter(CommHandle *c, const void *send, void *recv, int64_t count_per_rank, int dtype, void *stream);
const char *nccl_version_string();
// NCCL device API (LSA: load/store-accessible peers) for the fused all-gather of p: a symmetric window
// of at least `bytes` registered on the communicator (collective; grown on demand) and the device
// communicator with one LSA barrier per vector-kernel block.  nullptr when the transport is not NCCL,
// not every rank is load/store accessible (no NVLink path) or PLSSVM_NO_LSA is set.
void *comm_lsa_buffer(CommHandle *c, size_t bytes);
ncclWindow_t comm_lsa_window(const CommHandle *c);
const ncclDevComm *comm_lsa_devcomm(const CommHandle *c);
void comm_lsa_destroy(CommHandle *c);

}  // namespace plssvm
