// comm.cu -- NCCL plumbing for the row-sharded multi-GPU mode (one process per GPU).
// Per CG iteration: all-gather of the p shards and sum all-reduces of the CG scalars
// (north_star; the paper sums per-device vectors through the host).
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

#include "common.cuh"
#include "driver.h"

namespace plssvm {

struct CommHandle {
    ncclComm_t nccl;
    int rank, nranks, device;
    bool callbacks;
    plssvm_comm_callbacks_t cb;
};

#define PLS_NCCL(call)                                                                                \
    do {                                                                                              \
        ncclResult_t r_ = (call);                                                                     \
        if (r_ != ncclSuccess) throw ::plssvm::Error(5, std::string(#call) + " -> " + ncclGetErrorString(r_)); \
    } while (0)

int comm_rank(const CommHandle *c) { return c->rank; }
int comm_size(const CommHandle *c) { return c->nranks; }
int comm_device(const CommHandle *c) { return c->device; }

// Out-of-place sum all-reduce (send: this rank's partials, recv: the global values).
void comm_allreduce_sum_f64(CommHandle *c, const double *send, double *recv, int64_t count, void *stream) {
    if (c->callbacks) {  // the user callback is in place: stage the partials in recv first
        PLS_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice,
                                 static_cast<cudaStream_t>(stream)));
        if (c->cb.allreduce_sum_f64(c->cb.ctx, recv, count, stream) != 0)
            throw Error(PLSSVM_E_NCCL, "user allreduce callback failed");
        return;
    }
    PLS_NCCL(ncclAllReduce(send, recv, static_cast<size_t>(count), ncclDouble, ncclSum, c->nccl,
                           static_cast<cudaStream_t>(stream)));
}

// In-place all-gather: rank r's shard lives at buf + r * count_per_rank.
void comm_allgather(CommHandle *c, void *buf, int64_t count_per_rank, int dtype, void *stream) {
    if (c->callbacks) {
        if (c->cb.allgather(c->cb.ctx, buf, count_per_rank, dtype, stream) != 0)
            throw Error(PLSSVM_E_NCCL, "user allgather callback failed");
        return;
    }
    const size_t es = dtype == PLSSVM_F32 ? 4 : 8;
    char *b = static_cast<char *>(buf);
    PLS_NCCL(ncclAllGather(b + static_cast<size_t>(c->rank) * count_per_rank * es, b,
                           static_cast<size_t>(count_per_rank), dtype == PLSSVM_F32 ? ncclFloat : ncclDouble, c->nccl,
                           static_cast<cudaStream_t>(stream)));
}

bool comm_has_reduce_scatter(const CommHandle *c) { return !c->callbacks || c->cb.reduce_scatter_sum != nullptr; }

// recv[count_per_rank] <- this rank's block of sum over ranks of send[nranks * count_per_rank].
void comm_reduce_scatter(CommHandle *c, const void *send, void *recv, int64_t count_per_rank, int dtype, void *stream) {
    if (c->callbacks) {
        if (!c->cb.reduce_scatter_sum || c->cb.reduce_scatter_sum(c->cb.ctx, send, recv, count_per_rank, dtype, stream) != 0)
            throw Error(PLSSVM_E_NCCL, "user reduce_scatter callback failed");
        return;
    }
    PLS_NCCL(ncclReduceScatter(send, recv, static_cast<size_t>(count_per_rank), dtype == PLSSVM_F32 ? ncclFloat : ncclDouble,
                               ncclSum, c->nccl, static_cast<cudaStream_t>(stream)));
}

const char *nccl_version_string() {
    static std::string v;
    if (v.empty()) {
        int code = 0;
        ncclGetVersion(&code);
        v = "NCCL " + std::to_string(code / 10000) + "." + std::to_string((code / 100) % 100) + "." +
            std::to_string(code % 100);
    }
    return v.c_str();
}

}  // namespace plssvm

using plssvm::CommHandle;

extern "C" int plssvm_comm_unique_id_impl(void *id128) {
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return PLSSVM_E_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    memcpy(id128, &id, sizeof(id));
    return PLSSVM_OK;
}

extern "C" int plssvm_comm_init_impl(const void *id128, int32_t nranks, int32_t rank, int32_t device, void **out) {
    if (cudaSetDevice(device) != cudaSuccess) return PLSSVM_E_CUDA;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    auto *h = new CommHandle{nullptr, rank, nranks, device, false, {}};
    ncclResult_t r = ncclCommInitRank(&h->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        delete h;
        return PLSSVM_E_NCCL;
    }
    *out = h;
    return PLSSVM_OK;
}

extern "C" int plssvm_comm_init_callbacks_impl(const plssvm_comm_callbacks_t *cb, int32_t nranks, int32_t rank,
                                               int32_t device, void **out) {
    *out = new CommHandle{nullptr, rank, nranks, device, true, *cb};
    return PLSSVM_OK;
}

extern "C" int plssvm_comm_destroy_impl(void *c) {
    auto *h = static_cast<CommHandle *>(c);
    if (!h) return PLSSVM_OK;
    if (!h->callbacks) ncclCommDestroy(h->nccl);
    delete h;
    return PLSSVM_OK;
}
