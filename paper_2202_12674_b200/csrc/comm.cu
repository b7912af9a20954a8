// comm.cu -- the exchange step of the row-sharded multi-GPU mode.
// Per CG iteration: all-gather of the p shards, sum all-reduces of the CG scalars and (implicit
// circulant mode) a reduce-scatter of the partial products (north_star; the paper sums per-device
// vectors through the host, and uses no GPU-to-GPU communication).
// Three transports behind one handle:
//   NCCL       one process per GPU (plssvm_comm_init) or one thread per GPU (ncclCommInitAll, the
//              num_gpus mode of multi.cu)
//   CALLBACKS  a caller-supplied transport (MPI, or the host-staged gloo exchange of the tests)
//   PEER       the library's own single-process transport over peer memory: every rank pulls what it
//              needs from the other ranks' device buffers (cudaMemcpyPeerAsync, NVLink P2P) and sums in
//              rank order -- deterministic and identical on every rank; cross-device ordering by CUDA
//              events, host threads meet at an enqueue barrier.  The all-gather of p is fused into the
//              CG update kernel (direct peer stores, driver.cu); ranks may share a device.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "driver.h"

namespace plssvm {

#define PLS_NCCL(call)                                                                                \
    do {                                                                                              \
        ncclResult_t r_ = (call);                                                                     \
        if (r_ != ncclSuccess) throw ::plssvm::Error(5, std::string(#call) + " -> " + ncclGetErrorString(r_)); \
    } while (0)

int comm_rank(const CommHandle *c) { return c->rank; }
int comm_size(const CommHandle *c) { return c->nranks; }
int comm_device(const CommHandle *c) { return c->device; }
bool comm_is_peer(const CommHandle *c) { return c->kind == COMM_PEER; }

// ---- PEER transport --------------------------------------------------------------------------
void PeerGroup::barrier() {
    const uint64_t g = gen.load(std::memory_order_acquire);
    if (arrived.fetch_add(1, std::memory_order_acq_rel) == P - 1) {
        arrived.store(0, std::memory_order_relaxed);
        gen.fetch_add(1, std::memory_order_acq_rel);
    } else {
        int spins = 0;
        while (gen.load(std::memory_order_acquire) == g) {
            if (aborted.load(std::memory_order_acquire))
                throw Error(PLSSVM_E_NCCL, "multi-GPU call aborted: another rank failed");
            if (++spins > 64) std::this_thread::yield();
        }
    }
    if (aborted.load(std::memory_order_acquire)) throw Error(PLSSVM_E_NCCL, "multi-GPU call aborted: another rank failed");
}

void PeerGroup::abort() { aborted.store(true, std::memory_order_release); }

namespace {

// recv[k] = sum_q stage[q * count + k] in rank order (every rank sums the same values in the same
// order, so the all-reduced scalars are bitwise identical on all ranks).
template <typename T>
__global__ void k_peer_sum(const T *__restrict__ stage, int P, int64_t count, T *__restrict__ recv) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        T s = T(0);
        for (int q = 0; q < P; ++q) s += stage[static_cast<int64_t>(q) * count + k];
        recv[k] = s;
    }
}

void *peer_stage(CommHandle *c, size_t bytes, cudaStream_t s) {
    PeerGroup *G = c->group;
    const int r = c->rank;
    if (G->stage_bytes[r] < bytes) {
        if (G->stage[r]) PLS_CUDA(cudaFreeAsync(G->stage[r], s));
        G->stage[r] = nullptr;
        PLS_CUDA(cudaMallocAsync(&G->stage[r], bytes, s));
        G->stage_bytes[r] = bytes;
    }
    return G->stage[r];
}

// Phase 1: publish `ptr`, mark this rank's data ready on its stream, meet the others, and make this
// stream wait for every rank's data.
void peer_ready(CommHandle *c, const void *ptr, cudaStream_t s) {
    PeerGroup *G = c->group;
    G->ptr[c->rank] = ptr;
    PLS_CUDA(cudaEventRecord(G->ready[c->rank], s));
    G->barrier();
    for (int q = 0; q < G->P; ++q)
        if (q != c->rank) PLS_CUDA(cudaStreamWaitEvent(s, G->ready[q], 0));
}
// Phase 2: every rank has finished reading the others' buffers before anyone writes them again.
void peer_done(CommHandle *c, cudaStream_t s) {
    PeerGroup *G = c->group;
    PLS_CUDA(cudaEventRecord(G->done[c->rank], s));
    G->barrier();
    for (int q = 0; q < G->P; ++q)
        if (q != c->rank) PLS_CUDA(cudaStreamWaitEvent(s, G->done[q], 0));
}

template <typename T>
void peer_sum_launch(const void *stage, int P, int64_t count, void *recv, cudaStream_t s) {
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(count, 256), 4 * 148));
    k_peer_sum<T><<<std::max(1u, blocks), 256, 0, s>>>(static_cast<const T *>(stage), P, count, static_cast<T *>(recv));
    PLS_CHECK_LAUNCH();
}

void peer_allreduce(CommHandle *c, const double *send, double *recv, int64_t count, cudaStream_t s) {
    PeerGroup *G = c->group;
    const size_t bytes = static_cast<size_t>(count) * sizeof(double);
    char *st = static_cast<char *>(peer_stage(c, bytes * G->P, s));
    peer_ready(c, send, s);
    for (int q = 0; q < G->P; ++q)
        PLS_CUDA(cudaMemcpyPeerAsync(st + q * bytes, c->device, G->ptr[q], G->dev[q], bytes, s));
    peer_done(c, s);  // nobody overwrites a send buffer (in place: recv) before all copies are done
    peer_sum_launch<double>(st, G->P, count, recv, s);
}

void peer_allgather(CommHandle *c, void *buf, int64_t count_per_rank, size_t es, cudaStream_t s) {
    PeerGroup *G = c->group;
    const size_t bytes = static_cast<size_t>(count_per_rank) * es;
    peer_ready(c, buf, s);
    for (int q = 0; q < G->P; ++q)
        if (q != c->rank)
            PLS_CUDA(cudaMemcpyPeerAsync(static_cast<char *>(buf) + q * bytes, c->device,
                                         static_cast<const char *>(G->ptr[q]) + q * bytes, G->dev[q], bytes, s));
    peer_done(c, s);
}

void peer_reduce_scatter(CommHandle *c, const void *send, void *recv, int64_t count, int dtype, cudaStream_t s) {
    PeerGroup *G = c->group;
    const size_t es = dtype == PLSSVM_F32 ? 4 : 8, bytes = static_cast<size_t>(count) * es;
    char *st = static_cast<char *>(peer_stage(c, bytes * G->P, s));
    peer_ready(c, send, s);
    for (int q = 0; q < G->P; ++q)
        PLS_CUDA(cudaMemcpyPeerAsync(st + q * bytes, c->device, static_cast<const char *>(G->ptr[q]) + c->rank * bytes,
                                     G->dev[q], bytes, s));
    peer_done(c, s);
    if (dtype == PLSSVM_F32)
        peer_sum_launch<float>(st, G->P, count, recv, s);
    else
        peer_sum_launch<double>(st, G->P, count, recv, s);
}

}  // namespace

// Fused all-gather (PEER): the p update kernel already stored this rank's band into every rank's p;
// only the cross-device order remains: the next product waits for every rank's update.  (Writes into
// a peer's p happen after that peer's product of the same iteration: the scalar all-reduces between
// them order it.)
void comm_peer_fence(CommHandle *c, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PeerGroup *G = c->group;
    PLS_CUDA(cudaEventRecord(G->ready[c->rank], s));
    G->barrier();
    for (int q = 0; q < G->P; ++q)
        if (q != c->rank) PLS_CUDA(cudaStreamWaitEvent(s, G->ready[q], 0));
    G->barrier();  // the ready events are re-recorded by the next collective only after everyone waited
}

// Publishes this rank's pointer and returns every rank's (setup of the fused all-gather).
std::vector<void *> comm_peer_exchange_ptr(CommHandle *c, void *ptr) {
    PeerGroup *G = c->group;
    G->ptr[c->rank] = ptr;
    G->barrier();
    std::vector<void *> all(G->P);
    for (int q = 0; q < G->P; ++q) all[q] = const_cast<void *>(G->ptr[q]);
    G->barrier();
    return all;
}
bool comm_peer_direct(const CommHandle *c) { return c->kind == COMM_PEER && c->group->direct; }

// ---- NCCL device API: symmetric window of p (fused all-gather) --------------
// Every rank's full p lives in one NCCL symmetric window (ncclMemAlloc + ncclCommWindowRegister,
// NCCL_WIN_COLL_SYMMETRIC); the p update kernel stores the new band straight into every LSA peer's
// window (ncclGetLsaPointer: NVLink loads/stores) and meets the peers in a per-block LSA barrier
// (kernels.cuh k_update_p_lsa) -- the all-gather of p becomes part of the update kernel.
struct LsaState {
    void *base = nullptr;
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    ncclDevComm dev{};
    bool have_dev = false, failed = false;
};

// Every rank must take the same path (the LSA update replaces a collective): the outcome of this rank's
// setup is agreed by an all-reduce (min) before use.
static bool lsa_agree(CommHandle *c, bool ok) {
    int *d = nullptr;
    int h = ok ? 1 : 0;
    cudaStream_t s = nullptr;
    bool agreed = false;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess && cudaMalloc(&d, sizeof(int)) == cudaSuccess &&
        cudaMemcpyAsync(d, &h, sizeof(int), cudaMemcpyHostToDevice, s) == cudaSuccess &&
        ncclAllReduce(d, d, 1, ncclInt32, ncclMin, c->nccl, s) == ncclSuccess &&
        cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s) == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess)
        agreed = h == 1;
    if (d) cudaFree(d);
    if (s) cudaStreamDestroy(s);
    return agreed;
}

void *comm_lsa_buffer(CommHandle *c, size_t bytes) {
    if (c->kind != COMM_NCCL || !c->lsa_allowed || std::getenv("PLSSVM_NO_LSA")) return nullptr;
    if (!c->lsa) c->lsa = new LsaState{};
    LsaState *L = c->lsa;
    if (L->failed) return nullptr;
    bytes = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    if (L->have_dev && bytes <= L->bytes) return L->base;
    bool ok = true;
    if (!L->have_dev) {
        ncclDevCommRequirements reqs{};
        reqs.lsaBarrierCount = kVecBlocks;  // one barrier per block of the vector kernels
        ok = ncclDevCommCreate(c->nccl, &reqs, &L->dev) == ncclSuccess;
        L->have_dev = ok;
        ok = ok && L->dev.lsaSize == c->nranks;  // a rank without load/store access: NCCL's all-gather
    }
    if (ok) {  // (collective: every rank trains the same problem size)
        if (L->win) ncclCommWindowDeregister(c->nccl, L->win);
        if (L->base) ncclMemFree(L->base);
        L->win = nullptr;
        L->base = nullptr;
        L->bytes = 0;
        ok = ncclMemAlloc(&L->base, bytes) == ncclSuccess &&
             ncclCommWindowRegister(c->nccl, L->base, bytes, &L->win, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess;
        if (ok) L->bytes = bytes;
    }
    if (!lsa_agree(c, ok)) {
        L->failed = true;
        return nullptr;
    }
    return L->base;
}
ncclWindow_t comm_lsa_window(const CommHandle *c) { return c->lsa ? c->lsa->win : nullptr; }
const ncclDevComm *comm_lsa_devcomm(const CommHandle *c) { return c->lsa ? &c->lsa->dev : nullptr; }
void comm_lsa_destroy(CommHandle *c) {
    LsaState *L = c->lsa;
    if (!L) return;
    if (c->nccl) {
        if (L->win) ncclCommWindowDeregister(c->nccl, L->win);
        if (L->base) ncclMemFree(L->base);
        if (L->have_dev) ncclDevCommDestroy(c->nccl, &L->dev);
    }
    delete L;
    c->lsa = nullptr;
}

// ---- dispatch -----------------------------------------------------------------------------------
// Out-of-place sum all-reduce (send: this rank's partials, recv: the global values).
void comm_allreduce_sum_f64(CommHandle *c, const double *send, double *recv, int64_t count, void *stream) {
    if (c->kind == COMM_CALLBACKS) {  // the user callback is in place: stage the partials in recv first
        PLS_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice,
                                 static_cast<cudaStream_t>(stream)));
        if (c->cb.allreduce_sum_f64(c->cb.ctx, recv, count, stream) != 0)
            throw Error(PLSSVM_E_NCCL, "user allreduce callback failed");
        return;
    }
    if (c->kind == COMM_PEER) return peer_allreduce(c, send, recv, count, static_cast<cudaStream_t>(stream));
    PLS_NCCL(ncclAllReduce(send, recv, static_cast<size_t>(count), ncclDouble, ncclSum, c->nccl,
                           static_cast<cudaStream_t>(stream)));
}

// In-place all-gather: rank r's shard lives at buf + r * count_per_rank.
void comm_allgather(CommHandle *c, void *buf, int64_t count_per_rank, int dtype, void *stream) {
    if (c->kind == COMM_CALLBACKS) {
        if (c->cb.allgather(c->cb.ctx, buf, count_per_rank, dtype, stream) != 0)
            throw Error(PLSSVM_E_NCCL, "user allgather callback failed");
        return;
    }
    const size_t es = dtype == PLSSVM_F32 ? 4 : 8;
    if (c->kind == COMM_PEER) return peer_allgather(c, buf, count_per_rank, es, static_cast<cudaStream_t>(stream));
    char *b = static_cast<char *>(buf);
    PLS_NCCL(ncclAllGather(b + static_cast<size_t>(c->rank) * count_per_rank * es, b,
                           static_cast<size_t>(count_per_rank), dtype == PLSSVM_F32 ? ncclFloat : ncclDouble, c->nccl,
                           static_cast<cudaStream_t>(stream)));
}

bool comm_has_reduce_scatter(const CommHandle *c) {
    return c->kind != COMM_CALLBACKS || c->cb.reduce_scatter_sum != nullptr;
}

// recv[count_per_rank] <- this rank's block of sum over ranks of send[nranks * count_per_rank].
void comm_reduce_scatter(CommHandle *c, const void *send, void *recv, int64_t count_per_rank, int dtype, void *stream) {
    if (c->kind == COMM_CALLBACKS) {
        if (!c->cb.reduce_scatter_sum || c->cb.reduce_scatter_sum(c->cb.ctx, send, recv, count_per_rank, dtype, stream) != 0)
            throw Error(PLSSVM_E_NCCL, "user reduce_scatter callback failed");
        return;
    }
    if (c->kind == COMM_PEER)
        return peer_reduce_scatter(c, send, recv, count_per_rank, dtype, static_cast<cudaStream_t>(stream));
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

// ncclCommInitAll over `devs` (single process, one communicator per device; distinct devices).
void comm_nccl_init_all(const std::vector<int> &devs, std::vector<ncclComm_t> &out) {
    out.assign(devs.size(), nullptr);
    PLS_NCCL(ncclCommInitAll(out.data(), static_cast<int>(devs.size()), devs.data()));
}
void comm_nccl_abort(ncclComm_t c) {
    if (c) ncclCommAbort(c);
}
void comm_nccl_destroy(ncclComm_t c) {
    if (c) ncclCommDestroy(c);
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
    auto *h = new CommHandle{};
    h->kind = plssvm::COMM_NCCL;
    h->rank = rank;
    h->nranks = nranks;
    h->device = device;
    h->lsa_allowed = true;
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
    auto *h = new CommHandle{};
    h->kind = plssvm::COMM_CALLBACKS;
    h->rank = rank;
    h->nranks = nranks;
    h->device = device;
    h->cb = *cb;
    *out = h;
    return PLSSVM_OK;
}

extern "C" int plssvm_comm_destroy_impl(void *c) {
    auto *h = static_cast<CommHandle *>(c);
    if (!h) return PLSSVM_OK;
    plssvm::comm_lsa_destroy(h);
    if (h->kind == plssvm::COMM_NCCL && h->nccl) ncclCommDestroy(h->nccl);
    delete h;
    return PLSSVM_OK;
}
