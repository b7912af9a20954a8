// comm.h -- communicator handle of the multi-GPU modes (comm.cu, multi.cu).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstdint>
#include <vector>

#include "../../include/plssvm.h"

namespace plssvm {

enum CommKind : int { COMM_NCCL = 0, COMM_CALLBACKS = 1, COMM_PEER = 2 };

// The ranks of one single-process multi-GPU call (multi.cu): one host thread per rank, each on its
// own stream; collectives meet at a host barrier and order the devices with CUDA events.
struct PeerGroup {
    int P = 0;
    std::vector<int> dev;                 // device of each rank
    std::vector<cudaEvent_t> ready, done;  // per rank, created on the rank's device
    std::vector<const void *> ptr;        // buffer each rank published for the current collective
    std::vector<void *> stage;            // per-rank staging buffer on its device (stream-ordered)
    std::vector<size_t> stage_bytes;
    bool direct = false;                  // every rank can store into every other rank's memory
    std::atomic<int> arrived{0};
    std::atomic<uint64_t> gen{0};
    std::atomic<bool> aborted{false};
    void barrier();  // throws Error(PLSSVM_E_NCCL) when another rank failed
    void abort();
};

struct LsaState;  // comm.cu: NCCL symmetric window of p + device communicator (fused all-gather)

struct CommHandle {
    int kind = COMM_NCCL;
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1, device = 0;
    plssvm_comm_callbacks_t cb{};
    PeerGroup *group = nullptr;  // COMM_PEER
    LsaState *lsa = nullptr;     // COMM_NCCL, created on first use
    bool lsa_allowed = false;    // one process per GPU (plssvm_comm_init): collective window (de)registration
};

void comm_nccl_init_all(const std::vector<int> &devs, std::vector<ncclComm_t> &out);
void comm_nccl_abort(ncclComm_t c);
void comm_nccl_destroy(ncclComm_t c);

}  // namespace plssvm
