// multi.cu -- single-process multi-GPU (options.num_gpus, SURVEY §8(b) "Multi-GPU: single process,
// num_gpus devices via ncclCommInitAll"; the paper's library drives every device from one call,
// P:418-426).  One host thread per rank, each running the same row-sharded driver (driver.cu) as a
// one-process-per-GPU rank would, with a communicator of this call:
//   NCCL  ncclCommInitAll over the devices (distinct devices)
//   PEER  the peer-memory transport of comm.cu (all-gather of p fused into the CG update kernel);
//         ranks may share a device (the one-GPU tests run P = 2, 3 ranks this way).
// Training: rank 0 (on options.device) writes alpha and b; predict: the test points are split.
// Any rank's failure aborts the others (barrier flag / ncclCommAbort) and is reported once.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "driver.h"

namespace plssvm {

int resolve_num_gpus(const plssvm_options_t &o) {
    if (o.num_gpus > 0) return o.num_gpus;
    if (const char *e = std::getenv("PLSSVM_NUM_GPUS")) {
        const int v = std::atoi(e);
        if (v >= 1) return v;
    }
    return 1;
}

namespace {

// Device buffer on a given device, freed at scope exit.
struct DevBuf {
    void *p = nullptr;
    int dev = 0;
    void *alloc(int device, size_t bytes) {
        dev = device;
        PLS_CUDA(cudaSetDevice(device));
        PLS_CUDA(cudaMalloc(&p, bytes > 0 ? bytes : 1));
        return p;
    }
    ~DevBuf() {
        if (p) {
            cudaSetDevice(dev);
            cudaFree(p);
        }
    }
};

// The communicators of one call.
struct Ranks {
    int P = 0, kind = COMM_PEER;
    std::vector<int> dev;
    PeerGroup peer;
    std::vector<CommHandle> h;
    std::vector<ncclComm_t> nccl;
    std::atomic<bool> failed{false};

    Ranks(int P_, const plssvm_options_t &o) : P(P_) {
        int ndev = 0;
        PLS_CUDA(cudaGetDeviceCount(&ndev));
        dev.resize(P);
        for (int r = 0; r < P; ++r) dev[r] = (o.device + r) % ndev;
        const bool distinct = P <= ndev;
        if (o.transport == PLSSVM_TRANSPORT_NCCL && !distinct)
            throw Error(PLSSVM_E_INVALID_ARG, "transport NCCL needs num_gpus <= the visible device count (" +
                                                  std::to_string(ndev) + ")");
        kind = (o.transport == PLSSVM_TRANSPORT_PEER || (o.transport == PLSSVM_TRANSPORT_AUTO && !distinct)) ? COMM_PEER
                                                                                                          : COMM_NCCL;
        h.resize(P);
        for (int r = 0; r < P; ++r) {
            h[r].kind = kind;
            h[r].rank = r;
            h[r].nranks = P;
            h[r].device = dev[r];
        }
        if (kind == COMM_NCCL) {
            comm_nccl_init_all(dev, nccl);
            for (int r = 0; r < P; ++r) h[r].nccl = nccl[r];
            return;
        }
        peer.P = P;
        peer.dev = dev;
        peer.ready.assign(P, nullptr);
        peer.done.assign(P, nullptr);
        peer.ptr.assign(P, nullptr);
        peer.stage.assign(P, nullptr);
        peer.stage_bytes.assign(P, 0);
        bool direct = true;
        for (int r = 0; r < P; ++r) {
            PLS_CUDA(cudaSetDevice(dev[r]));
            PLS_CUDA(cudaEventCreateWithFlags(&peer.ready[r], cudaEventDisableTiming));
            PLS_CUDA(cudaEventCreateWithFlags(&peer.done[r], cudaEventDisableTiming));
            for (int q = 0; q < P; ++q) {
                if (dev[q] == dev[r]) continue;
                int can = 0;
                PLS_CUDA(cudaDeviceCanAccessPeer(&can, dev[r], dev[q]));
                if (!can) {
                    direct = false;
                    continue;
                }
                const cudaError_t e = cudaDeviceEnablePeerAccess(dev[q], 0);  // NVLink P2P loads / stores
                if (e == cudaErrorPeerAccessAlreadyEnabled)
                    cudaGetLastError();
                else
                    PLS_CUDA(e);
            }
        }
        peer.direct = direct;
        for (int r = 0; r < P; ++r) h[r].group = &peer;
    }
    ~Ranks() {
        for (int r = 0; r < static_cast<int>(nccl.size()); ++r) {
            cudaSetDevice(dev[r]);
            if (failed.load())
                comm_nccl_abort(nccl[r]);
            else
                comm_nccl_destroy(nccl[r]);
        }
        for (int r = 0; r < static_cast<int>(peer.ready.size()); ++r) {
            cudaSetDevice(dev[r]);
            if (peer.stage[r]) cudaFree(peer.stage[r]);  // stream-ordered allocation; the streams are idle
            if (peer.ready[r]) cudaEventDestroy(peer.ready[r]);
            if (peer.done[r]) cudaEventDestroy(peer.done[r]);
        }
    }
    // First failure wins; the other ranks are released from their collectives.
    void fail() {
        if (failed.exchange(true)) return;
        if (kind == COMM_PEER)
            peer.abort();
        else
            for (int r = 0; r < P; ++r) comm_nccl_abort(nccl[r]), nccl[r] = nullptr;
    }
};

struct RankResult {
    int status = PLSSVM_OK;
    int err_code = 0;
    std::string err;
    bool aborted = false;  // failed only because another rank did
};

// Runs body(r) on P threads; rethrows the root-cause error, else returns the statuses.
template <typename F>
std::vector<RankResult> run_ranks(Ranks &R, F body) {
    std::vector<RankResult> res(R.P);
    std::vector<std::thread> th;
    for (int r = 0; r < R.P; ++r)
        th.emplace_back([&, r] {
            try {
                PLS_CUDA(cudaSetDevice(R.dev[r]));
                res[r].status = body(r);
            } catch (const Error &e) {
                res[r].aborted = R.failed.load();
                res[r].err_code = e.code;
                res[r].err = e.what();
                R.fail();
            } catch (const std::exception &e) {
                res[r].aborted = R.failed.load();
                res[r].err_code = PLSSVM_E_CUDA;
                res[r].err = e.what();
                R.fail();
            }
        });
    for (auto &t : th) t.join();
    int first = -1;
    for (int r = 0; r < R.P; ++r)
        if (res[r].err_code && (first < 0 || (res[first].aborted && !res[r].aborted))) first = r;
    if (first >= 0)
        throw Error(res[first].err_code, "rank " + std::to_string(first) + " (device " + std::to_string(R.dev[first]) +
                                             "): " + res[first].err);
    return res;
}

// The caller's device buffer `src` (on device `from`) as seen by a rank on device `to`: the pointer
// itself on the same device, else a copy.
const void *rank_input(DevBuf &keep, const void *src, size_t bytes, int from, int to) {
    if (from == to || bytes == 0) return src;
    void *d = keep.alloc(to, bytes);
    PLS_CUDA(cudaMemcpyPeer(d, to, src, from, bytes));
    return d;
}

}  // namespace

// Device-pointer inputs may still be written by work on the caller's stream: finish it before other
// devices copy them (the ranks run on their own streams).
void settle_caller_stream(const plssvm_options_t &o) {
    if (!o.device_pointers || !o.stream) return;
    PLS_CUDA(cudaSetDevice(o.device));
    PLS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(o.stream)));
}

int train_multi(const Problem &pb, const plssvm_options_t &o, int P, void *alpha, void *b, plssvm_stats_t *st) {
    settle_caller_stream(o);
    Ranks R(P, o);
    const size_t es = pb.dtype == PLSSVM_F32 ? 4 : 8;
    std::vector<plssvm_stats_t> stats(P);
    auto res = run_ranks(R, [&](int r) {
        plssvm_options_t orr = o;
        orr.device = R.dev[r];
        orr.num_gpus = 1;
        orr.comm = &R.h[r];
        orr.stream = r == 0 ? o.stream : nullptr;
        if (r != 0) orr.residual_trace = nullptr;  // (the scalars are global: rank 0 writes the trace)
        Problem pr = pb;
        DevBuf kx, ky, ka, kb;
        std::vector<char> ha, hb;
        void *a_out = alpha, *b_out = b;
        if (o.device_pointers) {
            pr.X = rank_input(kx, pb.X, static_cast<size_t>(pb.m * pb.d) * es, o.device, R.dev[r]);
            pr.y = rank_input(ky, pb.y, static_cast<size_t>(pb.m) * es, o.device, R.dev[r]);
            PLS_CUDA(cudaSetDevice(R.dev[r]));
            if (r != 0) {
                a_out = ka.alloc(R.dev[r], static_cast<size_t>(pb.m) * es);
                b_out = kb.alloc(R.dev[r], es);
            }
        } else if (r != 0) {
            ha.resize(static_cast<size_t>(pb.m) * es);
            hb.resize(es);
            a_out = ha.data();
            b_out = hb.data();
        }
        PLS_CUDA(cudaSetDevice(R.dev[r]));
        return train(pr, orr, a_out, b_out, &stats[r]);
    });
    if (st) {
        *st = stats[0];
        st->transport_used = R.kind == COMM_NCCL ? PLSSVM_TRANSPORT_NCCL : PLSSVM_TRANSPORT_PEER;
        for (int r = 1; r < P; ++r) {  // the call's time is the slowest rank's
            st->t_total = std::max(st->t_total, stats[r].t_total);
            st->bytes_per_gpu = std::max(st->bytes_per_gpu, stats[r].bytes_per_gpu);
        }
    }
    return res[0].status;
}

int predict_multi(const Problem &pb, const void *alpha, double b, const void *Z, int64_t n, const plssvm_options_t &o,
                  int P, void *decision, int32_t *labels, double *t_kernel) {
    settle_caller_stream(o);
    Ranks R(P, o);
    const size_t es = pb.dtype == PLSSVM_F32 ? 4 : 8;
    std::vector<double> tk(2 * P, 0.0);
    run_ranks(R, [&](int r) {
        const int64_t z0 = n * r / P, z1 = n * (r + 1) / P, nr = z1 - z0;
        if (nr == 0) return static_cast<int>(PLSSVM_OK);
        plssvm_options_t orr = o;
        orr.device = R.dev[r];
        orr.num_gpus = 1;
        orr.comm = nullptr;
        orr.stream = r == 0 ? o.stream : nullptr;
        Problem pr = pb;
        const char *Zr = static_cast<const char *>(Z) + static_cast<size_t>(z0 * pb.d) * es;
        void *dec = decision ? static_cast<char *>(decision) + static_cast<size_t>(z0) * es : nullptr;
        int32_t *lab = labels ? labels + z0 : nullptr;
        DevBuf kx, ka, kz, kd, kl;
        const void *al = alpha;
        const bool other = o.device_pointers && R.dev[r] != o.device;
        if (other) {
            pr.X = rank_input(kx, pb.X, static_cast<size_t>(pb.m * pb.d) * es, o.device, R.dev[r]);
            al = rank_input(ka, alpha, static_cast<size_t>(pb.m) * es, o.device, R.dev[r]);
            Zr = static_cast<const char *>(rank_input(kz, Zr, static_cast<size_t>(nr * pb.d) * es, o.device, R.dev[r]));
            if (dec) dec = kd.alloc(R.dev[r], static_cast<size_t>(nr) * es);
            if (lab) lab = static_cast<int32_t *>(kl.alloc(R.dev[r], static_cast<size_t>(nr) * sizeof(int32_t)));
        }
        PLS_CUDA(cudaSetDevice(R.dev[r]));
        const int s = predict(pr, al, b, Zr, nr, orr, dec, lab, &tk[2 * r]);
        if (other) {  // results back to the caller's device
            if (dec)
                PLS_CUDA(cudaMemcpyPeer(static_cast<char *>(decision) + static_cast<size_t>(z0) * es, o.device, dec,
                                        R.dev[r], static_cast<size_t>(nr) * es));
            if (lab) PLS_CUDA(cudaMemcpyPeer(labels + z0, o.device, lab, R.dev[r], static_cast<size_t>(nr) * sizeof(int32_t)));
        }
        return s;
    });
    if (t_kernel) {
        t_kernel[0] = t_kernel[1] = 0.0;
        for (int r = 0; r < P; ++r) {
            t_kernel[0] = std::max(t_kernel[0], tk[2 * r]);
            t_kernel[1] += tk[2 * r + 1];
        }
    }
    return PLSSVM_OK;
}

}  // namespace plssvm
