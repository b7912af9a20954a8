// driver.cu -- host driver of the hot path: buffers, mode selection, the CG loop, bias.
//
// One call of train<T>() performs, on this process' GPU:
//   a0 stage X to HBM + transform to the padded feature-major layout
//   a1 q cache / norms / Q_mm                                    (Eq. 12)
//   a2 rhs + CG init (x0 = 0: r = p = rhs)                        (Eq. 14)
//   a3 Q~p  implicit tiles (Eq. 16)  or  a3'+a3'' cached precompute + streaming GEMV
//   a4 fused CG updates, a5 convergence test on delta (Shewchuk)
//   a6 bias + alpha (Eq. 15)
//   a8 (row-sharded multi-GPU) NCCL all-gather of p, all-reduce of the CG scalars
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <atomic>
#include <mutex>
#include <vector>

#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include "driver.h"
#include "kernels.cuh"
#include "ozaki_engine.cuh"
#include "tc_engine.cuh"

namespace plssvm {

namespace {

// NVTX range over a phase of a call (SURVEY §5 tracing): visible to nsys / ncu --nvtx when a tool is
// attached, a no-op otherwise (header-only NVTX v3, no link dependency).
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx &) = delete;
    Nvtx &operator=(const Nvtx &) = delete;
};

// ---- stream-ordered device allocations, freed at scope exit -------------------------------
struct Arena {
    cudaStream_t s;
    std::vector<void *> ptrs;
    int64_t bytes = 0;
    explicit Arena(cudaStream_t st) : s(st) {}
    template <typename T>
    T *alloc(int64_t n) {
        void *p = nullptr;
        const size_t sz = std::max<int64_t>(n, 1) * sizeof(T);
        PLS_CUDA(cudaMallocAsync(&p, sz, s));
        ptrs.push_back(p);
        bytes += static_cast<int64_t>(sz);
        return static_cast<T *>(p);
    }
    ~Arena() {
        for (void *p : ptrs) cudaFreeAsync(p, s);
    }
};

// The stream of a call without a user stream: one non-blocking library stream per host thread and
// device, created once.  (Creating, synchronising and destroying a stream in every call cost ~170 us
// of host time per call, while the GPU idled: profiles/r02_host_overhead.txt.)  Calls on one thread
// are sequential and every call synchronises its stream before it returns, so the stream is idle
// between calls.
cudaStream_t library_stream() {
    int dev = 0;
    PLS_CUDA(cudaGetDevice(&dev));
    thread_local struct Pool {
        std::vector<cudaStream_t> s;
        ~Pool() {
            for (cudaStream_t x : s)
                if (x) cudaStreamDestroy(x);
        }
    } pool;
    if (static_cast<int>(pool.s.size()) <= dev) pool.s.resize(dev + 1, nullptr);
    if (!pool.s[dev]) PLS_CUDA(cudaStreamCreateWithFlags(&pool.s[dev], cudaStreamNonBlocking));
    return pool.s[dev];
}

struct StreamGuard {
    cudaStream_t s = nullptr;
    explicit StreamGuard(void *user) : s(user ? static_cast<cudaStream_t>(user) : library_stream()) {}
};

struct Events {
    std::vector<cudaEvent_t> ev;
    cudaEvent_t make() {
        cudaEvent_t e;
        PLS_CUDA(cudaEventCreate(&e));
        ev.push_back(e);
        return e;
    }
    ~Events() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

double elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    PLS_CUDA(cudaEventElapsedTime(&ms, a, b));
    return 1e-3 * ms;
}

// Pinned host buffer for the CG control snapshots, allocated once per host thread and grown on
// demand: cudaMallocHost costs ~1 ms and sat inside every training call's CG phase (the GPU idles
// meanwhile).  Calls on one thread are sequential (plssvm.h thread-safety rule), so one buffer
// per thread suffices; portable across devices.
char *pinned_scratch(size_t bytes) {
    thread_local struct Buf {
        char *p = nullptr;
        size_t n = 0;
        ~Buf() {
            if (p) cudaFreeHost(p);
        }
    } b;
    if (b.n < bytes) {
        if (b.p) cudaFreeHost(b.p);
        b.p = nullptr;
        b.n = 0;
        PLS_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&b.p), bytes, cudaHostAllocPortable));
        b.n = bytes;
    }
    return b.p;
}

// Timing events of the CG loop (per-launch product events, collective events), created once per
// host thread and device and reused by every call (creating ~100 events per call cost host time
// while the GPU waited for the loop's first launches).  Calls on one thread are sequential.
cudaEvent_t *event_pool(int n) {
    int dev = 0;
    PLS_CUDA(cudaGetDevice(&dev));
    thread_local struct Pool {
        std::vector<std::vector<cudaEvent_t>> per_dev;
        ~Pool() {
            for (auto &v : per_dev)
                for (cudaEvent_t e : v) cudaEventDestroy(e);
        }
    } pool;
    if (static_cast<int>(pool.per_dev.size()) <= dev) pool.per_dev.resize(dev + 1);
    std::vector<cudaEvent_t> &v = pool.per_dev[dev];
    while (static_cast<int>(v.size()) < n) {
        cudaEvent_t e;
        PLS_CUDA(cudaEventCreate(&e));
        v.push_back(e);
    }
    return v.data();
}

// Thread-local pinned staging for host-built index lists (tile lists, pair-tile lists, peer pointers):
// their H2D copies are then truly asynchronous -- a cudaMemcpyAsync from pageable memory waits for the
// stream to drain first, which put a host round trip per list into every call.  Bump allocation inside
// one call; reset at the start of the next (after the last upload's event: no copy of this thread is
// then in flight); growing synchronises once.
struct Upload {
    char *p = nullptr;
    size_t cap = 0, off = 0;
    cudaEvent_t last = nullptr;
    int dev = -1;
    ~Upload() {
        if (last) cudaEventDestroy(last);
        if (p) cudaFreeHost(p);
    }
};
Upload &upload_buf() {
    thread_local Upload u;
    return u;
}
void upload_reset() {
    Upload &u = upload_buf();
    if (u.last) PLS_CUDA(cudaEventSynchronize(u.last));
    u.off = 0;
}
template <typename V>
void upload(V *dst, const V *src, size_t n, cudaStream_t s) {
    Upload &u = upload_buf();
    const size_t bytes = n * sizeof(V), padded = (bytes + 255) / 256 * 256;
    if (bytes == 0) return;
    if (u.off + padded > u.cap) {
        if (u.last) PLS_CUDA(cudaEventSynchronize(u.last));  // every earlier copy from the buffer is done
        if (u.p) PLS_CUDA(cudaFreeHost(u.p));
        u.p = nullptr;
        u.cap = std::max<size_t>({2 * u.cap, padded, size_t(1) << 20});
        PLS_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&u.p), u.cap, cudaHostAllocPortable));
        u.off = 0;
    }
    int dev = 0;
    PLS_CUDA(cudaGetDevice(&dev));
    if (u.last && u.dev != dev) {  // events belong to a device
        PLS_CUDA(cudaEventSynchronize(u.last));
        cudaEventDestroy(u.last);
        u.last = nullptr;
    }
    if (!u.last) {
        PLS_CUDA(cudaEventCreateWithFlags(&u.last, cudaEventDisableTiming));
        u.dev = dev;
    }
    std::memcpy(u.p + u.off, src, bytes);
    PLS_CUDA(cudaMemcpyAsync(dst, u.p + u.off, bytes, cudaMemcpyHostToDevice, s));
    PLS_CUDA(cudaEventRecord(u.last, s));
    u.off += padded;
}

void setup_mempool(int dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
}

template <typename T>
const T *stage_input(Arena &A, const void *src, int64_t n, bool device_ptr, cudaStream_t s) {
    if (device_ptr) return static_cast<const T *>(src);
    T *d = A.alloc<T>(n);
    PLS_CUDA(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
}

// Device-side input validation (replaces host scans of the caller's arrays): every listed array
// is checked for non-finite values, labels for {-1, +1} with both classes.  Arrays with row_len > 0
// (point-major rows: X, Z) also give the largest row peak max_k |x_ik| / rms_k(x_ik) that the engine
// choice needs (oz_choose) -- in the SAME pass and the same single sync.  Throws the plssvm.h status
// with a message.  Outputs are untouched (nothing is written before this).  Returns the peak (0 if no
// array asked for it) and the largest |exponent| of the row maxima (k_row_peak).
struct RowStats {
    float rho = 0.f;
    int emax = 0;
};
template <typename T>
struct VCheck {
    const T *a;
    int64_t n;
    unsigned bit;
    int64_t row_len;  // > 0: rows of this length feed the row-peak reduction
};
template <typename T>
RowStats validate_inputs(Arena &A, std::initializer_list<VCheck<T>> arrays, const T *y, int64_t m, cudaStream_t s,
                         int64_t &launches) {
    unsigned *flags = A.alloc<unsigned>(3);  // [0] validation bits, [1] row peak (float bits), [2] max |E|
    PLS_CUDA(cudaMemsetAsync(flags, 0, 3 * sizeof(unsigned), s));
    bool first = true;
    for (const VCheck<T> &v : arrays) {
        // row arrays: k_row_peak checks finiteness in the same pass (k_validate then only checks labels)
        if (v.row_len == 0 || (first && y)) {
            k_validate<T><<<4 * 148, 256, 0, s>>>(v.a, v.row_len > 0 ? 0 : v.n, v.bit, first ? y : nullptr, m, flags);
            PLS_CHECK_LAUNCH();
            ++launches;
        }
        first = false;
        if (v.row_len > 0) {
            const int64_t rows = v.n / v.row_len;
            k_row_peak<T><<<static_cast<unsigned>(std::max<int64_t>(1, ceil_div(rows * 32, 256))), 256, 0, s>>>(
                v.a, rows, v.row_len, v.row_len, flags + 1, flags, v.bit);
            PLS_CHECK_LAUNCH();
            ++launches;
        }
    }
    unsigned *h = reinterpret_cast<unsigned *>(pinned_scratch(3 * sizeof(unsigned)));
    PLS_CUDA(cudaMemcpyAsync(h, flags, 3 * sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    PLS_CUDA(cudaStreamSynchronize(s));
    if (h[0] & V_NONFINITE_X) throw Error(PLSSVM_E_INVALID_ARG, "X is not finite");
    if (h[0] & V_NONFINITE_Z) throw Error(PLSSVM_E_INVALID_ARG, "Z is not finite");
    if (h[0] & V_NONFINITE_ALPHA) throw Error(PLSSVM_E_INVALID_ARG, "alpha is not finite");
    if (h[0] & V_NONFINITE_P) throw Error(PLSSVM_E_INVALID_ARG, "p is not finite");
    if (y) {
        if (h[0] & V_BADLABEL) throw Error(PLSSVM_E_LABELS, "labels must be +1 or -1");
        if (!(h[0] & V_POS) || !(h[0] & V_NEG)) throw Error(PLSSVM_E_LABELS, "both classes (+1 and -1) must be present");
    }
    RowStats r;
    std::memcpy(&r.rho, &h[1], sizeof(float));
    r.emax = static_cast<int>(h[2]);
    return r;
}

// rows = padded point count of the destination array (its column count is dpad).
template <typename T>
void launch_transform(const T *X, int64_t m, int64_t d, T *Xt, int64_t rows, int64_t dpad, cudaStream_t s,
                      int64_t &launches) {
    dim3 grid(static_cast<unsigned>(ceil_div(rows, 32)), static_cast<unsigned>(ceil_div(dpad, 32)));
    k_transform<T><<<grid, dim3(32, 8), 0, s>>>(X, m, d, Xt, rows, dpad, Engine<T>::kPointMajor ? 1 : 0);
    PLS_CHECK_LAUNCH();
    ++launches;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link needed).
// 2-D row-major array [outer][inner] of 4- or 8-byte elements, box {box_inner, box_outer},
// 128-byte swizzle (box_inner * elem = 128 B).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        PLS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw Error(PLSSVM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    return encode;
}

CUtensorMap make_tmap_2d(void *base, int elem_bytes, int64_t inner, int64_t outer, uint32_t box_inner,
                         uint32_t box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner * elem_bytes)};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = tmap_encoder()(&m, elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(PLSSVM_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

// Pre-swizzled digit blocks (ozaki_engine.cuh k_ozaki_split) as a 2-D byte array of 128-byte rows;
// one box = box_rows rows (a whole digit-plane group of one slab block), no swizzle.
CUtensorMap make_tmap_digit_blocks(int8_t *base, int64_t bytes, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {128u, static_cast<cuuint64_t>(bytes / 128)};
    const cuuint64_t strides[1] = {128u};
    const cuuint32_t box[2] = {128u, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = tmap_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(PLSSVM_E_CUDA, "cuTensorMapEncodeTiled (digits) failed: " + std::to_string(int(r)));
    return m;
}

// The column-operand view of the same digit blocks: a 3-D map (128 B, 128-byte row within a 4 KiB
// plane, plane) whose box {128, 16, planes} is one 64-point half of a 128-point block -- rows
// 16 r .. 16 r + 15 of each of the first `planes` planes -- landing in shared memory as [planes][64 x 32 B],
// the B-half image the 2-SM UMMA reads.
CUtensorMap make_tmap_digit_halves(int8_t *base, int64_t bytes, uint32_t planes) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {128u, 32u, static_cast<cuuint64_t>(bytes / 4096)};
    const cuuint64_t strides[2] = {128u, 4096u};
    const cuuint32_t box[3] = {128u, 16u, planes};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = tmap_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(PLSSVM_E_CUDA, "cuTensorMapEncodeTiled (digit halves) failed: " + std::to_string(int(r)));
    return m;
}
CUtensorMap make_tmap_2d_f32(float *base, int64_t inner, int64_t outer, uint32_t box_inner, uint32_t box_outer) {
    return make_tmap_2d(base, 4, inner, outer, box_inner, box_outer);
}

// Tile-kernel operands: A = row operand array (rows_a points), B = column operand array.
Ops<double> make_ops(double *A, int64_t rows_a, double *B, int64_t rows_b, int64_t dpad) {
    using E = Engine<double>;
    Ops<double> o;
    o.a = make_tmap_2d(A, 8, dpad, rows_a, E::BK, kTile);
    o.b = make_tmap_2d(B, 8, dpad, rows_b, E::BK, E::TN);
    return o;
}
Ops<float> make_ops(float *A, int64_t, float *B, int64_t, int64_t ld) { return Ops<float>{A, B, ld}; }

// Row-band geometry of this rank: padded length mpad (multiple of 128 * P), tiles per rank.
struct Geometry {
    int64_t m1, mpad, dpad, ld, nb, g0;
    int T, band0, band1, P, rank;
};

template <typename T>
Geometry geometry(int64_t m, int64_t d, int P, int rank) {
    Geometry g;
    g.m1 = m - 1;
    g.P = P;
    g.rank = rank;
    g.mpad = round_up(m, static_cast<int64_t>(kTile) * P);
    g.dpad = round_up(d, Engine<T>::BK);
    g.ld = Engine<T>::kPointMajor ? g.dpad : g.mpad;
    g.T = static_cast<int>(g.mpad / kTile);
    const int per = g.T / P;
    g.band0 = rank * per;
    g.band1 = g.band0 + per;
    g.nb = static_cast<int64_t>(per) * kTile;
    g.g0 = static_cast<int64_t>(g.band0) * kTile;
    return g;
}

// Tiles of this rank: rows I of the band against every column block J; inside the band only
// the upper triangle J >= I (mirrored), outside it the full row (row sums only).
// Each entry is (I, J * NSUB + h): column sub-block h of width 128 / NSUB.  Raster order for
// L2 reuse: row blocks in groups of kGroup; inside a group the column sub-blocks advance
// slowest and the group's rows fastest, so the ~2 x 148 co-resident CTAs touch kGroup row
// blocks and a few column blocks of X instead of a whole row of tiles (all of X).
std::vector<int2> band_tiles(const Geometry &g, int nsub) {
    constexpr int kGroup = 8;
    std::vector<int2> t;
    for (int I0 = g.band0; I0 < g.band1; I0 += kGroup) {
        const int I1 = std::min(I0 + kGroup, g.band1);
        for (int J = 0; J < g.T; ++J)
            for (int I = I0; I < I1; ++I) {
                const bool inband = (J >= g.band0 && J < g.band1);
                if (!inband || J >= I)
                    for (int h = 0; h < nsub; ++h) t.push_back(make_int2(I, J * nsub + h));  // halves adjacent:
            }                                                                             // packed ordinal = idx/nsub
    }
    return t;
}

int dtype_of(float) { return PLSSVM_F32; }
int dtype_of(double) { return PLSSVM_F64; }

// Circulant assignment of the symmetric tile pairs (SURVEY §8(e) option ii): tile row I owns
// the pairs (I, (I + j) mod T), j = 0..T/2, except that for even T the pair j = T/2 belongs to
// the smaller row only -- every unordered pair exactly once, ~T/2 tiles per row.  This rank
// takes the tile rows of its band.
std::vector<int2> circulant_tiles(const Geometry &g, int nsub) {
    std::vector<int2> t;
    const int half = g.T / 2;
    for (int I = g.band0; I < g.band1; ++I)
        for (int j = 0; j <= half; ++j) {
            if (g.T % 2 == 0 && j == half && I >= half) continue;
            const int J = (I + j) % g.T;
            if (j > 0 && J == I) continue;  // T == 1
            for (int h = 0; h < nsub; ++h) t.push_back(make_int2(I, J * nsub + h));
        }
    return t;
}

// Digit blocks of a point-major padded array (ozaki_engine.cuh k_ozaki_split, ONE layout DA of
// 128-point blocks): TMA maps whose boxes carry the first LV (pass 0) or all S planes of a slab
// block -- t4 / t8 for the row operand (a whole 128-point block), h4 / h8 for the column operand
// (one 64-point half of a block: 16 of each plane's 32 rows of 128 B, planes 4 KiB apart).  Both
// roles read the same bytes, so a point's digits are stored and cached once.
struct OzOperand {
    int8_t *DA = nullptr;
    double *sc = nullptr;
    CUtensorMap t4, t8;  // row-operand boxes
    CUtensorMap h4, h8;  // column-operand (half-block) boxes
    int nk = 0;
};

template <typename T>
struct Ctx {
    Geometry g;
    KParams<T> kp;
    T invC;
    cudaStream_t s;
    CommHandle *comm;
    // device buffers
    T *Xt, *q, *nrm, *ylab, *x, *r, *p, *y, *Ypart, *partials, *xfull, *Qc;
    double *scal;
    unsigned *counter;
    int2 *tiles;
    int ntiles;
    bool cached;
    bool tc = false;             // fp32: tcgen05 3xTF32 contraction
    float *Xhi = nullptr, *Xlo = nullptr;
    CUtensorMap tm_hi, tm_lo;
    CUtensorMap tw_ahi, tw_alo, tw_bhi, tw_blo;  // wide (128 x 256, SWIZZLE_64B) kernel
    bool wide = false, wide_ok = true;
    int2 *wtiles = nullptr;
    int nwtiles = 0;
    int64_t dpad_tc = 0;
    int nsplit = 1;  // cached GEMV: column splits per row block
    int64_t launches = 0, launches_cg = 0;
    Ops<T> ops;
    bool circ = false;               // implicit multi-GPU: circulant pairs + reduce-scatter
    bool lowrank = false;            // linear kernel, O(md) product (mode LOWRANK)
    bool packed = false;             // cached mode, symmetric-packed tiles (k_gemv_sym)
    int64_t nstored = 0;             // stored tiles of the packed layout
    const T *Xraw = nullptr;         // the caller's row-major X on the device (staged or given)
    int64_t m = 0, d = 0;
    T *tpart = nullptr, *tvec = nullptr;
    double *tloc = nullptr;          // [2d]: local partial, global sum (multi-GPU)
    double *psum = nullptr;          // [lr_parts]: slices of sum(p)
    int lr_parts = 1;
    int64_t lr_rpb = 1;
    T *yfull = nullptr, *ysc = nullptr, *Yfin = nullptr;
    int nsub_eff = 1;
    int *ctrl = nullptr;             // device CG control block (kernels.cuh Ctl)
    bool oz = false;                 // fp64: int8 tensor-core digit engine (ozaki_engine.cuh)
    OzOperand ozx;
    int4 *oz_pt = nullptr;            // 2-SM pair-tiles (ozaki_engine.cuh)
    int *oz_pk = nullptr;
    int oz_npt = 0;
    int4 *oz_pt_mv = nullptr;         // one GPU: the products' pair-tiles with no dropped half
    int oz_npt_mv = 0;                // (oz_pair_tiles_matvec; 0 = use oz_pt)
    const int *cur_ctrl = nullptr;   // ctrl inside the CG loop (loop kernels early-exit when done)
    bool fsplit = false;             // PLSSVM_MULTI_GPU_FEATURES: this rank's feature slice only,
                                     // partial products summed by an all-reduce
    int nranks = 1;                  // communicator size (g.P is the row-shard count)
    T *yred = nullptr;               // fsplit: the all-reduced product
    bool graph_used = false;         // the CG loop ran as one CUDA graph (WHILE node)
    int pap_slot = S_PAP;            // scalar slot of finalize's p.Q~p (Chronopoulos-Gear: S_CG_DELTA)
    // collective timing (stats.t_comm, SURVEY §8(d) "NCCL time separated with events"): event
    // pairs around every collective of the current CG iteration, when set
    cudaEvent_t *cev = nullptr;
    int ncev = 0, cev_cap = 0;
    // PEER transport with direct peer access: every rank's full p (device array), for the p update
    // that stores its band into all of them (the all-gather fused into k_update_p)
    T **peer_p = nullptr;
    bool lsa = false;  // p in the NCCL symmetric window (k_update_p_lsa)
    // blocks of the CG vector kernels: one per 64 band rows, at most kVecBlocks (a fixed function of
    // the band length, so every kernel, loop and rank reduces in the same order); small problems no
    // longer pay for 296 blocks in every grid reduction / barrier (C0: 4 blocks)
    int vb = kVecBlocks;
    int npeer = 0;
};

// Runs `f` (one collective on c.s) between two of the iteration's timing events, if any.
template <typename T, typename F>
void timed_comm(Ctx<T> &c, F f) {
    const bool t = c.cev && c.ncev + 2 <= c.cev_cap;
    if (t) PLS_CUDA(cudaEventRecord(c.cev[c.ncev++], c.s));
    f();
    if (t) PLS_CUDA(cudaEventRecord(c.cev[c.ncev++], c.s));
}

// cudaFuncSetAttribute is per function and device: each attribute group is applied once per device
// (the ~30 calls cost a few us each and ran on every training / predict call).  The group's bit is
// set only after every attribute call succeeded, under a mutex, so a concurrent caller on the same
// device waits for the setup instead of launching before the smem limit is raised, and a failed
// setup is retried by the next call.
template <typename F>
void once_per_device(int group, F apply) {
    static std::mutex mu;
    static uint64_t done[8] = {};  // group -> mask of devices already configured
    int dev = 0;
    PLS_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = uint64_t(1) << (dev & 63);
    std::lock_guard<std::mutex> lock(mu);
    if (done[group] & bit) return;
    apply();
    done[group] |= bit;
}

template <typename T>
void set_smem_attrs() {
    once_per_device(std::is_same<T, double>::value ? 0 : 1, [] {
    const int bytes = static_cast<int>(Engine<T>::SMEM_BYTES);
    PLS_CUDA(cudaFuncSetAttribute(k_matvec_implicit<LINEAR, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_matvec_implicit<POLYNOMIAL, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_matvec_implicit<RBF, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_precompute<LINEAR, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_precompute<POLYNOMIAL, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_precompute<RBF, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_predict_tiles<LINEAR, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_predict_tiles<POLYNOMIAL, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_predict_tiles<RBF, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PLS_CUDA(cudaFuncSetAttribute(k_matvec_implicit<LINEAR, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    PLS_CUDA(cudaFuncSetAttribute(k_matvec_implicit<POLYNOMIAL, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    PLS_CUDA(cudaFuncSetAttribute(k_matvec_implicit<RBF, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    PLS_CUDA(cudaFuncSetAttribute(k_precompute<LINEAR, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    PLS_CUDA(cudaFuncSetAttribute(k_precompute<POLYNOMIAL, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    PLS_CUDA(cudaFuncSetAttribute(k_precompute<RBF, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    PLS_CUDA(cudaFuncSetAttribute(k_predict_tiles<LINEAR, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    PLS_CUDA(cudaFuncSetAttribute(k_predict_tiles<POLYNOMIAL, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    PLS_CUDA(cudaFuncSetAttribute(k_predict_tiles<RBF, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    });
}

void tc_set_attrs();

// fp32 tensor-core engine setup: hi/lo split arrays (point-major) + TMA descriptors.
template <typename T>
void setup_tc(Ctx<T> &c, Arena &A, const T *Xs, int64_t m, int64_t d) {
    if constexpr (std::is_same<T, float>::value) {
        const Geometry &g = c.g;
        c.dpad_tc = round_up(d, Tc::BK);
        c.Xhi = A.alloc<float>(g.mpad * c.dpad_tc);
        c.Xlo = A.alloc<float>(g.mpad * c.dpad_tc);
        const int64_t n = g.mpad * c.dpad_tc;
        k_split_tf32<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, c.s>>>(Xs, m, d, c.Xhi, c.Xlo, g.mpad, c.dpad_tc);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        c.tm_hi = make_tmap_2d_f32(c.Xhi, c.dpad_tc, g.mpad, Tc::BK, kTile);
        c.tm_lo = make_tmap_2d_f32(c.Xlo, c.dpad_tc, g.mpad, Tc::BK, kTile);
        c.tw_ahi = make_tmap_2d(c.Xhi, 4, c.dpad_tc, g.mpad, TcW::BK, kTile, CU_TENSOR_MAP_SWIZZLE_64B);
        c.tw_alo = make_tmap_2d(c.Xlo, 4, c.dpad_tc, g.mpad, TcW::BK, kTile, CU_TENSOR_MAP_SWIZZLE_64B);
        c.tw_bhi = make_tmap_2d(c.Xhi, 4, c.dpad_tc, g.mpad, TcW::BK, 2 * kTile, CU_TENSOR_MAP_SWIZZLE_64B);
        c.tw_blo = make_tmap_2d(c.Xlo, 4, c.dpad_tc, g.mpad, TcW::BK, 2 * kTile, CU_TENSOR_MAP_SWIZZLE_64B);
        tc_set_attrs();
    }
}

template <int KT, int MODE>
void tc_launch(int grid, cudaStream_t s, const CUtensorMap &ah, const CUtensorMap &al, const CUtensorMap &bh,
               const CUtensorMap &bl, int64_t dpad, const int2 *tiles, int tilesI, const float *qa, const float *na,
               const float *qb, const float *nb_, const float *p, KParams<float> kp, float invC, const double *scal,
               int64_t m1, int band0, int band1, float *Ypart, int64_t band_rows, float *Qc, int T_tiles,
               const int *ctrl) {
    k_tile_tc<KT, MODE><<<grid, Tc::THREADS, Tc::SMEM_BYTES, s>>>(ah, al, bh, bl, dpad, tiles, tilesI, qa, na, qb, nb_, p,
                                                                 kp, invC, scal, m1, band0, band1, Ypart, band_rows,
                                                                 Qc, T_tiles, ctrl);
    PLS_CHECK_LAUNCH();
}

template <int MODE, typename... Args>
void tc_dispatch(int kernel, Args &&...args) {
    switch (kernel) {
        case LINEAR: tc_launch<LINEAR, MODE>(args...); break;
        case POLYNOMIAL: tc_launch<POLYNOMIAL, MODE>(args...); break;
        default: tc_launch<RBF, MODE>(args...);
    }
}

void tc_set_attrs() {
    once_per_device(2, [] {
    const int bytes = static_cast<int>(Tc::SMEM_BYTES);
#define PLS_TC_ATTR(K, M) PLS_CUDA(cudaFuncSetAttribute(k_tile_tc<K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))
    PLS_TC_ATTR(LINEAR, TC_MATVEC); PLS_TC_ATTR(POLYNOMIAL, TC_MATVEC); PLS_TC_ATTR(RBF, TC_MATVEC);
    PLS_TC_ATTR(LINEAR, TC_PRECOMPUTE); PLS_TC_ATTR(POLYNOMIAL, TC_PRECOMPUTE); PLS_TC_ATTR(RBF, TC_PRECOMPUTE);
    PLS_TC_ATTR(LINEAR, TC_PREDICT); PLS_TC_ATTR(POLYNOMIAL, TC_PREDICT); PLS_TC_ATTR(RBF, TC_PREDICT);
#undef PLS_TC_ATTR
    const int wb = static_cast<int>(TcW::SMEM_BYTES);
    PLS_CUDA(cudaFuncSetAttribute(k_tile_tc_wide<LINEAR, TC_MATVEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, wb));
    PLS_CUDA(cudaFuncSetAttribute(k_tile_tc_wide<POLYNOMIAL, TC_MATVEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, wb));
    PLS_CUDA(cudaFuncSetAttribute(k_tile_tc_wide<RBF, TC_MATVEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, wb));
    PLS_CUDA(cudaFuncSetAttribute(k_tile_tc_wide<LINEAR, TC_PREDICT>, cudaFuncAttributeMaxDynamicSharedMemorySize, wb));
    PLS_CUDA(cudaFuncSetAttribute(k_tile_tc_wide<POLYNOMIAL, TC_PREDICT>, cudaFuncAttributeMaxDynamicSharedMemorySize, wb));
    PLS_CUDA(cudaFuncSetAttribute(k_tile_tc_wide<RBF, TC_PREDICT>, cudaFuncAttributeMaxDynamicSharedMemorySize, wb));
    });
}

template <int KT, int MODE>
void tcw_launch(int grid, cudaStream_t s, const CUtensorMap &ah, const CUtensorMap &al, const CUtensorMap &bh,
                const CUtensorMap &bl, int64_t dpad, const int2 *tiles, int tilesI, int T_tiles, const float *qa,
                const float *na, const float *qb, const float *nb_, const float *p, KParams<float> kp, float invC,
                const double *scal, int64_t m1, float *Ypart, int64_t band_rows, const int *ctrl) {
    k_tile_tc_wide<KT, MODE><<<grid, TcW::THREADS, TcW::SMEM_BYTES, s>>>(ah, al, bh, bl, dpad, tiles, tilesI, T_tiles, qa,
                                                                        na, qb, nb_, p, kp, invC, scal, m1, Ypart,
                                                                        band_rows, ctrl);
    PLS_CHECK_LAUNCH();
}

template <int MODE, typename... Args>
void tcw_dispatch(int kernel, Args &&...args) {
    switch (kernel) {
        case LINEAR: tcw_launch<LINEAR, MODE>(args...); break;
        case POLYNOMIAL: tcw_launch<POLYNOMIAL, MODE>(args...); break;
        default: tcw_launch<RBF, MODE>(args...);
    }
}

// Wide tiles (I, Jw) of the upper triangle for one GPU: Jw from I/2 (grouped raster).
std::vector<int2> wide_tiles(int T) {
    std::vector<int2> t;
    const int TW = (T + 1) / 2;
    for (int I0 = 0; I0 < T; I0 += 8)
        for (int Jw = 0; Jw < TW; ++Jw)
            for (int I = I0; I < std::min(I0 + 8, T); ++I)
                if (Jw >= I / 2) t.push_back(make_int2(I, Jw));
    return t;
}

// ---- fp64 on the int8 tensor cores (ozaki_engine.cuh) -------------------------------------
constexpr int kOzS = 7;  // balanced base-256 digits per point: fp64-level products
using OzC = Oz<kOzS>;
// digits of the engine for value type T: 7 for fp64, 3 for fp32 (PLSSVM_FP32_OZAKI)
template <typename T>
constexpr int oz_digits() { return std::is_same<T, double>::value ? 7 : 3; }

int num_sms() {
    int dev = 0, n = 0;
    PLS_CUDA(cudaGetDevice(&dev));
    PLS_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

// S digit planes of the point-major padded array Xp (fp64 with S = 7, fp32 with S = 3).  Maps:
// t8 / h8 carry all S planes of a slab block, t4 / h4 the first LV planes (S = 7's pass 1).
template <int S, typename TIN>
OzOperand oz_prepare(Arena &A, const TIN *Xp, int64_t rows, int64_t m_valid, int64_t dpad, int64_t d, bool row_role,
                     bool col_role, cudaStream_t s, int64_t &launches) {
    using O = Oz<S>;
    OzOperand o;
    const int64_t d8 = round_up(d, O::BK);
    const int64_t bytes = S * rows * d8;
    o.DA = A.alloc<int8_t>(bytes);
    o.sc = A.alloc<double>(rows);
    k_ozaki_split<S, TIN><<<static_cast<unsigned>(ceil_div(rows * 32, 256)), 256, 0, s>>>(Xp, rows, m_valid, dpad, d8,
                                                                                         o.DA, o.sc);
    PLS_CHECK_LAUNCH();
    ++launches;
    if (row_role) {  // (the full-plane boxes span O::BOXSL consecutive slabs of a pipeline stage)
        o.t4 = make_tmap_digit_blocks(o.DA, bytes, O::LV * 32);
        o.t8 = make_tmap_digit_blocks(o.DA, bytes, O::BOXSL * S * 32);
    }
    if (col_role) {
        o.h4 = make_tmap_digit_halves(o.DA, bytes, O::LV);
        o.h8 = make_tmap_digit_halves(o.DA, bytes, O::BOXSL * S);
    }
    o.nk = static_cast<int>(d8 / O::BK);
    return o;
}

// fp64 engine choice (plssvm.h plssvm_fp64_engine_t): OZAKI, DMMA, or AUTO.  AUTO takes OZAKI only
// when its worst-case error is no larger than the textbook fp64 one: per inner product
// |s~ - s| <= u|s| + kOzC64 d u ||x_i||inf ||x_j||inf (ozaki_engine.cuh), and an fp64 dot obeys
// gamma_d sum|x_ik x_jk| <= ~d u ||x_i||_2 ||x_j||_2 (Cauchy-Schwarz form); with the row peak
// rho = ||x||_inf / rms(x), ||x_i||inf ||x_j||inf = rho_i rho_j ||x_i||_2 ||x_j||_2 / d, so OZAKI's bound is
// the smaller one iff kOzC64 rho_i rho_j <= d: AUTO checks kOzC64 rho_max^2 <= d.  (N(0,1)-like data:
// rho_max ~ 5 -> d >= 330; C1's d = 1024 allows rho <= 8.9, C2 / C4's 4096 rho <= 17.7.)
constexpr double kOzC64 = 13.04;  // 1 (input rounding to the row grid) + 12.04 (dropped levels 7..12)
constexpr int64_t kOzMaxD = 16384;
constexpr int64_t kOzMinRows = 384;  // AUTO: padded point counts up to this use DMMA
// The epilogue converts 2^k V with k = E_i + E_j - 36 (and 2^{k-24} W) by building the exponent
// directly (ozaki_engine.cuh scaled_exact): 1 <= 1074 + k - 24 and 1074 + k <= 2045 need
// -1014 <= E_i + E_j <= 1007, i.e. row maxima within 2^-480 .. 2^480 (~1e-144 .. 1e144).
constexpr int kOzMaxExp = 480;
// rs = the largest row peak and row-maximum exponent of the operand arrays (validate_inputs),
// most_rows = the largest padded point count among them.
bool oz_choose(int engine, const RowStats &rs, int64_t most_rows, int64_t d) {
    if (engine == PLSSVM_FP64_DMMA) return false;
    const double rho = rs.rho;
    // int32 level sums: |acc_l| <= 7 d8 2^14 < 2^31 needs d8 <= 18724; limit 16384 (ozaki_engine.cuh)
    const bool fits = round_up(d, OzC::BK) <= kOzMaxD && rs.emax <= kOzMaxExp;
    if (engine == PLSSVM_FP64_OZAKI) {
        if (round_up(d, OzC::BK) > kOzMaxD)
            throw Error(PLSSVM_E_INVALID_ARG, "fp64_engine OZAKI supports d <= " + std::to_string(kOzMaxD) +
                                                  " (int32 digit-product sums); use AUTO or DMMA");
        if (rs.emax > kOzMaxExp)
            throw Error(PLSSVM_E_INVALID_ARG, "fp64_engine OZAKI supports row maxima within 2^-" +
                                                  std::to_string(kOzMaxExp) + " .. 2^" + std::to_string(kOzMaxExp) +
                                                  " (digit-scale exponents); use AUTO or DMMA");
        return true;
    }
    if (!fits) return false;
    // tiny problems: the persistent 2-SM kernel's fixed cost (~20 us: TMEM allocation, barriers,
    // two TMEM passes) exceeds the whole DMMA product (profiles/r01_small_engines.txt: 256 x 16
    // 24.6 vs 16.7 us per product)
    if (most_rows <= kOzMinRows) return false;
    return kOzC64 * rho * rho <= static_cast<double>(d);
}

// fp32 engine choice (plssvm.h plssvm_fp32_engine_t): AUTO = OZAKI under the same criterion as fp64
// with the fp32 unit u32 = 2^-24: the 3-digit split (22 bits below the row maximum, levels <= 2) has
// |s~ - s| <= u32|s| + kOzC32 d u32 ||x_i||inf ||x_j||inf (input rounding 2^-23 of the row scale: 8 d u32;
// dropped levels 3..4: 32.2 d u32), so AUTO needs kOzC32 rho_max^2 <= d (C3's d = 2048: rho <= 7.1),
// else TCGEN05 (3xTF32); d > 16384 also TCGEN05.
constexpr double kOzC32 = 40.2;
bool oz_choose_f32(int engine, const RowStats &rs, int64_t d) {
    if (engine == PLSSVM_FP32_TCGEN05 || engine == PLSSVM_FP32_FFMA) return false;
    const double rho = rs.rho;  // (fp32 exponents are always in the conversion's range)
    const bool fits = round_up(d, Oz<3>::BK) <= kOzMaxD;
    if (engine == PLSSVM_FP32_OZAKI) {
        if (!fits) throw Error(PLSSVM_E_INVALID_ARG, "fp32_engine OZAKI supports d <= " + std::to_string(kOzMaxD));
        return true;
    }
    if (!fits) return false;
    return kOzC32 * rho * rho <= static_cast<double>(d);
}

template <typename T>
void oz_set_attrs() {
    once_per_device(std::is_same<T, double>::value ? 3 : 4, [] {
    constexpr int S = oz_digits<T>();
    const int bytes = static_cast<int>(Oz<S>::SMEM_BYTES);
#define PLS_OZ_ATTR(K, M) \
    PLS_CUDA(cudaFuncSetAttribute(k_tile_ozaki<K, S, M, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))
    PLS_OZ_ATTR(LINEAR, OZ_MATVEC); PLS_OZ_ATTR(POLYNOMIAL, OZ_MATVEC); PLS_OZ_ATTR(RBF, OZ_MATVEC);
    PLS_OZ_ATTR(LINEAR, OZ_PRECOMPUTE); PLS_OZ_ATTR(POLYNOMIAL, OZ_PRECOMPUTE); PLS_OZ_ATTR(RBF, OZ_PRECOMPUTE);
    PLS_OZ_ATTR(LINEAR, OZ_PREDICT); PLS_OZ_ATTR(POLYNOMIAL, OZ_PREDICT); PLS_OZ_ATTR(RBF, OZ_PREDICT);
#undef PLS_OZ_ATTR
    });
}

// Decomposition experiments (results are WRONG when set): 1 = no epilogue, 2 = no TMA, 4 = no MMAs.
// Only in the experiment build (_build.build(variant="exp"), -DPLSSVM_OZ_EXPERIMENTS, a separate .so
// the tools load explicitly); the product library has no switch that changes what is computed.
int oz_debug_flags() {
#ifdef PLSSVM_OZ_EXPERIMENTS
    static int f = [] {
        const char *e = std::getenv("PLSSVM_OZ_DEBUG");
        return e ? std::atoi(e) : 0;
    }();
    return f;
#else
    return 0;
#endif
}

// One persistent CTA per SM (the 512-column TMEM allocation admits one per SM anyway), in
// clusters of 2 (cta_group::2): the grid is an even number of CTAs, at most the SM count.
template <int KT, int MODE, typename T>
void oz_launch(int npt, cudaStream_t s, const OzOperand &ra, const OzOperand &cb, const int4 *ptiles, const int *pk,
               int rowsI, const T *qv, const T *na, const T *nb_, const T *p, KParams<T> kp, T invC,
               const double *scal, int64_t m1, int band0, int band1, T *Ypart, int64_t band_rows, T *Qc, int T_tiles,
               const int *ctrl) {
    constexpr int S = oz_digits<T>();
    using O = Oz<S>;
    if (npt <= 0) return;
    // Only co-resident clusters (a pair must fit in one GPC): a statically scheduled grid with one
    // cluster too many would run that cluster's tiles as a second wave.
    static std::atomic<int> max_clusters[3][3] = {};
    int mc = max_clusters[KT][MODE].load();
    if (mc == 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(num_sms()), 1, 1);
        cfg.blockDim = dim3(O::THREADS, 1, 1);
        cfg.dynamicSmemBytes = O::SMEM_BYTES;
        PLS_CUDA(cudaOccupancyMaxActiveClusters(&mc, k_tile_ozaki<KT, S, MODE, T>, &cfg));
        if (mc <= 0) mc = num_sms() / 2;
        max_clusters[KT][MODE].store(mc);
        if (std::getenv("PLSSVM_DEBUG")) std::fprintf(stderr, "[plssvm] k_tile_ozaki co-resident pairs: %d\n", mc);
    }
    const int grid = 2 * std::min(npt, mc);
    k_tile_ozaki<KT, S, MODE, T><<<grid, O::THREADS, O::SMEM_BYTES, s>>>(
        ra.t4, ra.t8, cb.h4, cb.h8, ra.nk, ptiles, pk, npt, rowsI, ra.sc, cb.sc, qv, na, nb_, p, kp, invC, scal, m1,
        band0, band1, Ypart, band_rows, Qc, T_tiles, ctrl, oz_debug_flags());
    PLS_CHECK_LAUNCH();
}

// Pair-tiles of the 2-SM kernel from a tile list (I, J) (NSUB = 1): row blocks b0, b0 + 2, ...
// of [b0, b1) paired with the next one; entry (I0 | use << 24, J) where use bit r marks (I0 + r, J)
// as a listed tile.  pk[2 t + r] = that tile's ordinal in the list (packed cached layout), -1
// if unused.  Raster: groups of oz_group_rows() row blocks, column blocks slowest inside a group (L2 reuse).
// Row blocks per raster group: the group's row-operand digits (7 planes x 128 rows x d8 bytes per
// block) should stay L2-resident while the co-resident pairs sweep the column blocks -- 32 blocks
// up to ~40 MB (C1: DRAM reads per product 902 -> 405 MB, ncu), fewer for wide points (C2 at 32:
// 117 MB, L2 thrash, +4 % time).  PLSSVM_OZ_GROUP overrides it in the experiment build only.
int oz_group_rows(int64_t d8, int S) {
#ifdef PLSSVM_OZ_EXPERIMENTS
    static int forced = [] {
        const char *e = std::getenv("PLSSVM_OZ_GROUP");
        const int v = e ? std::atoi(e) : 0;
        return v >= 2 ? (v & ~1) : 0;
    }();
    if (forced) return forced;
#endif
    const int64_t per_block = int64_t(S) * 128 * d8;
    const int64_t budget = int64_t(40) << 20;
    return per_block * 32 <= budget ? 32 : per_block * 16 <= budget ? 16 : 8;
}

void oz_pair_tiles(const std::vector<int2> &tl, int b0, int b1, int T, int64_t d8, int S, std::vector<int4> &pt,
                   std::vector<int> &pk) {
    std::vector<int> ord(static_cast<size_t>(b1 - b0) * T, -1);
    for (size_t k = 0; k < tl.size(); ++k) ord[static_cast<size_t>(tl[k].x - b0) * T + tl[k].y] = static_cast<int>(k);
    pt.clear();
    pk.clear();
    const int G = oz_group_rows(d8, S);
    for (int P0 = b0; P0 < b1; P0 += G)
        for (int J = 0; J < T; ++J)
            for (int I0 = P0; I0 < std::min(P0 + G, b1); I0 += 2) {
                const int o0 = ord[static_cast<size_t>(I0 - b0) * T + J];
                const int o1 = (I0 + 1 < b1) ? ord[static_cast<size_t>(I0 + 1 - b0) * T + J] : -1;
                if (o0 < 0 && o1 < 0) continue;
                const int use = (o0 >= 0 ? 1 : 0) | (o1 >= 0 ? 2 : 0);
                pt.push_back(make_int4(I0, I0 + 1, J, use));
                pk.push_back(o0);
                pk.push_back(o1);
            }
}

// Pair-tiles of the one-GPU implicit PRODUCT (OZ_MATVEC) with no dropped half.  The upper-triangle
// list puts column block J's tiles (I, J), I = 0..J, in one column: J + 1 tiles, odd for every even
// J, so oz_pair_tiles computes and drops the lower block (J + 1, J) of every diagonal pair-tile --
// T/2 wasted half pair-tiles (C1: 4160 pair-tiles for 4128 of work, 57 instead of 56 rounds of the
// 74 co-resident CTA pairs).  The product's epilogue treats a tile and its mirror alike (row sums of
// (I, J) -> slot J of block I, column sums -> slot I of block J, whichever of I, J is larger), so
// the tile {J1, J2} of two consecutive odd columns J1 < J2 can be computed as (J2, J1) in column J1:
// every column even, every tile in exactly one pair (one single only when T(T+1)/2 is odd).  The
// same (slot, block) entries are written exactly once as before.  Rows of a column are paired in
// order (adjacent blocks except around the moved tiles) and the raster is oz_pair_tiles' (groups of
// G row blocks, column blocks slowest inside a group).  The cached precompute keeps oz_pair_tiles'
// list (its packed tiles are stored in the (I <= J) orientation).
void oz_pair_tiles_matvec(int T, int64_t d8, int S, std::vector<int4> &pt) {
    std::vector<std::vector<int>> rows(static_cast<size_t>(T));
    for (int J = 0; J < T; ++J)
        for (int I = 0; I <= J; ++I) rows[J].push_back(I);
    std::vector<int> odd;
    for (int J = 0; J < T; ++J)
        if (rows[J].size() % 2) odd.push_back(J);
    for (size_t k = 0; k + 1 < odd.size(); k += 2) {  // tile (J1, J2): column J2 -> column J1 as (J2, J1)
        const int J1 = odd[k], J2 = odd[k + 1];
        rows[J2].erase(std::find(rows[J2].begin(), rows[J2].end(), J1));
        rows[J1].push_back(J2);
    }
    const int G = oz_group_rows(d8, S);
    std::vector<std::pair<std::pair<int, int>, int4>> items;  // ((group, J), pair)
    for (int J = 0; J < T; ++J) {
        std::vector<int> &r = rows[J];
        std::sort(r.begin(), r.end());
        for (size_t k = 0; k < r.size(); k += 2) {
            const bool two = k + 1 < r.size();
            const int I0 = r[k], I1 = two ? r[k + 1] : r[k];
            items.push_back({{I0 / G, J}, make_int4(I0, I1, J, two ? 3 : 1)});
        }
    }
    std::stable_sort(items.begin(), items.end(),
                     [](const auto &a, const auto &b) { return a.first < b.first; });
    pt.clear();
    for (const auto &it : items) pt.push_back(it.second);
}

template <int MODE, typename T, typename... Args>
void oz_dispatch(int kernel, Args &&...args) {
    switch (kernel) {
        case LINEAR: oz_launch<LINEAR, MODE, T>(args...); break;
        case POLYNOMIAL: oz_launch<POLYNOMIAL, MODE, T>(args...); break;
        default: oz_launch<RBF, MODE, T>(args...);
    }
}

template <typename T>
bool launch_oz(Ctx<T> &c, const T *pfull, int b0, int b1, int64_t brows, bool precompute) {
    if (!c.oz) return false;
    const Geometry &g = c.g;
    const T *cq = c.q, *cn = c.nrm;
    if (precompute)
        oz_dispatch<OZ_PRECOMPUTE, T>(c.kp.kernel, c.oz_npt, c.s, c.ozx, c.ozx, c.oz_pt, c.oz_pk, 0, cq, cn, cn,
                                      static_cast<const T *>(nullptr), c.kp, c.invC, static_cast<const double *>(c.scal),
                                      g.m1, g.band0, g.band1, static_cast<T *>(nullptr), g.nb, c.Qc,
                                      c.packed ? -1 : g.T, static_cast<const int *>(nullptr));
    else if (c.oz_npt_mv > 0)
        oz_dispatch<OZ_MATVEC, T>(c.kp.kernel, c.oz_npt_mv, c.s, c.ozx, c.ozx, c.oz_pt_mv, c.oz_pk, 0, cq, cn, cn, pfull,
                                  c.kp, c.invC, static_cast<const double *>(c.scal), g.m1, b0, b1, c.Ypart, brows,
                                  static_cast<T *>(nullptr), g.T, c.cur_ctrl);
    else
        oz_dispatch<OZ_MATVEC, T>(c.kp.kernel, c.oz_npt, c.s, c.ozx, c.ozx, c.oz_pt, c.oz_pk, 0, cq, cn, cn, pfull,
                                  c.kp, c.invC, static_cast<const double *>(c.scal), g.m1, b0, b1, c.Ypart, brows,
                                  static_cast<T *>(nullptr), g.T, c.cur_ctrl);
    ++c.launches;
    return true;
}

// (Re)build the 2-SM pair-tile list from the current single-tile list.
template <typename T>
void oz_build_pairs(Ctx<T> &c, Arena &A, const std::vector<int2> &tl, int b0, int b1) {
    if (!c.oz) return;
    std::vector<int4> pt;
    std::vector<int> pk;
    oz_pair_tiles(tl, b0, b1, c.g.T, int64_t(c.ozx.nk) * 32, oz_digits<T>(), pt, pk);
    c.oz_npt = static_cast<int>(pt.size());
    c.oz_pt = A.alloc<int4>(c.oz_npt);
    c.oz_pk = A.alloc<int>(2 * c.oz_npt);
    upload(c.oz_pt, pt.data(), pt.size(), c.s);
    upload(c.oz_pk, pk.data(), pk.size(), c.s);
    c.oz_npt_mv = 0;
    if (c.g.P == 1 && b0 == 0 && b1 == c.g.T) {  // one GPU, upper triangle: products with no dropped half
        std::vector<int4> pm;
        oz_pair_tiles_matvec(c.g.T, int64_t(c.ozx.nk) * 32, oz_digits<T>(), pm);
        c.oz_npt_mv = static_cast<int>(pm.size());
        c.oz_pt_mv = A.alloc<int4>(c.oz_npt_mv);
        upload(c.oz_pt_mv, pm.data(), pm.size(), c.s);
    }
}

template <typename T>
bool launch_tc(Ctx<T> &c, const T *pfull, int b0, int b1, int64_t brows) {
    if constexpr (std::is_same<T, float>::value) {
        const Geometry &g = c.g;
        if (c.wide) {
            tcw_dispatch<TC_MATVEC>(c.kp.kernel, c.nwtiles, c.s, c.tw_ahi, c.tw_alo, c.tw_bhi, c.tw_blo, c.dpad_tc,
                                    c.wtiles, 0, g.T, c.q, c.nrm, c.q, c.nrm, pfull, c.kp, c.invC, c.scal, g.m1,
                                    c.Ypart, brows, c.cur_ctrl);
            ++c.launches;
            return true;
        }
        tc_dispatch<TC_MATVEC>(c.kp.kernel, c.ntiles, c.s, c.tm_hi, c.tm_lo, c.tm_hi, c.tm_lo, c.dpad_tc, c.tiles, 0, c.q,
                               c.nrm, c.q, c.nrm, pfull, c.kp, c.invC, c.scal, g.m1, b0, b1, c.Ypart, brows,
                               static_cast<float *>(nullptr), g.T, c.cur_ctrl);
        ++c.launches;
        return true;
    }
    return false;
}

template <typename T>
bool launch_tc_precompute(Ctx<T> &c) {
    if constexpr (std::is_same<T, float>::value) {
        const Geometry &g = c.g;
        tc_dispatch<TC_PRECOMPUTE>(c.kp.kernel, c.ntiles, c.s, c.tm_hi, c.tm_lo, c.tm_hi, c.tm_lo, c.dpad_tc, c.tiles, 0,
                                   c.q, c.nrm, c.q, c.nrm, static_cast<const float *>(nullptr), c.kp, c.invC, c.scal,
                                   g.m1, g.band0, g.band1, static_cast<float *>(nullptr), g.nb, c.Qc,
                                   c.packed ? -1 : g.T, static_cast<const int *>(nullptr));
        ++c.launches;
        return true;
    }
    return false;
}

// Cached GEMV split-K factor: >= 16 CTAs per SM in total (several waves of the ~3 resident
// CTAs per SM), so the last partial wave costs little even when the band has few row blocks.
int gemv_splits(const Geometry &g) {
    const int rowblocks = static_cast<int>(g.nb / kTile);
    return std::max(1, std::min(g.T, static_cast<int>(ceil_div(16 * 148, rowblocks))));
}

// Q~ times the full vector `pfull` -> Ypart (slots) ; returns the number of slots to finalize.
template <typename T>
int launch_qtilde_product(Ctx<T> &c, const T *pfull) {
    const Geometry &g = c.g;
    if (c.cached && c.packed) {
        const int b0p = c.circ ? 0 : g.band0;
        const int64_t brows = c.circ ? g.mpad : g.nb;
        if (c.circ) PLS_CUDA(cudaMemsetAsync(c.Ypart, 0, static_cast<size_t>(g.T) * g.mpad * sizeof(T), c.s));
        constexpr int per_cta = 4;  // stored tiles per CTA (amortises launch + reduction bubbles)
        k_gemv_sym<T><<<static_cast<unsigned>(ceil_div(c.nstored, per_cta)), 256, 0, c.s>>>(
            c.Qc, c.tiles, c.nsub_eff, c.nstored, per_cta, pfull, b0p, brows, c.Ypart, c.cur_ctrl);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        if (!c.circ) {
            c.Yfin = c.Ypart;
            return g.T;
        }
        k_slot_sum<T><<<c.vb, kVecThreads, 0, c.s>>>(c.Ypart, g.T, g.mpad, g.m1, c.yfull, c.cur_ctrl);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        timed_comm(c, [&] { comm_reduce_scatter(c.comm, c.yfull, c.ysc, g.nb, dtype_of(T()), c.s); });
        c.Yfin = c.ysc;
        return 1;
    }
    if (c.cached) {
        const int rowblocks = static_cast<int>(g.nb / kTile);
        k_gemv_tiled<T><<<rowblocks * c.nsplit, 256, 0, c.s>>>(c.Qc, pfull, g.T, c.nsplit, g.nb, c.Ypart,
                                                                c.cur_ctrl);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        return c.nsplit;
    }
    if (c.lowrank) {  // Q~p = B^T (X (X^T (B p))) + (p + 1 sum p)/C, O(md)
        const int64_t r0 = g.g0, r1 = std::max<int64_t>(std::min<int64_t>(g.g0 + g.nb, c.m), g.g0);
        // X^T B p = sum_{i < m-1} p_i x_i - (sum p) x_{m-1}: the column sums of this rank's rows (and the
        // slices of sum p), then the fixed-order reduce, which adds the x_{m-1} term on the rank holding it
        const bool owns_last = c.m - 1 >= r0 && c.m - 1 < r1;
        k_colsum_partial<T><<<c.lr_parts, 256, 0, c.s>>>(c.Xraw, c.d, r0, r1, c.lr_rpb, nullptr, pfull, c.m, c.tpart,
                                                         c.psum, c.cur_ctrl);
        k_colsum_reduce<T><<<static_cast<unsigned>(ceil_div(c.d, 256)), 256, 0, c.s>>>(
            c.tpart, c.lr_parts, c.d, c.tvec, c.tloc, c.cur_ctrl, c.psum, owns_last ? c.Xraw + (c.m - 1) * c.d : nullptr,
            c.scal);
        PLS_CHECK_LAUNCH();
        c.launches += 2;
        if (c.comm) {  // t = sum over ranks (out of place: idempotent after convergence)
            comm_allreduce_sum_f64(c.comm, c.tloc, c.tloc + c.d, c.d, c.s);
            k_cast<T><<<static_cast<unsigned>(ceil_div(c.d, 256)), 256, 0, c.s>>>(c.tloc + c.d, c.d, c.tvec);
            PLS_CHECK_LAUNCH();
            ++c.launches;
        }
        k_lastdot<T><<<1, 256, 0, c.s>>>(c.Xraw + (c.m - 1) * c.d, c.tvec, c.d, c.scal, c.cur_ctrl);
        k_rowdot<T><<<static_cast<unsigned>(ceil_div(g.nb * 32, 256)), 256, 0, c.s>>>(
            c.Xraw, c.d, g.g0, g.nb, c.tvec, 1, T(0), pfull, c.m, c.invC, c.scal, c.Ypart, nullptr, c.cur_ctrl);
        PLS_CHECK_LAUNCH();
        c.launches += 2;
        c.Yfin = c.Ypart;
        return 1;
    }
    // circulant multi-GPU: partial products for ALL rows (band = everything), zero-initialised
    const int b0 = c.circ ? 0 : g.band0, b1 = c.circ ? g.T : g.band1;
    const int64_t brows = c.circ ? g.mpad : g.nb;
    const int nslots = g.T * c.nsub_eff;
    if (c.circ) PLS_CUDA(cudaMemsetAsync(c.Ypart, 0, static_cast<size_t>(nslots) * g.mpad * sizeof(T), c.s));
    if (c.tc) {
        launch_tc<T>(c, pfull, b0, b1, brows);
    } else if (launch_oz<T>(c, pfull, b0, b1, brows, false)) {
        // fp64 on the int8 tensor cores
    } else {
        const size_t sm = Engine<T>::SMEM_BYTES;
        switch (c.kp.kernel) {
            case LINEAR:
                k_matvec_implicit<LINEAR, T><<<c.ntiles, Engine<T>::THREADS, sm, c.s>>>(
                    c.ops, g.dpad, c.tiles, c.q, c.nrm, pfull, c.kp, c.invC, c.scal, g.m1, b0, b1, c.Ypart, brows,
                    c.cur_ctrl);
                break;
            case POLYNOMIAL:
                k_matvec_implicit<POLYNOMIAL, T><<<c.ntiles, Engine<T>::THREADS, sm, c.s>>>(
                    c.ops, g.dpad, c.tiles, c.q, c.nrm, pfull, c.kp, c.invC, c.scal, g.m1, b0, b1, c.Ypart, brows,
                    c.cur_ctrl);
                break;
            default:
                k_matvec_implicit<RBF, T><<<c.ntiles, Engine<T>::THREADS, sm, c.s>>>(
                    c.ops, g.dpad, c.tiles, c.q, c.nrm, pfull, c.kp, c.invC, c.scal, g.m1, b0, b1, c.Ypart, brows,
                    c.cur_ctrl);
        }
        PLS_CHECK_LAUNCH();
        ++c.launches;
    }
    if (!c.circ) {
        c.Yfin = c.Ypart;
        return nslots;
    }
    k_slot_sum<T><<<c.vb, kVecThreads, 0, c.s>>>(c.Ypart, nslots, g.mpad, g.m1, c.yfull, c.cur_ctrl);
    PLS_CHECK_LAUNCH();
    ++c.launches;
    timed_comm(c, [&] { comm_reduce_scatter(c.comm, c.yfull, c.ysc, g.nb, dtype_of(T()), c.s); });
    c.Yfin = c.ysc;
    return 1;
}

template <typename T>
void launch_precompute(Ctx<T> &c) {
    if (c.tc && launch_tc_precompute<T>(c)) return;
    if (launch_oz<T>(c, static_cast<const T *>(nullptr), 0, 0, 0, true)) return;
    const Geometry &g = c.g;
    const size_t sm = Engine<T>::SMEM_BYTES;
    switch (c.kp.kernel) {
        case LINEAR:
            k_precompute<LINEAR, T><<<c.ntiles, Engine<T>::THREADS, sm, c.s>>>(c.ops, g.mpad, g.dpad, c.tiles, c.q, c.nrm, c.kp,
                                                                    c.invC, c.scal, g.m1, g.band0, g.band1, c.Qc, c.packed ? 1 : 0);
            break;
        case POLYNOMIAL:
            k_precompute<POLYNOMIAL, T><<<c.ntiles, Engine<T>::THREADS, sm, c.s>>>(c.ops, g.mpad, g.dpad, c.tiles, c.q, c.nrm, c.kp,
                                                                        c.invC, c.scal, g.m1, g.band0, g.band1, c.Qc, c.packed ? 1 : 0);
            break;
        default:
            k_precompute<RBF, T><<<c.ntiles, Engine<T>::THREADS, sm, c.s>>>(c.ops, g.mpad, g.dpad, c.tiles, c.q, c.nrm, c.kp,
                                                                 c.invC, c.scal, g.m1, g.band0, g.band1, c.Qc, c.packed ? 1 : 0);
    }
    PLS_CHECK_LAUNCH();
    ++c.launches;
}

template <typename T>
void finalize(Ctx<T> &c, int nslots, const T *pband, int mode, T *pout, int par, int set_delta0) {
    const Geometry &g = c.g;
    const T *Y = c.Yfin;
    int nsub = (c.cached || c.circ) ? 1 : c.nsub_eff;
    if constexpr (std::is_same<T, double>::value) {
        if (c.fsplit) {
            // this rank's partial product (its feature slice) -> sum over the ranks,
            // then the usual finalize on the summed vector (one slot)
            k_finalize<T><<<c.vb, kVecThreads, 0, c.s>>>(Y, nslots, nsub, g.band0, g.nb, g.g0, g.m1, c.p + g.g0,
                                                               c.yred, 0, c.ylab, c.r, nullptr, c.scal, 0, 0,
                                                               c.partials, c.counter, 0, c.cur_ctrl, S_PAP);
            PLS_CHECK_LAUNCH();
            ++c.launches;
            timed_comm(c, [&] { comm_allreduce_sum_f64(c.comm, c.yred, c.yred, g.nb, c.s); });
            Y = c.yred;
            nslots = 1;
            nsub = 1;
        }
    }
    k_finalize<T><<<c.vb, kVecThreads, 0, c.s>>>(Y, nslots, nsub, g.band0, g.nb, g.g0, g.m1, pband, c.y, mode,
                                                       c.ylab, c.r, pout, c.scal, par, set_delta0, c.partials,
                                                       c.counter, 1, c.cur_ctrl, c.pap_slot);
    PLS_CHECK_LAUNCH();
    ++c.launches;
}

// Row-sharded exchanges; with the feature split the CG vectors and scalars are replicated.
template <typename T>
void allreduce(Ctx<T> &c, int slot, int count) {
    if (c.comm && !c.fsplit)
        timed_comm(c, [&] { comm_allreduce_sum_f64(c.comm, c.scal + slot + S_L, c.scal + slot, count, c.s); });
}
template <typename T>
void allgather(Ctx<T> &c, T *full) {
    if (c.comm && !c.fsplit) timed_comm(c, [&] { comm_allgather(c.comm, full, c.g.nb, dtype_of(T()), c.s); });
}

// Common setup: geometry, buffers, H2D, transform, q.  Returns the context.
template <typename T>
void setup(Ctx<T> &c, Arena &A, const Problem &pb, const plssvm_options_t &o, bool need_labels, Events &E,
           cudaEvent_t e_h2d, cudaEvent_t e_tr, cudaEvent_t e_q) {
    int P = 1, rank = 0;
    c.nranks = c.comm ? comm_size(c.comm) : 1;
    c.fsplit = c.nranks > 1 && o.multi_gpu == PLSSVM_MULTI_GPU_FEATURES;
    if (c.comm && !c.fsplit) {
        P = comm_size(c.comm);
        rank = comm_rank(c.comm);
    }
    // Feature split (paper §III-C5): all points, features [f0, f0 + dl) of this rank; the 1/C
    // terms of Eq. 16 (delta_ij/C and the 1/C inside Q_mm) are added by rank 0 only, so the sum
    // of the ranks' partial products is Q~p exactly once.
    int64_t f0 = 0, dl = pb.d;
    bool root = true;
    if (c.fsplit) {
        const int fr = comm_rank(c.comm);
        f0 = feature_begin(pb.d, c.nranks, fr);
        dl = feature_begin(pb.d, c.nranks, fr + 1) - f0;
        root = fr == 0;
    }
    c.g = geometry<T>(pb.m, dl, P, rank);
    c.vb = static_cast<int>(std::min<int64_t>(kVecBlocks, std::max<int64_t>(1, ceil_div(c.g.nb, 64))));
    const Geometry &g = c.g;
    c.kp = KParams<T>{pb.kernel, static_cast<T>(pb.gamma), pb.degree, static_cast<T>(pb.coef0)};
    c.invC = root ? static_cast<T>(1.0 / pb.C) : T(0);
    const bool dev = o.device_pointers != 0;
    const T *Xs = nullptr;
    if (c.fsplit) {  // strided copy of the column slice X[:, f0:f0+dl]
        T *sl = A.alloc<T>(pb.m * dl);
        PLS_CUDA(cudaMemcpy2DAsync(sl, dl * sizeof(T), static_cast<const T *>(pb.X) + f0, pb.d * sizeof(T),
                                   dl * sizeof(T), pb.m, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.s));
        Xs = sl;
    } else {
        Xs = stage_input<T>(A, pb.X, pb.m * pb.d, dev, c.s);
    }
    c.Xraw = Xs;
    c.m = pb.m;
    c.d = dl;
    RowStats rho;  // largest row peak / exponent of X (this rank's slice), for the engine choice
    if (need_labels) {
        c.ylab = const_cast<T *>(stage_input<T>(A, pb.y, pb.m, dev, c.s));
        rho = validate_inputs<T>(A, {VCheck<T>{Xs, pb.m * dl, V_NONFINITE_X, dl}}, c.ylab, pb.m, c.s, c.launches);
    } else {
        c.ylab = A.alloc<T>(pb.m);
        PLS_CUDA(cudaMemsetAsync(c.ylab, 0, pb.m * sizeof(T), c.s));
        rho = validate_inputs<T>(A, {VCheck<T>{Xs, pb.m * dl, V_NONFINITE_X, dl}}, static_cast<const T *>(nullptr), 0,
                                 c.s, c.launches);
    }
    PLS_CUDA(cudaEventRecord(e_h2d, c.s));
    // The int8 engines split the caller's row-major X directly (padding rows read as 0) and the q /
    // norm pass reads it too: no transformed copy.  The other engines use the transformed layout.
    if constexpr (std::is_same<T, double>::value) {
        c.oz = oz_choose(o.fp64_engine, rho, g.mpad, dl);
        if (c.oz) {
            c.ozx = oz_prepare<7, double>(A, Xs, g.mpad, pb.m, dl, dl, true, true, c.s, c.launches);
            oz_set_attrs<double>();
        }
    } else {
        if (o.fp32_engine == PLSSVM_FP32_OZAKI || o.fp32_engine == PLSSVM_FP32_AUTO) {
            c.oz = oz_choose_f32(o.fp32_engine, rho, dl);  // fp32 on the int8 tensor cores (3 digits)
            if (c.oz) {
                c.ozx = oz_prepare<3, float>(A, Xs, g.mpad, pb.m, dl, dl, true, true, c.s, c.launches);
                oz_set_attrs<float>();
            }
        }
        c.tc = !c.oz && o.fp32_engine != PLSSVM_FP32_FFMA;
        if (c.tc) setup_tc<T>(c, A, Xs, pb.m, dl);
    }
    if (!c.oz) {
        c.Xt = A.alloc<T>(g.dpad * g.mpad);
        launch_transform<T>(Xs, pb.m, dl, c.Xt, g.mpad, g.dpad, c.s, c.launches);
        c.ops = make_ops(c.Xt, g.mpad, c.Xt, g.mpad, g.ld);
    }
    PLS_CUDA(cudaEventRecord(e_tr, c.s));
    c.q = A.alloc<T>(g.mpad);
    c.nrm = A.alloc<T>(g.mpad);
    c.scal = A.alloc<double>(S_COUNT);
    PLS_CUDA(cudaMemsetAsync(c.scal, 0, S_COUNT * sizeof(double), c.s));
    // (int8 engines: from the caller's row-major X, row stride dl)
    k_q_norms<T><<<static_cast<unsigned>(ceil_div(g.mpad * 32, 256)), 256, 0, c.s>>>(
        c.oz ? Xs : c.Xt, g.mpad, g.dpad, pb.m, dl, c.kp, c.invC, c.ylab, c.q, c.nrm, c.scal, c.oz ? dl : 0);
    PLS_CHECK_LAUNCH();
    ++c.launches;
    PLS_CUDA(cudaEventRecord(e_q, c.s));
    c.partials = A.alloc<T>(2 * kVecBlocks);  // (k_cg_fused: one array per reduction)
    c.counter = A.alloc<unsigned>(1);
    PLS_CUDA(cudaMemsetAsync(c.counter, 0, sizeof(unsigned), c.s));
    std::vector<int2> tl = band_tiles(g, c.oz ? OzC::NSUB : Engine<T>::NSUB);
    c.ntiles = static_cast<int>(tl.size());
    c.tiles = A.alloc<int2>(c.ntiles);
    upload(c.tiles, tl.data(), tl.size(), c.s);
    oz_build_pairs<T>(c, A, tl, g.band0, g.band1);
    set_smem_attrs<T>();
}

// Product configuration once the mode is known: slot buffers, and for implicit multi-GPU the
// circulant tile list (+ full-length partial product and reduce-scatter target).
template <typename T>
void configure_product(Ctx<T> &c, Arena &A) {
    const Geometry &g = c.g;
    c.nsub_eff = c.tc ? 1 : c.oz ? OzC::NSUB : Engine<T>::NSUB;
    c.nsplit = gemv_splits(g);
    c.circ = g.P > 1 && !c.lowrank && (!c.cached || c.packed) && comm_has_reduce_scatter(c.comm);
    if (c.fsplit) c.yred = A.alloc<T>(g.nb);
    if (c.lowrank) {
        const int64_t r0 = g.g0, r1 = std::min<int64_t>(g.g0 + g.nb, c.m);
        const int64_t rows = std::max<int64_t>(r1 - r0, 1);
        c.lr_rpb = std::max<int64_t>(1, ceil_div(rows, 4 * 148));
        c.lr_parts = static_cast<int>(ceil_div(rows, c.lr_rpb));
        c.tpart = A.alloc<T>(static_cast<int64_t>(c.lr_parts) * c.d);
        c.tvec = A.alloc<T>(c.d);
        c.tloc = A.alloc<double>(2 * c.d);
        c.psum = A.alloc<double>(c.lr_parts);
        c.Ypart = A.alloc<T>(g.nb);
        c.Yfin = c.Ypart;
        return;
    }
    if (c.circ) {
        std::vector<int2> tl = circulant_tiles(g, c.nsub_eff);
        c.ntiles = static_cast<int>(tl.size());
        c.tiles = A.alloc<int2>(c.ntiles);
        upload(c.tiles, tl.data(), tl.size(), c.s);
        oz_build_pairs<T>(c, A, tl, g.band0, g.band1);
        c.Ypart = A.alloc<T>(static_cast<int64_t>(g.T) * c.nsub_eff * g.mpad);
        c.yfull = A.alloc<T>(g.mpad);
        c.ysc = A.alloc<T>(g.nb);
    } else if (c.packed) {
        c.Ypart = A.alloc<T>(static_cast<int64_t>(g.T) * g.nb);
    } else {
        c.Ypart = A.alloc<T>(static_cast<int64_t>(c.cached ? c.nsplit : g.T * c.nsub_eff) * g.nb);
    }
    c.nstored = c.packed ? c.ntiles / c.nsub_eff : 0;
    c.Yfin = c.Ypart;
    c.wide = c.tc && g.P == 1 && !c.cached && !c.lowrank && !c.circ && c.wide_ok;
    if (c.wide) {
        std::vector<int2> wl = wide_tiles(g.T);
        c.nwtiles = static_cast<int>(wl.size());
        c.wtiles = A.alloc<int2>(c.nwtiles);
        upload(c.wtiles, wl.data(), wl.size(), c.s);
    }
}

// Stored 128 x 128 tiles of the packed layout for this rank (upper triangle for one GPU, the
// circulant pairs otherwise) -- computed without building the list, for the fit test.
int64_t packed_tile_count(const Geometry &g) {
    if (g.P == 1) return static_cast<int64_t>(g.T) * (g.T + 1) / 2;
    int64_t n = 0;
    const int half = g.T / 2;
    for (int I = g.band0; I < g.band1; ++I) n += half + 1 - ((g.T % 2 == 0 && I >= half) ? 1 : 0);
    return n;
}

// Mode selection (north_star: "mode picked by measurement"; SURVEY §8 decision 8): cached
// whenever the Q~ band fits the budget -- the precompute costs about one implicit product and
// every later product becomes an HBM stream (≈ 50-100x cheaper than a recompute).
template <typename T>
bool choose_cached(const Geometry &g, const plssvm_options_t &o, CommHandle *comm, cudaStream_t s, int64_t need) {
    if (o.mode == PLSSVM_MODE_IMPLICIT) return false;
    // memory this process' stream-ordered pool holds but does not use counts as free (it is
    // reused by the allocation below without re-mapping; trimming it would cost ~1 s per 100 GB)
    int dev = 0;
    PLS_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    uint64_t pool_idle = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t reserved = 0, used = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        pool_idle = reserved > used ? reserved - used : 0;
    }
    size_t free_b = 0, total_b = 0;
    PLS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    free_b += pool_idle;
    int64_t budget = o.cache_budget_bytes > 0 ? o.cache_budget_bytes : static_cast<int64_t>(0.9 * free_b);
    budget = std::min<int64_t>(budget, static_cast<int64_t>(free_b) - (int64_t(1) << 28));
    bool fits = need <= budget;
    if (comm) {  // every rank must take the same decision (the collectives differ between modes)
        double *buf = nullptr;
        PLS_CUDA(cudaMallocAsync(&buf, 2 * sizeof(double), s));
        const double one = fits ? 1.0 : 0.0;
        double all = 0.0;
        PLS_CUDA(cudaMemcpyAsync(buf, &one, sizeof(double), cudaMemcpyHostToDevice, s));
        comm_allreduce_sum_f64(comm, buf, buf + 1, 1, s);
        PLS_CUDA(cudaMemcpyAsync(&all, buf + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
        PLS_CUDA(cudaStreamSynchronize(s));
        PLS_CUDA(cudaFreeAsync(buf, s));
        fits = all >= comm_size(comm) - 0.5;
    }
    if (fits) return true;
    if (o.mode == PLSSVM_MODE_CACHED)
        throw Error(PLSSVM_E_OOM, "cached mode: Q~ band of " + std::to_string(need) + " bytes does not fit (" +
                                      std::to_string(budget) + " available on this rank)");
    return false;
}

// Mode: LOWRANK if asked; else cached when the Q~ storage fits (symmetric-packed tiles when one
// GPU or a reduce-scatter is available: half the bytes of full rows), else implicit.
template <typename T>
void select_mode(Ctx<T> &c, const plssvm_options_t &o) {
    const Geometry &g = c.g;
    c.lowrank = o.mode == PLSSVM_MODE_LOWRANK;
    if (c.fsplit) {  // the paper's feature split recomputes the partial entries
        c.lowrank = c.cached = c.packed = false;
        return;
    }
    const bool can_pack = g.P == 1 || (c.comm && comm_has_reduce_scatter(c.comm));
    const int64_t need = (can_pack ? packed_tile_count(g) * kTile * kTile : g.nb * g.mpad) * static_cast<int64_t>(sizeof(T));
    c.cached = !c.lowrank && choose_cached<T>(g, o, c.comm, c.s, need);
    c.packed = c.cached && can_pack;
}

// delta of the current iterate from a control snapshot (Shewchuk: double-buffered by parity).
double delta_now(const double *hs, int64_t it, bool cgcg) { return cgcg ? hs[S_CG_GAMMA] : hs[S_DELTA + (it & 1)]; }

template <typename T>
int train_impl(const Problem &pb, const plssvm_options_t &o, void *alpha_out, void *b_out, plssvm_stats_t *st) {
    PLS_CUDA(cudaSetDevice(o.device));
    upload_reset();
    setup_mempool(o.device);
    StreamGuard sg(o.stream);
    Ctx<T> c{};
    c.s = sg.s;
    c.comm = static_cast<CommHandle *>(o.comm);
    Arena A(c.s);
    Events E;
    cudaEvent_t e0 = E.make(), e_h2d = E.make(), e_tr = E.make(), e_q = E.make(), e_alloc = E.make(), e_pre = E.make(),
                e_cg = E.make(), e_end = E.make();
    const auto wall0 = std::chrono::steady_clock::now();
    PLS_CUDA(cudaEventRecord(e0, c.s));
    {
        Nvtx r("plssvm setup: stage, validate, split, q");
        setup<T>(c, A, pb, o, true, E, e_h2d, e_tr, e_q);
    }
    const Geometry &g = c.g;

    c.x = A.alloc<T>(g.nb);
    c.r = A.alloc<T>(g.nb);
    c.y = A.alloc<T>(g.nb);
    // one process per GPU over NCCL: p in the communicator's symmetric window, so the p update stores
    // every rank's band straight into every rank's p (k_update_p_lsa: the all-gather fused in)
    c.p = nullptr;
    if (c.comm && !c.fsplit && o.cg_variant != PLSSVM_CG_SINGLE_REDUCTION && o.replace_every <= 0)
        c.p = static_cast<T *>(comm_lsa_buffer(c.comm, static_cast<size_t>(g.mpad) * sizeof(T)));
    c.lsa = c.p != nullptr;
    if (!c.p) c.p = A.alloc<T>(g.mpad);
    c.xfull = A.alloc<T>(g.mpad);
    PLS_CUDA(cudaMemsetAsync(c.p, 0, g.mpad * sizeof(T), c.s));
    T *pband = c.p + g.g0;

    select_mode<T>(c, o);
    configure_product<T>(c, A);
    if (c.cached) c.Qc = A.alloc<T>(c.packed ? c.nstored * kTile * kTile : g.nb * g.mpad);
    PLS_CUDA(cudaEventRecord(e_alloc, c.s));
    if (c.cached) {
        Nvtx r("plssvm precompute");
        launch_precompute<T>(c);
    }
    PLS_CUDA(cudaEventRecord(e_pre, c.s));

    // ---- CG init (a2) ----
    const int64_t imax = o.max_iter > 0 ? o.max_iter : g.m1;
    if (o.x0 == 0) {
        k_init<T><<<c.vb, kVecThreads, 0, c.s>>>(c.x, c.r, pband, c.ylab, g.nb, g.g0, g.m1, T(0), 1, c.scal,
                                                       c.partials, c.counter, 1);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        allreduce(c, S_DELTA0, 2);
    } else {
        k_init<T><<<c.vb, kVecThreads, 0, c.s>>>(c.x, c.r, pband, c.ylab, g.nb, g.g0, g.m1, T(1), 0, c.scal,
                                                       c.partials, c.counter, 1);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        PLS_CUDA(cudaMemcpyAsync(c.xfull + g.g0, c.x, g.nb * sizeof(T), cudaMemcpyDeviceToDevice, c.s));
        allgather(c, c.xfull);
        const int ns = launch_qtilde_product<T>(c, c.xfull);
        finalize<T>(c, ns, nullptr, 1, pband, 0, 1);  // r = rhs - Q~x0, p = r, delta0
        allreduce(c, S_DELTA0, 2);
    }
    allgather(c, c.p);

    // ---- CG loop (a3-a5, a8): the convergence test runs on the device (k_update_p), the host
    // enqueues iterations in batches of kBatch and reads the control block once per batch --
    // no host round trip per iteration; iterations enqueued after convergence are no-ops.
    Nvtx r_cg("plssvm CG loop, bias, alpha");  // (to the end of the call)
    c.ctrl = A.alloc<int>(C_COUNT);
    const int imax_i = static_cast<int>(std::min<int64_t>(imax, INT32_MAX));
    const int fixed_i = static_cast<int>(std::min<int64_t>(std::max<int64_t>(o.fixed_iter, 0), INT32_MAX));
    const int repl_i = static_cast<int>(std::min<int64_t>(std::max<int64_t>(o.replace_every, 0), INT32_MAX));
    k_cg_start<<<1, 1, 0, c.s>>>(c.scal, c.ctrl, pb.eps * pb.eps, imax_i, fixed_i, repl_i);
    PLS_CHECK_LAUNCH();
    ++c.launches;
    // residual trace (options.residual_trace, SPEC CGTrace): delta_k copied on the stream after
    // every iteration's update (the global scalar slots), square roots taken on the host at the end
    const bool want_trace = o.residual_trace != nullptr && o.residual_trace_len > 0;
    if (want_trace && o.cg_variant == PLSSVM_CG_SINGLE_REDUCTION)
        throw Error(PLSSVM_E_INVALID_ARG, "options.residual_trace needs the Shewchuk CG variant");
    const int64_t trace_n = want_trace ? std::min<int64_t>(o.residual_trace_len, imax + 1) : 0;
    double *trace_d = want_trace ? A.alloc<double>(trace_n) : nullptr;
    if (want_trace)
        PLS_CUDA(cudaMemcpyAsync(trace_d, c.scal + S_DELTA0, sizeof(double), cudaMemcpyDeviceToDevice, c.s));
    double *hs = reinterpret_cast<double *>(pinned_scratch(S_COUNT * sizeof(double) + C_COUNT * sizeof(int)));
    int *hctrl = reinterpret_cast<int *>(hs + S_COUNT);
    const int64_t launches_before_cg = c.launches;
    // Batches: the first has kBatch iterations; each later one is sized from the convergence rate of
    // the previous batch (the iterations still needed to reach delta <= eps^2 delta_0, + 1), so a
    // C1 training takes 2-3 host round trips instead of one per 8 iterations, with few no-op
    // iterations at the end (one GPU; several ranks keep batches of kBatch).
    constexpr int kBatch = 8, kBatchMax = 32;
    constexpr int kCommEv = 12;  // event slots per iteration for collectives (<= 5 collectives)
    // Two event sets, alternating by batch: the host reads a batch's launch times (cudaEventElapsedTime,
    // ~2.7 us per call, profiles/r02_host_api_cost.txt) while the GPU runs the next batch, and the last
    // batch's while it runs the bias / alpha kernels -- not at a batch boundary with the GPU idle.
    const int kSet = 2 * kBatchMax + (c.comm ? kBatchMax * kCommEv : 0);
    cudaEvent_t *evp = event_pool(2 * kSet);
    auto mv0 = [&](int set) { return evp + set * kSet; };
    auto mv1 = [&](int set) { return evp + set * kSet + kBatchMax; };
    auto cev = [&](int set, int b) { return evp + set * kSet + 2 * kBatchMax + b * kCommEv; };
    int ncev[2][kBatchMax] = {};
    int pend_set = -1, pend_n = 0;  // the batch whose events are complete but not read yet
    double t_comm = 0.0;
    double t_mv = 0.0, t_mv_min = 1e30;
    int64_t it = 0;
    c.cur_ctrl = c.ctrl;
    // One CG iteration (a3 product, a4 fused updates, a5 test in k_update_p, a8 exchanges).
    // k = host-side iteration index (only the residual-replacement period uses it); `loop` /
    // `use_loop`: the CUDA-graph WHILE condition k_update_p sets.
    // Chronopoulos-Gear variant: c.p (full) carries r (the product's operand), c.r (band) the
    // search direction p, scg the recurrence s = Q~ p; one all-reduce of (gamma, delta).
    const bool cgcg = o.cg_variant == PLSSVM_CG_SINGLE_REDUCTION;
    auto read_times = [&]() {  // the pending batch's product (and collective) times
        if (pend_set < 0) return;
        for (int b = 0; b < pend_n; ++b) {
            const double tm = elapsed(mv0(pend_set)[b], mv1(pend_set)[b]);
            t_mv += tm;
            t_mv_min = std::min(t_mv_min, tm);
            for (int k = 0; k + 1 < ncev[pend_set][b]; k += 2)
                t_comm += elapsed(cev(pend_set, b)[k], cev(pend_set, b)[k + 1]);
        }
        pend_set = -1;
    };
    // one cooperative launch for the vector work of an iteration: one GPU, no exchange, no residual
    // replacement (the three-kernel sequence otherwise; PLSSVM_CG_UNFUSED=1 forces it for A/B runs)
    const bool unfused_env = std::getenv("PLSSVM_CG_UNFUSED") != nullptr;  // (read per call: the A/B test)
    const bool fused = !cgcg && c.comm == nullptr && !c.fsplit && o.replace_every <= 0 && c.npeer == 0 && !unfused_env;
    if (c.comm && comm_is_peer(c.comm) && comm_peer_direct(c.comm) && !c.fsplit && !cgcg) {
        // fused all-gather of p (PEER transport): learn every rank's p buffer once
        std::vector<void *> all = comm_peer_exchange_ptr(c.comm, c.p);
        c.npeer = static_cast<int>(all.size());
        c.peer_p = A.alloc<T *>(c.npeer);
        upload(reinterpret_cast<void **>(c.peer_p), all.data(), all.size(), c.s);
    }
    T *scg = nullptr;
    if (cgcg) {
        scg = A.alloc<T>(g.nb);
        PLS_CUDA(cudaMemsetAsync(scg, 0, g.nb * sizeof(T), c.s));
        c.pap_slot = S_CG_DELTA;
    }
    auto trace_after = [&](int64_t k) {  // delta_{k+1} -> trace[k + 1]
        if (trace_d && k + 1 < trace_n)
            PLS_CUDA(cudaMemcpyAsync(trace_d + k + 1, c.scal + S_DELTA + ((k & 1) ^ 1), sizeof(double),
                                     cudaMemcpyDeviceToDevice, c.s));
    };
    auto enqueue_iteration = [&](int64_t k, cudaEvent_t ev0, cudaEvent_t ev1, cudaGraphConditionalHandle loop,
                                 int use_loop) {
        if (cgcg) {
            if (ev0) PLS_CUDA(cudaEventRecord(ev0, c.s));
            const int ns = launch_qtilde_product<T>(c, c.p);  // w = Q~ r
            if (ev1) PLS_CUDA(cudaEventRecord(ev1, c.s));
            finalize<T>(c, ns, pband, 0, nullptr, 0, 0);  // w -> c.y, delta = w.r (partial)
            allreduce(c, S_CG_GAMMA, 2);                   // (gamma, delta): the one reduction
            k_cgcg_update<T><<<c.vb, kVecThreads, 0, c.s>>>(c.x, pband, c.r, scg, c.y, g.nb, c.scal, c.ctrl,
                                                                  c.partials, c.counter, loop, use_loop);
            PLS_CHECK_LAUNCH();
            ++c.launches;
            allgather(c, c.p);
            return;
        }
        const int par = static_cast<int>(k & 1);
        if (ev0) PLS_CUDA(cudaEventRecord(ev0, c.s));
        const int ns = launch_qtilde_product<T>(c, c.p);
        if (ev1) PLS_CUDA(cudaEventRecord(ev1, c.s));
        if (fused) {  // finalize + update_xr + update_p as one cooperative launch (bit-identical)
            const T *Yf = c.Yfin;
            const int nsub = (c.cached || c.circ) ? 1 : c.nsub_eff;
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(c.vb);
            lc.blockDim = dim3(kVecThreads);
            lc.stream = c.s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            PLS_CUDA(cudaLaunchKernelEx(&lc, k_cg_fused<T>, Yf, ns, nsub, g.band0, g.nb, g.g0, g.m1, c.x, c.r, pband,
                                        c.y, c.scal, c.ctrl, c.partials, loop, use_loop));
            ++c.launches;
            trace_after(k);
            return;
        }
        finalize<T>(c, ns, pband, 0, nullptr, 0, 0);
        allreduce(c, S_PAP, 1);
        k_update_xr<T><<<c.vb, kVecThreads, 0, c.s>>>(c.x, c.r, pband, c.y, g.nb, c.scal, c.ctrl, c.partials,
                                                            c.counter);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        allreduce(c, S_DELTA + (par ^ 1), 1);
        if (o.replace_every > 0 && k > 0 && k % o.replace_every == 0) {
            // explicit residual r = rhs - Q~x (Shewchuk B2 replacement, option R > 0)
            PLS_CUDA(cudaMemcpyAsync(c.xfull + g.g0, c.x, g.nb * sizeof(T), cudaMemcpyDeviceToDevice, c.s));
            allgather(c, c.xfull);
            const int ns2 = launch_qtilde_product<T>(c, c.xfull);
            finalize<T>(c, ns2, nullptr, 1, nullptr, -1, 0);
            allreduce(c, S_DELTA + (par ^ 1), 1);
        }
        if (c.lsa) {  // fused all-gather through the NCCL device API (stores + LSA barrier in the kernel)
            k_update_p_lsa<T><<<c.vb, kVecThreads, 0, c.s>>>(pband, c.r, g.nb, c.scal, c.ctrl, c.counter,
                                                                   *comm_lsa_devcomm(c.comm), comm_lsa_window(c.comm),
                                                                   g.g0);
            PLS_CHECK_LAUNCH();
            ++c.launches;
            trace_after(k);
            return;
        }
        k_update_p<T><<<c.vb, kVecThreads, 0, c.s>>>(pband, c.r, g.nb, c.scal, c.ctrl, c.counter, loop,
                                                           use_loop, c.peer_p, c.npeer, g.g0);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        trace_after(k);
        if (c.npeer > 0)  // p already stored into every rank's buffer: only the cross-device order remains
            timed_comm(c, [&] { comm_peer_fence(c.comm, c.s); });
        else
            allgather(c, c.p);
    };
    const bool graph_ok = c.comm == nullptr && o.replace_every <= 0 && !want_trace;
    const bool use_graph = graph_ok && (o.cg_loop == PLSSVM_CG_GRAPH ||
                                        (o.cg_loop == PLSSVM_CG_AUTO && (c.cached || c.lowrank || g.m1 <= 8192)));
    if (o.cg_loop == PLSSVM_CG_GRAPH && !graph_ok)
        throw Error(PLSSVM_E_INVALID_ARG,
                    "cg_loop GRAPH needs a single GPU (no comm), replace_every = 0 and no residual_trace");
    if (use_graph) {
        // The whole loop as ONE graph launch: entry kernel sets the WHILE
        // condition from the control block, the body (captured once) is one iteration, and
        // k_update_p's last block clears the condition when Shewchuk's loop condition fails.
        cudaStream_t cap = nullptr;
        cudaGraph_t G = nullptr;
        cudaGraphExec_t GE = nullptr;
        struct GraphFree {
            cudaStream_t &s;
            cudaGraph_t &g;
            cudaGraphExec_t &e;
            ~GraphFree() {
                if (e) cudaGraphExecDestroy(e);
                if (g) cudaGraphDestroy(g);
                if (s) cudaStreamDestroy(s);
            }
        } gf{cap, G, GE};
        PLS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        PLS_CUDA(cudaGraphCreate(&G, 0));
        cudaGraphConditionalHandle loop;
        PLS_CUDA(cudaGraphConditionalHandleCreate(&loop, G, 0u, 0u));
        cudaKernelNodeParams kn = {};
        const int *ctrl_c = c.ctrl;
        void *kargs[] = {&loop, &ctrl_c};
        kn.func = reinterpret_cast<void *>(k_cg_loop_init);
        kn.gridDim = dim3(1);
        kn.blockDim = dim3(1);
        kn.kernelParams = kargs;
        cudaGraphNode_t n0, nw;
        PLS_CUDA(cudaGraphAddKernelNode(&n0, G, nullptr, 0, &kn));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = loop;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        PLS_CUDA(cudaGraphAddNode(&nw, G, &n0, 1, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        const int64_t l0 = c.launches;
        cudaStream_t s_run = c.s;
        c.s = cap;
        PLS_CUDA(cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_iteration(0, nullptr, nullptr, loop, 1);
        } catch (...) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(cap, &junk);
            c.s = s_run;
            throw;
        }
        PLS_CUDA(cudaStreamEndCapture(cap, &body));
        c.s = s_run;
        const int64_t per_it = c.launches - l0;
        c.launches = l0;
        PLS_CUDA(cudaGraphInstantiate(&GE, G, 0ull));
        PLS_CUDA(cudaGraphLaunch(GE, c.s));
        PLS_CUDA(cudaMemcpyAsync(hs, c.scal, S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, c.s));
        PLS_CUDA(cudaMemcpyAsync(hctrl, c.ctrl, C_COUNT * sizeof(int), cudaMemcpyDeviceToHost, c.s));
        PLS_CUDA(cudaStreamSynchronize(c.s));
        it = hctrl[C_IT];
        c.launches += 1 + per_it * it;
        c.graph_used = true;
    } else {
        int batch = kBatch;
        double d_prev = -1.0;
        int64_t it_prev = 0;
        int set = 0;
        while (true) {
            for (int b = 0; b < batch; ++b) {
                if (c.comm) {
                    c.cev = cev(set, b);
                    c.ncev = 0;
                    c.cev_cap = kCommEv;
                }
                enqueue_iteration(it + b, mv0(set)[b], mv1(set)[b], 0ull, 0);
                ncev[set][b] = c.ncev;
                c.cev = nullptr;
            }
            PLS_CUDA(cudaMemcpyAsync(hs, c.scal, S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, c.s));
            PLS_CUDA(cudaMemcpyAsync(hctrl, c.ctrl, C_COUNT * sizeof(int), cudaMemcpyDeviceToHost, c.s));
            read_times();  // the previous batch's, while this one runs
            PLS_CUDA(cudaStreamSynchronize(c.s));
            const int64_t ran = hctrl[C_IT] - it;  // iterations of this batch that did work
            pend_set = set;
            pend_n = static_cast<int>(std::min<int64_t>(std::max<int64_t>(ran, 0), batch));
            set ^= 1;
            it = hctrl[C_IT];
            if (std::getenv("PLSSVM_DEBUG"))
                std::fprintf(stderr, "[plssvm] batch: it=%d done=%d d0=%.6e d[0]=%.6e d[1]=%.6e thr=%.6e pap=%.6e\n",
                             hctrl[C_IT], hctrl[C_DONE], hs[S_DELTA0], hs[S_DELTA], hs[S_DELTA + 1], hs[S_THR],
                             hs[S_PAP]);
            if (hctrl[C_DONE] != 0 || ran < batch) break;
            // next batch: iterations to the threshold at the last batch's rate (+ 1), or the fixed count
            const double dn = delta_now(hs, it, cgcg), base = d_prev > 0.0 ? d_prev : hs[S_DELTA0];
            int64_t next = kBatch;
            if (c.comm) {
                // several ranks: fixed batches (the CG-CG host snapshot holds this rank's partial of the
                // next gamma, so a rate-based size could differ between ranks and mismatch collectives)
            } else if (o.fixed_iter > 0) {
                next = o.fixed_iter - it;
            } else if (dn > 0.0 && base > dn && hs[S_THR] > 0.0 && it > it_prev) {
                const double rate = std::log(dn / base) / static_cast<double>(it - it_prev);  // < 0
                next = static_cast<int64_t>(std::ceil(std::log(hs[S_THR] / dn) / rate)) + 1;
            }
            batch = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({next, kBatchMax, imax - it})));
            d_prev = dn;
            it_prev = it;
        }
    }
    c.cur_ctrl = nullptr;
    int64_t matvecs = it + ((o.x0 == 0) ? 0 : 1) + (cgcg ? 1 : 0);  // CG-CG: the product of the final r
    if (o.replace_every > 0 && it > 1) matvecs += (it - 1) / o.replace_every;
    const double delta0 = hs[S_DELTA0];
    const double delta = delta_now(hs, it, cgcg);
    const double eps2 = pb.eps * pb.eps;
    int status = PLSSVM_OK;
    if (hctrl[C_DONE] == 2)  // name the iteration and the offending scalars
        throw Error(PLSSVM_E_NUMERICAL, "CG breakdown at iteration " + std::to_string(it) + ": p.Q~p = " +
                                            std::to_string(cgcg ? hs[S_CG_DELTA] : hs[S_PAP]) + ", delta = " +
                                            std::to_string(delta_now(hs, it, cgcg)) +
                                            " (p.Q~p must be > 0 and finite; Q~ is not positive definite for "
                                            "these kernel parameters, or the input overflowed)");
    c.launches_cg = c.launches - launches_before_cg;
    PLS_CUDA(cudaEventRecord(e_cg, c.s));
    if (status == PLSSVM_OK && o.fixed_iter <= 0 && delta > eps2 * delta0) status = PLSSVM_W_NOT_CONVERGED;

    if (status != PLSSVM_E_NUMERICAL) {
        // ---- bias + alpha (a6) ----
        if constexpr (std::is_same<T, double>::value) {
            if (c.fsplit) {  // Eq. 15 needs the full q and Q_mm: sum the ranks' feature-slice partials
                comm_allreduce_sum_f64(c.comm, c.q, c.q, g.mpad, c.s);
                comm_allreduce_sum_f64(c.comm, c.scal + S_QMM, c.scal + S_QMM, 1, c.s);
            }
        }
        k_bias_sums<T><<<c.vb, kVecThreads, 0, c.s>>>(c.x, c.q, g.nb, g.g0, c.scal, 0, c.partials, c.counter);
        PLS_CHECK_LAUNCH();
        k_bias_sums<T><<<c.vb, kVecThreads, 0, c.s>>>(c.x, c.q, g.nb, g.g0, c.scal, 1, c.partials, c.counter);
        PLS_CHECK_LAUNCH();
        c.launches += 2;
        allreduce(c, S_SUMX, 2);
        PLS_CUDA(cudaMemcpyAsync(c.xfull + g.g0, c.x, g.nb * sizeof(T), cudaMemcpyDeviceToDevice, c.s));
        allgather(c, c.xfull);
        const bool dev = o.device_pointers != 0;
        T *alpha_d = dev ? static_cast<T *>(alpha_out) : A.alloc<T>(pb.m);
        T *b_d = dev ? static_cast<T *>(b_out) : A.alloc<T>(1);
        k_assemble<T><<<static_cast<unsigned>(ceil_div(pb.m, 256)), 256, 0, c.s>>>(c.xfull, pb.m, c.scal, alpha_d, b_d);
        PLS_CHECK_LAUNCH();
        ++c.launches;
        if (!dev) {
            PLS_CUDA(cudaMemcpyAsync(alpha_out, alpha_d, pb.m * sizeof(T), cudaMemcpyDeviceToHost, c.s));
            PLS_CUDA(cudaMemcpyAsync(b_out, b_d, sizeof(T), cudaMemcpyDeviceToHost, c.s));
        }
    }
    // true residual (options.true_residual, SURVEY §5 metrics): one more product of the final x
    double rel_true = -1.0;
    if (o.true_residual && status != PLSSVM_E_NUMERICAL) {
        const int ns = launch_qtilde_product<T>(c, c.xfull);
        finalize<T>(c, ns, nullptr, 1, nullptr, S_TRUE - S_DELTA, 0);  // mode 1 into slot S_TRUE
        allreduce(c, S_TRUE, 1);
        PLS_CUDA(cudaMemcpyAsync(hs + S_TRUE, c.scal + S_TRUE, sizeof(double), cudaMemcpyDeviceToHost, c.s));
    }
    const int64_t trace_w = want_trace ? std::min<int64_t>(trace_n, it + 1) : 0;
    if (trace_w > 0)
        PLS_CUDA(cudaMemcpyAsync(o.residual_trace, trace_d, trace_w * sizeof(double), cudaMemcpyDeviceToHost, c.s));
    PLS_CUDA(cudaEventRecord(e_end, c.s));
    read_times();  // the last batch's, while the bias / alpha work runs
    PLS_CUDA(cudaStreamSynchronize(c.s));
    for (int64_t k = 0; k < trace_w; ++k) o.residual_trace[k] = std::sqrt(std::max(o.residual_trace[k], 0.0));
    if (o.true_residual && status != PLSSVM_E_NUMERICAL) rel_true = delta0 > 0 ? std::sqrt(hs[S_TRUE] / delta0) : 0.0;
    if (st) {
        st->rel_residual_true = rel_true;
        st->stop_reason = hctrl[C_DONE] == 3 ? PLSSVM_STOP_STAGNATED
                          : o.fixed_iter > 0  ? PLSSVM_STOP_FIXED
                          : delta <= eps2 * delta0 ? PLSSVM_STOP_CONVERGED
                                                   : PLSSVM_STOP_MAX_ITER;
        st->transport_used = 0;
        st->allgather_fused = (c.lsa || c.npeer > 0) ? 1 : 0;
        st->iterations = it;
        st->matvecs = matvecs + (rel_true >= 0.0 ? 1 : 0);
        st->rel_residual = delta0 > 0 ? std::sqrt(delta / delta0) : 0.0;
        st->mode_used = c.lowrank ? PLSSVM_MODE_LOWRANK : (c.cached ? PLSSVM_MODE_CACHED : PLSSVM_MODE_IMPLICIT);
        st->num_ranks = c.nranks;
        st->cg_loop_used = c.graph_used ? PLSSVM_CG_GRAPH : PLSSVM_CG_BATCHED;
        st->fp32_engine_used = std::is_same<T, float>::value
                                   ? (c.oz ? PLSSVM_FP32_OZAKI : c.tc ? PLSSVM_FP32_TCGEN05 : PLSSVM_FP32_FFMA)
                                   : 0;
        st->t_h2d = elapsed(e0, e_h2d);
        st->t_transform = elapsed(e_h2d, e_tr);
        st->t_q = elapsed(e_tr, e_q);
        st->t_alloc = elapsed(e_q, e_alloc);
        st->t_precompute = elapsed(e_alloc, e_pre);
        st->t_cg = elapsed(e_pre, e_cg);
        st->t_bias_d2h = elapsed(e_cg, e_end);
        st->t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
        st->t_matvec = t_mv;
        st->t_comm = t_comm;
        st->t_matvec_min = it > 0 ? t_mv_min : 0.0;
        st->bytes_per_gpu = A.bytes;
        st->gpu_launches = c.launches;
        st->launches_in_cg = c.launches_cg;
        st->fp64_engine_used = std::is_same<T, double>::value ? (c.oz ? PLSSVM_FP64_OZAKI : PLSSVM_FP64_DMMA) : 0;
    }
    return status;
}

template <typename T>
int qtilde_matvec_impl(const Problem &pb, const void *pin, int32_t repeats, const plssvm_options_t &o, void *out,
                       double *t_kernel) {
    PLS_CUDA(cudaSetDevice(o.device));
    upload_reset();
    setup_mempool(o.device);
    StreamGuard sg(o.stream);
    Ctx<T> c{};
    c.s = sg.s;
    c.comm = static_cast<CommHandle *>(o.comm);
    Arena A(c.s);
    Events E;
    cudaEvent_t e0 = E.make(), e1 = E.make(), e2 = E.make(), e3 = E.make();
    setup<T>(c, A, pb, o, false, E, e0, e1, e2);
    const Geometry &g = c.g;
    c.y = A.alloc<T>(g.nb);
    c.p = A.alloc<T>(g.mpad);
    PLS_CUDA(cudaMemsetAsync(c.p, 0, g.mpad * sizeof(T), c.s));
    const bool dev = o.device_pointers != 0;
    PLS_CUDA(cudaMemcpyAsync(c.p, pin, g.m1 * sizeof(T), dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.s));
    validate_inputs<T>(A, {VCheck<T>{c.p, g.m1, V_NONFINITE_P, 0}}, static_cast<const T *>(nullptr), 0, c.s,
                       c.launches);
    select_mode<T>(c, o);  // throws E_OOM if CACHED does not fit
    configure_product<T>(c, A);
    double t_pre = 0.0;
    if (c.cached) {
        c.Qc = A.alloc<T>(c.packed ? c.nstored * kTile * kTile : g.nb * g.mpad);
        PLS_CUDA(cudaEventRecord(e0, c.s));
        launch_precompute<T>(c);
        PLS_CUDA(cudaEventRecord(e1, c.s));
        PLS_CUDA(cudaStreamSynchronize(c.s));
        t_pre = elapsed(e0, e1);
    }
    double tsum = 0.0, tmin = 1e30;
    int ns = 1;
    for (int rep = 0; rep < std::max(1, repeats); ++rep) {
        PLS_CUDA(cudaEventRecord(e2, c.s));
        ns = launch_qtilde_product<T>(c, c.p);
        PLS_CUDA(cudaEventRecord(e3, c.s));
        PLS_CUDA(cudaEventSynchronize(e3));
        const double t = elapsed(e2, e3);
        tsum += t;
        tmin = std::min(tmin, t);
    }
    finalize<T>(c, ns, c.p + g.g0, 0, nullptr, 0, 0);
    // gather the band results into the full vector (reuse p as the gather buffer)
    T *yfull = A.alloc<T>(g.mpad);
    PLS_CUDA(cudaMemcpyAsync(yfull + g.g0, c.y, g.nb * sizeof(T), cudaMemcpyDeviceToDevice, c.s));
    allgather(c, yfull);
    PLS_CUDA(cudaMemcpyAsync(out, yfull, g.m1 * sizeof(T), dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.s));
    PLS_CUDA(cudaStreamSynchronize(c.s));
    if (t_kernel) {
        t_kernel[0] = tsum / std::max(1, repeats);
        t_kernel[1] = tmin;
        t_kernel[2] = t_pre;
    }
    return PLSSVM_OK;
}

template <typename T>
int predict_impl(const Problem &pb, const void *alpha_in, double b, const void *Zin, int64_t n, const plssvm_options_t &o,
                 void *decision, int32_t *labels, double *t_kernel) {
    PLS_CUDA(cudaSetDevice(o.device));
    upload_reset();
    setup_mempool(o.device);
    StreamGuard sg(o.stream);
    cudaStream_t s = sg.s;
    Arena A(s);
    Events E;
    cudaEvent_t e0 = E.make(), e1 = E.make();
    int64_t launches = 0;
    const bool dev = o.device_pointers != 0;
    const int64_t m = pb.m, d = pb.d;
    using EN = Engine<T>;
    const int64_t mpad = round_up(m, kTile), npad = round_up(n, kTile);
    const int64_t dpad = round_up(d, EN::BK);
    // point-major: Xp[mpad][dpad], Zp[npad][dpad]; feature-major: both with ld = max(mpad, npad)
    const int64_t L = std::max(mpad, npad);
    const int64_t xrows = EN::kPointMajor ? mpad : L, zrows = EN::kPointMajor ? npad : L;
    const T *Xs = stage_input<T>(A, pb.X, m * d, dev, s);
    const T *Zs = stage_input<T>(A, Zin, n * d, dev, s);
    const T *al = stage_input<T>(A, alpha_in, m, dev, s);
    const RowStats rho = validate_inputs<T>(A, {VCheck<T>{Xs, m * d, V_NONFINITE_X, d}, VCheck<T>{Zs, n * d, V_NONFINITE_Z, d},
                                             VCheck<T>{al, m, V_NONFINITE_ALPHA, 0}},
                                         static_cast<const T *>(nullptr), 0, s, launches);
    if (pb.kernel == LINEAR && o.linear_w) {
        // f(z) = <w, z> + b with w = sum_i alpha_i x_i (Eq. 15): O((m + n) d)
        const int64_t rpb = std::max<int64_t>(1, ceil_div(m, 4 * 148));
        const int parts = static_cast<int>(ceil_div(m, rpb));
        T *wpart = A.alloc<T>(static_cast<int64_t>(parts) * d), *w = A.alloc<T>(d);
        T *f_d = (dev && decision) ? static_cast<T *>(decision) : A.alloc<T>(n);
        int32_t *l_d = (dev && labels) ? labels : A.alloc<int32_t>(n);
        PLS_CUDA(cudaEventRecord(e0, s));
        k_colsum_partial<T><<<parts, 256, 0, s>>>(Xs, d, 0, m, rpb, al, nullptr, m, wpart, nullptr, nullptr);
        k_colsum_reduce<T><<<static_cast<unsigned>(ceil_div(d, 256)), 256, 0, s>>>(wpart, parts, d, w, nullptr, nullptr);
        k_rowdot<T><<<static_cast<unsigned>(ceil_div(n * 32, 256)), 256, 0, s>>>(Zs, d, 0, n, w, 0, static_cast<T>(b),
                                                                                 nullptr, n, T(0), nullptr, f_d, l_d,
                                                                                 nullptr);
        PLS_CHECK_LAUNCH();
        PLS_CUDA(cudaEventRecord(e1, s));
        launches += 3;
        if (!dev) {
            if (decision) PLS_CUDA(cudaMemcpyAsync(decision, f_d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
            if (labels) PLS_CUDA(cudaMemcpyAsync(labels, l_d, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        }
        PLS_CUDA(cudaStreamSynchronize(s));
        if (t_kernel) {
            t_kernel[0] = elapsed(e0, e1);
            t_kernel[1] = static_cast<double>(launches);
        }
        return PLSSVM_OK;
    }
    bool oz64 = false;  // (the name: the Ozaki engine of either precision)
    if constexpr (std::is_same<T, double>::value) {
        oz64 = oz_choose(o.fp64_engine, rho, std::max(zrows, xrows), d);
    } else if (o.fp32_engine == PLSSVM_FP32_OZAKI || o.fp32_engine == PLSSVM_FP32_AUTO) {
        oz64 = oz_choose_f32(o.fp32_engine, rho, d);
    }
    // the int8 engines split (and take norms of) the caller's row-major X and Z directly; the other
    // engines use the transformed layouts
    T *Xl = nullptr, *Zl = nullptr;
    if (!oz64) {
        Xl = A.alloc<T>(dpad * xrows);
        Zl = A.alloc<T>(dpad * zrows);
        launch_transform<T>(Xs, m, d, Xl, xrows, dpad, s, launches);
        launch_transform<T>(Zs, n, d, Zl, zrows, dpad, s, launches);
    }
    T *alpha = A.alloc<T>(xrows);
    PLS_CUDA(cudaMemsetAsync(alpha, 0, xrows * sizeof(T), s));
    PLS_CUDA(cudaMemcpyAsync(alpha, al, m * sizeof(T), cudaMemcpyDeviceToDevice, s));
    T *nx = A.alloc<T>(xrows), *nz = A.alloc<T>(zrows);
    KParams<T> kp{pb.kernel, static_cast<T>(pb.gamma), pb.degree, static_cast<T>(pb.coef0)};
    if (pb.kernel == RBF) {
        if (oz64) {  // rows m .. xrows - 1 (n .. zrows - 1) get 0
            k_norms<T><<<static_cast<unsigned>(ceil_div(xrows * 32, 256)), 256, 0, s>>>(Xs, xrows, dpad, m, d, nx, d);
            k_norms<T><<<static_cast<unsigned>(ceil_div(zrows * 32, 256)), 256, 0, s>>>(Zs, zrows, dpad, n, d, nz, d);
        } else {
            k_norms<T><<<static_cast<unsigned>(ceil_div(xrows * 32, 256)), 256, 0, s>>>(Xl, xrows, dpad, xrows, d, nx);
            k_norms<T><<<static_cast<unsigned>(ceil_div(zrows * 32, 256)), 256, 0, s>>>(Zl, zrows, dpad, zrows, d, nz);
        }
        PLS_CHECK_LAUNCH();
        launches += 2;
    }
    const bool tc = std::is_same<T, float>::value && !oz64 && o.fp32_engine != PLSSVM_FP32_FFMA;
    const int tilesI = static_cast<int>(npad / kTile),
              tilesJ = static_cast<int>(mpad / (tc ? kTile : oz64 ? OzC::TN : EN::TN));
    T *Fpart = A.alloc<T>(static_cast<int64_t>(tilesJ) * npad);
    set_smem_attrs<T>();
    const size_t sm = EN::SMEM_BYTES;
    const int grid = tilesI * tilesJ;
    if constexpr (std::is_same<T, float>::value) {
        if (tc) {
            // fp32 on tcgen05 (3xTF32): hi/lo split of both operands, TMA descriptors
            const int64_t dtc = round_up(d, Tc::BK);
            float *Zh = A.alloc<float>(npad * dtc), *Zlo = A.alloc<float>(npad * dtc);
            float *Xh = A.alloc<float>(mpad * dtc), *Xlo = A.alloc<float>(mpad * dtc);
            k_split_tf32<<<static_cast<unsigned>(ceil_div(npad * dtc, 256)), 256, 0, s>>>(Zs, n, d, Zh, Zlo, npad, dtc);
            k_split_tf32<<<static_cast<unsigned>(ceil_div(mpad * dtc, 256)), 256, 0, s>>>(Xs, m, d, Xh, Xlo, mpad, dtc);
            PLS_CHECK_LAUNCH();
            launches += 2;
            const CUtensorMap zh = make_tmap_2d_f32(Zh, dtc, npad, Tc::BK, kTile);
            const CUtensorMap zl = make_tmap_2d_f32(Zlo, dtc, npad, Tc::BK, kTile);
            const CUtensorMap xh = make_tmap_2d_f32(Xh, dtc, mpad, Tc::BK, kTile);
            const CUtensorMap xl = make_tmap_2d_f32(Xlo, dtc, mpad, Tc::BK, kTile);
            tc_set_attrs();
            // 128 x 256 tiles (UMMA N = 256): test block I x two training blocks
            const CUtensorMap zwh = make_tmap_2d(Zh, 4, dtc, npad, TcW::BK, kTile, CU_TENSOR_MAP_SWIZZLE_64B);
            const CUtensorMap zwl = make_tmap_2d(Zlo, 4, dtc, npad, TcW::BK, kTile, CU_TENSOR_MAP_SWIZZLE_64B);
            const CUtensorMap xwh = make_tmap_2d(Xh, 4, dtc, mpad, TcW::BK, 2 * kTile, CU_TENSOR_MAP_SWIZZLE_64B);
            const CUtensorMap xwl = make_tmap_2d(Xlo, 4, dtc, mpad, TcW::BK, 2 * kTile, CU_TENSOR_MAP_SWIZZLE_64B);
            (void)zh; (void)zl; (void)xh; (void)xl;
            PLS_CUDA(cudaMemsetAsync(Fpart, 0, static_cast<size_t>(tilesJ) * npad * sizeof(T), s));
            PLS_CUDA(cudaEventRecord(e0, s));
            tcw_dispatch<TC_PREDICT>(pb.kernel, tilesI * static_cast<int>(ceil_div(tilesJ, 2)), s, zwh, zwl, xwh, xwl,
                                     dtc, static_cast<const int2 *>(nullptr), tilesI, tilesJ,
                                     static_cast<const float *>(nullptr), nz, static_cast<const float *>(nullptr), nx,
                                     alpha, kp, 0.f, static_cast<const double *>(nullptr), int64_t(0), Fpart, npad,
                                     static_cast<const int *>(nullptr));
        }
    }
    const bool oz = oz64;
    if (oz) {  // int8 tensor cores: test points = row operand, training points = columns
        OzOperand oz_z, oz_x;
        constexpr int S = oz_digits<T>();
        oz_z = oz_prepare<S, T>(A, Zs, npad, n, d, d, true, false, s, launches);
        oz_x = oz_prepare<S, T>(A, Xs, mpad, m, d, d, false, true, s, launches);
        oz_set_attrs<T>();
        PLS_CUDA(cudaEventRecord(e0, s));
        oz_dispatch<OZ_PREDICT, T>(pb.kernel, ((tilesI + 1) / 2) * tilesJ, s, oz_z, oz_x,
                                   static_cast<const int4 *>(nullptr), static_cast<const int *>(nullptr), tilesI,
                                   static_cast<const T *>(nullptr), static_cast<const T *>(nz),
                                   static_cast<const T *>(nx), static_cast<const T *>(alpha), kp, T(0),
                                   static_cast<const double *>(nullptr), int64_t(0), 0, 0, Fpart, npad,
                                   static_cast<T *>(nullptr), 0, static_cast<const int *>(nullptr));
    }
    const Ops<T> pops = (tc || oz64) ? Ops<T>{} : make_ops(Zl, zrows, Xl, xrows, EN::kPointMajor ? dpad : L);
    if (!tc && !oz) PLS_CUDA(cudaEventRecord(e0, s));
    if (!tc && !oz) switch (pb.kernel) {
        case LINEAR:
            k_predict_tiles<LINEAR, T><<<grid, Engine<T>::THREADS, sm, s>>>(pops, npad, dpad, nz, nx, alpha, kp, tilesI,
                                                                  Fpart);
            break;
        case POLYNOMIAL:
            k_predict_tiles<POLYNOMIAL, T><<<grid, Engine<T>::THREADS, sm, s>>>(pops, npad, dpad, nz, nx, alpha, kp,
                                                                                tilesI, Fpart);
            break;
        default:
            k_predict_tiles<RBF, T><<<grid, Engine<T>::THREADS, sm, s>>>(pops, npad, dpad, nz, nx, alpha, kp, tilesI,
                                                               Fpart);
    }
    PLS_CHECK_LAUNCH();
    PLS_CUDA(cudaEventRecord(e1, s));
    ++launches;
    T *f_d = (dev && decision) ? static_cast<T *>(decision) : A.alloc<T>(n);
    int32_t *l_d = (dev && labels) ? labels : A.alloc<int32_t>(n);
    k_predict_finalize<T><<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, s>>>(Fpart, tilesJ, npad, n, static_cast<T>(b),
                                                                                 f_d, l_d);
    PLS_CHECK_LAUNCH();
    ++launches;
    if (!dev) {
        if (decision) PLS_CUDA(cudaMemcpyAsync(decision, f_d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
        if (labels) PLS_CUDA(cudaMemcpyAsync(labels, l_d, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
    PLS_CUDA(cudaStreamSynchronize(s));
    if (t_kernel) {
        t_kernel[0] = elapsed(e0, e1);
        t_kernel[1] = static_cast<double>(launches);
    }
    return PLSSVM_OK;
}

}  // namespace

#ifdef PLSSVM_OZ_EXPERIMENTS
int exp_oz_profile(unsigned long long *out, int reset) {
    if (out) PLS_CUDA(cudaMemcpyFromSymbol(out, g_oz_prof, sizeof(g_oz_prof)));
    if (reset) {
        static unsigned long long zero[160][8] = {};
        PLS_CUDA(cudaMemcpyToSymbol(g_oz_prof, zero, sizeof(zero)));
    }
    return PLSSVM_OK;
}
#endif

int train(const Problem &pb, const plssvm_options_t &o, void *alpha, void *b, plssvm_stats_t *st) {
    Nvtx r("plssvm_train");
    return pb.dtype == PLSSVM_F32 ? train_impl<float>(pb, o, alpha, b, st) : train_impl<double>(pb, o, alpha, b, st);
}
int predict(const Problem &pb, const void *alpha, double b, const void *Z, int64_t n, const plssvm_options_t &o,
            void *decision, int32_t *labels, double *t_kernel) {
    Nvtx r("plssvm_predict");
    return pb.dtype == PLSSVM_F32 ? predict_impl<float>(pb, alpha, b, Z, n, o, decision, labels, t_kernel)
                                  : predict_impl<double>(pb, alpha, b, Z, n, o, decision, labels, t_kernel);
}
int qtilde_matvec(const Problem &pb, const void *p, int32_t repeats, const plssvm_options_t &o, void *out,
                  double *t_kernel) {
    Nvtx r("plssvm_qtilde_matvec");
    return pb.dtype == PLSSVM_F32 ? qtilde_matvec_impl<float>(pb, p, repeats, o, out, t_kernel)
                                  : qtilde_matvec_impl<double>(pb, p, repeats, o, out, t_kernel);
}

}  // namespace plssvm
