// kernels.cuh -- every device kernel of the hot path (sm_100a).
//
//   k_transform        row-major X -> padded feature-major X^T            (paper "transform")
//   k_q_norms          q_i = k(x_i, x_m), n_i = ||x_i||^2, Q_mm          (Eq. 12)
//   k_matvec_implicit  Ypart[slot][row] = partial Q~p per tile            (Eq. 16)
//   k_precompute       Q~ band tiles -> HBM (cached mode, north_star N1)
//   k_gemv_tiled       y_band = Q~_band p streamed from HBM (tiled layout)
//   k_finalize         y = sum_slots Ypart ; p.y  (deterministic)
//   k_update_xr        x += a p ; r -= a y ; r.r  (fused axpy + norm)
//   k_update_p         p = r + b p ; loop condition (and the CUDA-graph WHILE condition)
//   k_cg_fused         the three above in one cooperative launch (single GPU)
//   k_init / k_bias    CG start, Eq. 15 bias + alpha assembly
//   k_predict          f(z) = sum_i alpha_i k(x_i, z) + b                (Eq. 10)
#pragma once
#include <cooperative_groups.h>
#include <nccl_device.h>

#include "tile_engine.cuh"

namespace plssvm {

// Slots of the device scalar block (double precision storage for every dtype's scalars).
enum Scal : int {
    S_QMM = 0,      // Q_mm = k(x_m,x_m) + 1/C
    S_YM = 1,       // y_m
    S_PAP = 2,      // p . Q~p   (this iteration)
    S_DELTA0 = 3,   // delta_0 = r0.r0
    S_DELTA = 4,    // delta_k at S_DELTA + (k & 1)   (double-buffered by iteration parity)
    S_ALPHA = 6,    // CG alpha of the last update
    S_SUMX = 7,     // sum of x (bias)
    S_QX = 8,       // <q, x>  (bias)
    S_B = 9,        // bias b
    S_THR = 10,     // eps^2 delta_0 (the CG stopping threshold on delta)
    S_SP = 11,      // sum of p (linear low-rank product)
    S_CG_GAMMA = 12,  // Chronopoulos-Gear: gamma_i = r_i.r_i      } contiguous: one all-reduce
    S_CG_DELTA = 13,  //                    delta_i = (Q~ r_i).r_i }   of the pair per iteration
    S_CG_GPREV = 14,  //                    gamma_{i-1}
    S_CG_APREV = 15,  //                    alpha_{i-1}
    S_L = 16,       // slot s + S_L holds this rank's local partial of slot s; the multi-GPU
                    // all-reduce is out of place (local -> global), hence idempotent: iterations
                    // enqueued after convergence cannot corrupt the global scalars
    S_BEST = 32,    // stagnation guard: delta at the last 4x drop (replicated, never all-reduced)
    S_TRUE = 33,    // |rhs - Q~x|^2 after CG (options.true_residual; partial at S_TRUE + S_L)
    S_XLT = 34,     // low-rank product: <x_{m-1}, t> of the current product (k_lastdot; replicated)
    S_COUNT = 56
};

// Device-side CG control block (int32[4]): the loop runs without a host round trip per
// iteration; every loop kernel returns immediately once `done` is set, so the host can enqueue
// iterations in batches and read the state once per batch.
// Device CG control block.  C_DONE: 0 running, 1 finished (converged / imax / fixed count), 2 breakdown
// (S:259), 3 stagnated (R-20: residual replacement on, no 4x drop of delta within the window).
// C_REPL = replace_every (0: guard off), C_IBEST = iteration of the last 4x drop (S_BEST holds its delta).
enum Ctl : int { C_IT = 0, C_DONE = 1, C_IMAX = 2, C_FIXED = 3, C_REPL = 4, C_IBEST = 5, C_COUNT = 6 };
__device__ __forceinline__ bool cg_done(const int *ctrl) { return ctrl != nullptr && *(volatile const int *)(ctrl + C_DONE) != 0; }

// ---------------------------------------------------------------------------------------
// Deterministic grid reduction: every block writes its partial; the last block to finish
// sums the partials in block order and calls fin(total).
template <typename T, typename F>
__device__ __forceinline__ void grid_reduce(T v, T *partials, unsigned *counter, F fin) {
    __shared__ T red[kVecThreads / 32];
    __shared__ bool last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        T s = T(0);
        for (int w = 0; w < kVecThreads / 32; ++w) s += red[w];
        partials[blockIdx.x] = s;
        __threadfence();
        unsigned done = atomicAdd(counter, 1u);
        last = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {
        __threadfence();
        T s = T(0);
        // lane-strided partial sums, then a fixed shuffle tree: deterministic order
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += ((volatile T *)partials)[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) {
            fin(s);
            *counter = 0u;
        }
    }
}

// ---------------------------------------------------------------------------------------
// Input validation on the device (plssvm.h "Validation"): non-finite values of an array set its
// bit; labels must be +1 / -1 with both present.  One flag word, OR-reduced per warp.
enum VFlag : unsigned { V_BADLABEL = 1u, V_POS = 2u, V_NEG = 4u, V_NONFINITE_X = 8u, V_NONFINITE_Z = 16u,
                        V_NONFINITE_ALPHA = 32u, V_NONFINITE_P = 64u };
template <typename T>
__global__ void k_validate(const T *__restrict__ a, int64_t n, unsigned bit, const T *__restrict__ y, int64_t m,
                           unsigned *__restrict__ flags) {
    unsigned f = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        if (!isfinite(a[i])) f |= bit;
    if (y) {
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
            const T v = y[i];
            f |= (v == T(1)) ? V_POS : (v == T(-1)) ? V_NEG : V_BADLABEL;
        }
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// ---------------------------------------------------------------------------------------
// Layout transform (paper "transform"): X[m][d] point-major (host order) ->
//   feature-major X^T[dpad][ld] (fp32 FFMA engine, the paper's column-major layout), or
//   point-major   Xp[ld][dpad]  (fp64 DMMA engine, features contiguous),
// zero padding everywhere outside m x d (padded features are kernel-neutral, padded points are
// masked).  32x32 smem tile, the grid covers the padded extent (no separate memset).
template <typename T>
__global__ void k_transform(const T *__restrict__ X, int64_t m, int64_t d, T *__restrict__ Xt, int64_t ld,
                            int64_t dpad, int point_major) {
    __shared__ T t[32][33];
    const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 32, f0 = static_cast<int64_t>(blockIdx.y) * 32;
    if (point_major) {
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int64_t p = p0 + r, f = f0 + threadIdx.x;
            if (p < ld && f < dpad) Xt[p * dpad + f] = (p < m && f < d) ? X[p * d + f] : T(0);
        }
        return;
    }
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t p = p0 + r, f = f0 + threadIdx.x;
        t[r][threadIdx.x] = (p < m && f < d) ? X[p * d + f] : T(0);
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t f = f0 + r, p = p0 + threadIdx.x;
        if (f < dpad && p < ld) Xt[f * ld + p] = t[threadIdx.x][r];
    }
}

// Element (point i, feature k) of the engine's layout.
template <typename T>
__device__ __forceinline__ T elem(const T *X, int64_t i, int64_t k, int64_t mpad, int64_t dpad) {
    if constexpr (Engine<T>::kPointMajor) return X[i * dpad + k];
    else return X[k * mpad + i];
}

// q cache and norms: q_i = k(x_i, x_m) for i < m-1 (0 beyond), n_i = ||x_i||^2,
// S_QMM = k(x_m, x_m) + 1/C, S_YM = y_m.  RBF q uses the direct squared distance.
// One warp per point (lanes stride the features; fixed shuffle tree -> deterministic).
template <typename T>
__global__ void k_q_norms(const T *__restrict__ X, int64_t mpad, int64_t dpad, int64_t m, int64_t d, KParams<T> kp,
                          T invC, const T *__restrict__ y, T *__restrict__ q, T *__restrict__ nrm, double *scal,
                          int64_t ld_raw) {
    // ld_raw > 0: X is the caller's row-major m x d array (row stride ld_raw; rows >= m read as 0),
    // else the engine's padded layout
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= mpad) return;
    const int64_t xm = m - 1;
    const bool real = i < m;
    T s = T(0), n = T(0), dist = T(0);
    for (int64_t k = lane; k < d; k += 32) {
        const T a = ld_raw > 0 ? (real ? X[i * ld_raw + k] : T(0)) : elem(X, i, k, mpad, dpad);
        const T b = ld_raw > 0 ? X[xm * ld_raw + k] : elem(X, xm, k, mpad, dpad);
        s = fma(a, b, s);
        n = fma(a, a, n);
        const T t = a - b;
        dist = fma(t, t, dist);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        n += __shfl_xor_sync(0xffffffffu, n, o);
        dist += __shfl_xor_sync(0xffffffffu, dist, o);
    }
    if (lane != 0) return;
    T kv;
    if (kp.kernel == LINEAR) {
        kv = s;
    } else if (kp.kernel == POLYNOMIAL) {
        const T base = kp.gamma * s + kp.coef0;
        kv = T(1);
        for (int t = 0; t < kp.degree; ++t) kv *= base;
    } else {
        if constexpr (sizeof(T) == 4) kv = expf(-kp.gamma * dist);
        else kv = exp(-kp.gamma * dist);
    }
    nrm[i] = n;
    q[i] = (i < xm) ? kv : T(0);
    if (i == xm) {
        scal[S_QMM] = static_cast<double>(kv + invC);
        scal[S_YM] = static_cast<double>(y[xm]);
    }
}

// ---------------------------------------------------------------------------------------
// Shared epilogue: Q~ entry from the contracted value (Eq. 16 with cached q):
//   Q~_ij = k(x_i,x_j) + delta_ij/C - q_j - q_i + Q_mm  ;  0 outside the (m-1)-system.
template <int KT, typename T>
__device__ __forceinline__ T qtilde_value(T s, int64_t gi, int64_t gj, T ni, T nj, T qi, T qj, T Qmm, T invC,
                                          int64_t m1, const KParams<T> &kp) {
    const bool diag = (gi == gj);
    T v = kernel_value<KT, T>(s, ni, nj, diag, kp);
    v = v + (diag ? invC : T(0)) - qj - qi + Qmm;
    return (gi < m1 && gj < m1) ? v : T(0);
}

// Implicit Q~p over a list of 128x128 tiles (I, J).  Tiles with I < J inside this rank's row
// band [band0, band1) are used twice (mirroring): their row sums go to rows of I
// and their column sums (Q~_IJ^T p_I) to rows of J.  Every (slot, row-block) pair of the
// partial buffer Ypart[T][band_rows] is written exactly once per call, so the finalize sum
// is deterministic.  ld = the engine layout's leading dimension (dpad point-major, mpad
// feature-major).
template <int KT, typename T>
__global__ void __launch_bounds__(Engine<T>::THREADS, Engine<T>::MIN_BLOCKS)
    k_matvec_implicit(const __grid_constant__ Ops<T> ops, int64_t dpad, const int2 *__restrict__ tiles,
                      const T *__restrict__ q, const T *__restrict__ nrm, const T *__restrict__ p, KParams<T> kp,
                      T invC, const double *__restrict__ scal, int64_t m1, int band0, int band1,
                      T *__restrict__ Ypart, int64_t band_rows, const int *ctrl) {
    using E = Engine<T>;
    if (cg_done(ctrl)) return;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    T *smem = align_smem<T>(smem_raw);
    const int2 tile = tiles[blockIdx.x];
    const int I = tile.x, Jc = tile.y, J = Jc / E::NSUB;  // Jc: column sub-block of width TN
    const int64_t row0 = static_cast<int64_t>(I) * kTile, col0 = static_cast<int64_t>(Jc) * E::TN;
    T acc[E::R][E::CC];
    E::contract(ops, static_cast<int>(row0), static_cast<int>(col0), dpad, smem, acc);

    const T Qmm = static_cast<T>(scal[S_QMM]);
    T qi[E::R], ni[E::R], pi[E::R], qj[E::CC], nj[E::CC], pj[E::CC];
#pragma unroll
    for (int e = 0; e < E::R; ++e) {
        const int64_t gi = row0 + E::row_of(e);
        qi[e] = q[gi]; pi[e] = p[gi]; ni[e] = (KT == RBF) ? nrm[gi] : T(0);
    }
#pragma unroll
    for (int e = 0; e < E::CC; ++e) {
        const int64_t gj = col0 + E::col_of(e);
        qj[e] = q[gj]; pj[e] = p[gj]; nj[e] = (KT == RBF) ? nrm[gj] : T(0);
    }
    T rs[E::R], cs[E::CC];
#pragma unroll
    for (int e = 0; e < E::R; ++e) rs[e] = T(0);
#pragma unroll
    for (int e = 0; e < E::CC; ++e) cs[e] = T(0);
#pragma unroll
    for (int i = 0; i < E::R; ++i) {
        const int64_t gi = row0 + E::row_of(i);
#pragma unroll
        for (int j = 0; j < E::CC; ++j) {
            const int64_t gj = col0 + E::col_of(j);
            const T v = qtilde_value<KT, T>(acc[i][j], gi, gj, ni[i], nj[j], qi[i], qj[j], Qmm, invC, m1, kp);
            rs[i] = fma(v, pj[j], rs[i]);
            cs[j] = fma(v, pi[i], cs[j]);
        }
    }
    T *redr = smem;              // rows: up to 2 x 128
    T *redc = smem + 2 * kTile;  // cols: 4 x TN
    E::reduce_rows(rs, redr);
    E::reduce_cols(cs, redc);
    __syncthreads();
    // slots: row sums of tile (I, Jc) -> slot Jc (rows of I); column sums of a mirrored tile
    // -> slot I*NSUB (rows of column sub-block Jc).  See k_finalize for the slot validity rule.
    const bool mirrored = (I != J) && (J >= band0) && (J < band1);
    const int64_t lrow0 = row0 - static_cast<int64_t>(band0) * kTile;
    for (int t = threadIdx.x; t < kTile; t += E::THREADS)
        Ypart[static_cast<int64_t>(Jc) * band_rows + lrow0 + t] = E::row_total(redr, t);
    if (mirrored) {
        const int64_t lcol0 = col0 - static_cast<int64_t>(band0) * kTile;
        for (int t = threadIdx.x; t < E::TN; t += E::THREADS)
            Ypart[static_cast<int64_t>(I) * E::NSUB * band_rows + lcol0 + t] = E::col_total(redc, t);
    }
}

// Cached mode, one-time precompute: full rows [band0*128, band1*128) of Q~ (both triangles)
// into the band's tiled array Qc from the same tiles (upper tiles mirrored as transposed stores).
template <int KT, typename T>
__global__ void __launch_bounds__(Engine<T>::THREADS, Engine<T>::MIN_BLOCKS)
    k_precompute(const __grid_constant__ Ops<T> ops, int64_t mpad, int64_t dpad, const int2 *__restrict__ tiles,
                 const T *__restrict__ q, const T *__restrict__ nrm, KParams<T> kp, T invC,
                 const double *__restrict__ scal, int64_t m1, int band0, int band1, T *__restrict__ Qc, int packed) {
    using E = Engine<T>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    T *smem = align_smem<T>(smem_raw);
    const int2 tile = tiles[blockIdx.x];
    const int I = tile.x, Jc = tile.y, J = Jc / E::NSUB;
    const int64_t row0 = static_cast<int64_t>(I) * kTile, col0 = static_cast<int64_t>(Jc) * E::TN;
    T acc[E::R][E::CC];
    E::contract(ops, static_cast<int>(row0), static_cast<int>(col0), dpad, smem, acc);
    const T Qmm = static_cast<T>(scal[S_QMM]);
    const bool mirrored = (I != J) && (J >= band0) && (J < band1);
    // Stage the finished 128 x TN tile in shared memory (the ring is free), then write it with
    // coalesced row stores -- and, for a mirrored tile, the transpose with coalesced stores too.
    constexpr int SLD = E::TN + 1;  // padded row: conflict-light column reads
    T *S = smem;
#pragma unroll
    for (int i = 0; i < E::R; ++i) {
        const int lr = E::row_of(i);
        const int64_t gi = row0 + lr;
        const T qi = q[gi], ni = (KT == RBF) ? nrm[gi] : T(0);
#pragma unroll
        for (int j = 0; j < E::CC; ++j) {
            const int lc = E::col_of(j);
            const int64_t gj = col0 + lc;
            const T qj = q[gj], nj = (KT == RBF) ? nrm[gj] : T(0);
            S[lr * SLD + lc] = qtilde_value<KT, T>(acc[i][j], gi, gj, ni, nj, qi, qj, Qmm, invC, m1, kp);
        }
    }
    __syncthreads();
    // Tiled layout (see k_gemv_tiled): tile (Ib, J) of this band at ((Ib - band0) * T + J) * 128^2,
    // row-major 128 x 128 inside.  Every store below is a contiguous run (TLB- and DRAM-friendly).
    const int T_tiles = static_cast<int>(mpad / kTile);
    const int h = Jc % E::NSUB;
    // packed: the stored tile is ordinal blockIdx.x / NSUB of the tile list, no mirror copy
    T *dst = packed ? Qc + static_cast<int64_t>(blockIdx.x / E::NSUB) * (kTile * kTile) + h * E::TN
                    : Qc + (static_cast<int64_t>(I - band0) * T_tiles + J) * (kTile * kTile) + h * E::TN;
    for (int idx = threadIdx.x; idx < kTile * E::TN; idx += E::THREADS) {
        const int r = idx / E::TN, c = idx % E::TN;
        dst[r * kTile + c] = S[r * SLD + c];
    }
    if (mirrored && !packed) {
        T *mdst = Qc + (static_cast<int64_t>(J - band0) * T_tiles + I) * (kTile * kTile) + h * E::TN * kTile;
        for (int idx = threadIdx.x; idx < kTile * E::TN; idx += E::THREADS) {
            const int c = idx / kTile, r = idx % kTile;
            mdst[c * kTile + r] = S[r * SLD + c];
        }
    }
}

// Cached mode: y = Q~_band p from the tiled array (tile (Ib, J) = 128 x 128 row-major block at
// (Ib * T + J) * 128^2).  CTA = one row block x one split of the tile columns (split-K keeps
// >= ~4 CTAs per SM when there are few row blocks); warp w owns rows 16w..16w+15 and keeps
// 16 per-lane partial sums across all its tiles; 16-byte streaming loads
// (ld.global.nc.L1::no_allocate), every load independent.  Partial sums go to Ypart[split].
template <typename T>
__global__ void __launch_bounds__(256) k_gemv_tiled(const T *__restrict__ Qc, const T *__restrict__ p, int T_tiles,
                                                    int nsplit, int64_t nb, T *__restrict__ Ypart, const int *ctrl) {
    if (cg_done(ctrl)) return;
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    constexpr int VEC = 16 / sizeof(T);
    constexpr int LPR = kTile / (32 * VEC);  // 16-byte loads per lane per row (2 fp64, 1 fp32)
    const int Ib = blockIdx.x / nsplit, sp = blockIdx.x % nsplit;
    const int j0 = static_cast<int>(static_cast<int64_t>(sp) * T_tiles / nsplit);
    const int j1 = static_cast<int>(static_cast<int64_t>(sp + 1) * T_tiles / nsplit);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T acc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r] = T(0);
    for (int J = j0; J < j1; ++J) {
        const T *tile = Qc + (static_cast<int64_t>(Ib) * T_tiles + J) * (kTile * kTile) + (w * 16) * kTile;
        V pv[LPR];
#pragma unroll
        for (int u = 0; u < LPR; ++u) pv[u] = reinterpret_cast<const V *>(p + static_cast<int64_t>(J) * kTile)[u * 32 + lane];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int u = 0; u < LPR; ++u) {
                const V *src = reinterpret_cast<const V *>(tile + r * kTile) + u * 32 + lane;
                V a;
                if constexpr (sizeof(T) == 8) {
                    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(a.x), "=d"(a.y) : "l"(src));
                } else {
                    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(src));
                }
                const T *ae = reinterpret_cast<const T *>(&a);
                const T *pe = reinterpret_cast<const T *>(&pv[u]);
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[r] = fma(ae[v], pe[v], acc[r]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    }
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < 16; ++r) Ypart[static_cast<int64_t>(sp) * nb + static_cast<int64_t>(Ib) * kTile + w * 16 + r] = acc[r];
    }
}

// Cached mode, symmetric-packed layout: only the stored tile pairs (the
// upper triangle for one GPU, this rank's circulant pairs for several) are kept, each 128 x 128
// row-major block at ordinal t (the tile list order, NSUB entries per pair).  One CTA per stored
// tile streams it once and uses it twice: row sums Q~_IJ p_J -> rows of I (slot J) and, for
// I != J, column sums Q~_IJ^T p_I -> rows of J (slot I) -- half the HBM bytes of full rows.
// Warp w owns rows 16w..16w+15; lane l holds 4 columns of each row, taken as LPR 16-byte
// vectors that are each contiguous across the warp: column u*32*VEC + l*VEC + v (fp64: 2l, 2l+1,
// 64+2l, 65+2l; fp32: 4l..4l+3) -- every load instruction of a warp covers 512 contiguous bytes,
// so no 32-byte sector is fetched twice through the no-allocate L1 path.
template <typename T>
__global__ void __launch_bounds__(256, 4) k_gemv_sym(const T *__restrict__ Qc, const int2 *__restrict__ tiles, int nsub,
                                                     int64_t nstored, int per_cta, const T *__restrict__ p, int band0,
                                                     int64_t brows, T *__restrict__ Ypart, const int *ctrl) {
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    constexpr int VEC = 16 / sizeof(T);
    constexpr int LPR = 4 / VEC;  // 16-byte loads per lane per row (2 fp64, 1 fp32)
    __shared__ T redc[2][8][kTile + 4];
    if (cg_done(ctrl)) return;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * per_cta;
    int nsync = 0;  // column partials double-buffered by barrier count: one barrier per mirrored tile
    for (int64_t tt = t0; tt < t0 + per_cta && tt < nstored; ++tt) {
        const int buf = nsync & 1;
        const int2 tile = tiles[tt * nsub];
        const int I = tile.x, J = tile.y / nsub;
        const T *blk = Qc + tt * (kTile * kTile) + (w * 16) * kTile + lane * VEC;
        T pj[4], rs[16], cs[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            pj[v] = p[static_cast<int64_t>(J) * kTile + (v / VEC) * (32 * VEC) + lane * VEC + (v % VEC)];
            cs[v] = T(0);
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const T pi = p[static_cast<int64_t>(I) * kTile + w * 16 + r];
            T a[4];
#pragma unroll
            for (int u = 0; u < LPR; ++u) {
                const V *src = reinterpret_cast<const V *>(blk + r * kTile + u * (32 * VEC));
                V x;
                if constexpr (sizeof(T) == 8) {
                    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(x.x), "=d"(x.y) : "l"(src));
                } else {
                    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "l"(src));
                }
                const T *xe = reinterpret_cast<const T *>(&x);
#pragma unroll
                for (int v = 0; v < VEC; ++v) a[u * VEC + v] = xe[v];
            }
            T s = T(0);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                s = fma(a[v], pj[v], s);
                cs[v] = fma(a[v], pi, cs[v]);
            }
            rs[r] = s;
        }
        // row sums: 16 values x 32 lanes -> lane l holds row 16w + (l >> 1) (16 shuffles); each
        // tile row belongs to exactly one warp, so it is written straight to its slot.
        {
            T w8[8], w4[4], w2[2];
            const bool h1 = (lane >> 4) & 1, h2 = (lane >> 3) & 1, h3 = (lane >> 2) & 1, h4 = (lane >> 1) & 1;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                w8[i] = (h1 ? rs[i + 8] : rs[i]) + __shfl_xor_sync(0xffffffffu, h1 ? rs[i] : rs[i + 8], 16);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                w4[i] = (h2 ? w8[i + 4] : w8[i]) + __shfl_xor_sync(0xffffffffu, h2 ? w8[i] : w8[i + 4], 8);
#pragma unroll
            for (int i = 0; i < 2; ++i)
                w2[i] = (h3 ? w4[i + 2] : w4[i]) + __shfl_xor_sync(0xffffffffu, h3 ? w4[i] : w4[i + 2], 4);
            T w1 = (h4 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? w2[0] : w2[1], 2);
            w1 += __shfl_xor_sync(0xffffffffu, w1, 1);
            if ((lane & 1) == 0)
                Ypart[static_cast<int64_t>(J) * brows + static_cast<int64_t>(I - band0) * kTile + w * 16 + (lane >> 1)] = w1;
        }
        if (I != J) {  // tile-uniform branch
#pragma unroll
            for (int v = 0; v < 4; ++v) redc[buf][w][(v / VEC) * (32 * VEC) + lane * VEC + (v % VEC)] = cs[v];
            __syncthreads();
            ++nsync;
            if (threadIdx.x < kTile) {
                const int t = threadIdx.x;
                T s = T(0);
#pragma unroll
                for (int ww = 0; ww < 8; ++ww) s += redc[buf][ww][t];
                Ypart[static_cast<int64_t>(I) * brows + static_cast<int64_t>(J - band0) * kTile + t] = s;
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// Linear-kernel shortcuts (they change the cost model and are reported
// separately from the implicit FLOP/s).  X here is the caller's row-major m x d array.
//
// Weighted column sums: part[b][k] = sum_{i in rows of block b} c_i X[i][k], in increasing i, with
//   c_i = coef[i]     (coef != nullptr: all rows; predict: w = X^T alpha, Eq. 15)
//   c_i = p[i]        (coef == nullptr, the low-rank X^T B p: rows i < m-1 only -- the -sum(p) x_{m-1}
//                      term of B p = (p, -sum p) is added once in k_colsum_reduce)
// restricted to rows [r0, r1).  psum (low-rank): psum[b] = sum of block b's slice of p[0, m-1) (the
// slices cover all of p whatever the row band, so every rank forms the same sum(p)).  Column pairs
// (vec2 loads) and 8 rows per step with the loads issued ahead of the FMAs: the column sums are a
// streaming read of X and need many loads in flight (one dependent FMA chain per column kept the
// round-1 kernel at ~64 % of HBM).  Deterministic: fixed row order, then k_colsum_reduce.
template <typename T>
__global__ void __launch_bounds__(256) k_colsum_partial(const T *__restrict__ X, int64_t d, int64_t r0, int64_t r1,
                                                        int64_t rows_per_block, const T *__restrict__ coef,
                                                        const T *__restrict__ p, int64_t m, T *__restrict__ part,
                                                        double *__restrict__ psum, const int *ctrl) {
    using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
    if (cg_done(ctrl)) return;
    const int64_t b0 = r0 + static_cast<int64_t>(blockIdx.x) * rows_per_block;
    int64_t e1 = b0 + rows_per_block < r1 ? b0 + rows_per_block : r1;
    if (!coef && e1 > m - 1) e1 = m - 1;
    auto cf = [&](int64_t i) -> T { return coef ? coef[i] : p[i]; };
    if (psum) {  // this block's slice of sum_{i < m-1} p_i (fixed order)
        __shared__ double red[8];
        const int64_t chunk = (m - 1 + gridDim.x - 1) / gridDim.x;
        const int64_t s0 = static_cast<int64_t>(blockIdx.x) * chunk, s1 = s0 + chunk < m - 1 ? s0 + chunk : m - 1;
        double v = 0.0;
        for (int64_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) v += static_cast<double>(p[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += red[w];
            psum[blockIdx.x] = t;
        }
    }
    constexpr int U = 8;
    if ((d & 1) == 0) {
        const V2 *X2 = reinterpret_cast<const V2 *>(X);
        const int64_t d2 = d >> 1;
        for (int64_t k2 = threadIdx.x; k2 < d2; k2 += blockDim.x) {
            T s0 = T(0), s1 = T(0);
            int64_t i = b0;
            for (; i + U <= e1; i += U) {
                V2 v[U];
                T c[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    v[u] = X2[(i + u) * d2 + k2];
                    c[u] = cf(i + u);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    s0 = fma(c[u], v[u].x, s0);
                    s1 = fma(c[u], v[u].y, s1);
                }
            }
            for (; i < e1; ++i) {
                const V2 v = X2[i * d2 + k2];
                const T c = cf(i);
                s0 = fma(c, v.x, s0);
                s1 = fma(c, v.y, s1);
            }
            part[static_cast<int64_t>(blockIdx.x) * d + 2 * k2] = s0;
            part[static_cast<int64_t>(blockIdx.x) * d + 2 * k2 + 1] = s1;
        }
        return;
    }
    for (int64_t k = threadIdx.x; k < d; k += blockDim.x) {  // odd d: rows not 2-element aligned
        T s = T(0);
        int64_t i = b0;
        for (; i + U <= e1; i += U) {
            T v[U], c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                v[u] = X[(i + u) * d + k];
                c[u] = cf(i + u);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) s = fma(c[u], v[u], s);
        }
        for (; i < e1; ++i) s = fma(cf(i), X[i * d + k], s);
        part[static_cast<int64_t>(blockIdx.x) * d + k] = s;
    }
}

// out[k] = sum_b part[b][k] (fixed order).  Low-rank (psum != nullptr): sum(p) = sum_b psum[b] (every block,
// warp 0, lane-strided + shuffle tree: fixed order) -> scal[S_SP], and the rank whose band holds row m-1
// (xlast = X + (m-1) d, else nullptr) adds its -sum(p) x_{m-1} term.
template <typename T>
__global__ void __launch_bounds__(256) k_colsum_reduce(const T *__restrict__ part, int nparts, int64_t d,
                                                       T *__restrict__ out, double *out_local, const int *ctrl,
                                                       const double *__restrict__ psum = nullptr,
                                                       const T *__restrict__ xlast = nullptr, double *scal = nullptr) {
    if (cg_done(ctrl)) return;
    __shared__ double sp_sh;
    if (psum) {
        if (threadIdx.x < 32) {
            double v = 0.0;
            for (int b = threadIdx.x; b < nparts; b += 32) v += psum[b];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (threadIdx.x == 0) {
                sp_sh = v;
                if (blockIdx.x == 0 && scal) scal[S_SP] = v;
            }
        }
        __syncthreads();
    }
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= d) return;
    T s = T(0);
    for (int b = 0; b < nparts; ++b) s += part[static_cast<int64_t>(b) * d + k];
    if (psum && xlast) s = fma(static_cast<T>(-sp_sh), xlast[k], s);
    out[k] = s;
    if (out_local) out_local[k] = static_cast<double>(s);
}

template <typename T>
__global__ void k_cast(const double *__restrict__ a, int64_t n, T *__restrict__ b) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) b[i] = static_cast<T>(a[i]);
}

// <x_{m-1}, t> of the low-rank product, once (one block, fixed-order tree: every rank and every
// row-dot warp uses the same value) -> scal[S_XLT].  (Round 2: each warp of k_rowdot recomputed it,
// re-reading the 8 d bytes of x_{m-1} once per row: as many load instructions as the streamed rows.)
template <typename T>
__global__ void __launch_bounds__(256) k_lastdot(const T *__restrict__ xlast, const T *__restrict__ t, int64_t d,
                                                 double *scal, const int *ctrl) {
    if (cg_done(ctrl)) return;
    __shared__ T red[8];
    T s = T(0);
    for (int64_t k = threadIdx.x; k < d; k += blockDim.x) s = fma(xlast[k], t[k], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        T v = T(0);
        for (int w = 0; w < 8; ++w) v += red[w];
        scal[S_XLT] = static_cast<double>(v);
    }
}

// Row dot products with a d-vector: out[i] = <X[r0 + i], w> + add (one warp per row).
//  mode 0 (predict):  f_i = <z_i, w> + b, label
//  mode 1 (low-rank): v_i = <x_i, t> + u_i / C,  y_i = v_i - v_{m-1} for i < m-1 (0 beyond);
//                     v_{m-1} = <x_{m-1}, t> (scal[S_XLT], k_lastdot) - sum p / C
template <typename T>
__global__ void __launch_bounds__(256) k_rowdot(const T *__restrict__ X, int64_t d, int64_t r0, int64_t nrows,
                                                const T *__restrict__ w, int mode, T add, const T *__restrict__ p,
                                                int64_t m, T invC, const double *scal, T *__restrict__ out,
                                                int32_t *__restrict__ labels, const int *ctrl) {
    if (cg_done(ctrl)) return;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= nrows) return;
    const int64_t i = r0 + row;
    T s = T(0), sl = T(0);
    const bool real = i < m;
    if ((d & 1) == 0) {  // feature pairs (vec2 loads), 4 per lane in flight per step
        using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
        const int64_t d2 = d >> 1;
        const V2 *xr = reinterpret_cast<const V2 *>(X + (real ? i : 0) * d);
        const V2 *w2 = reinterpret_cast<const V2 *>(w);
        constexpr int U = 4;
        for (int64_t k0 = lane; k0 < d2; k0 += 32 * U) {
            V2 xv[U], wv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t k2 = k0 + 32 * u;
                const bool in = k2 < d2;
                wv[u] = in ? w2[k2] : V2{};
                xv[u] = (in && real) ? xr[k2] : V2{};
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                s = fma(xv[u].x, wv[u].x, s);
                s = fma(xv[u].y, wv[u].y, s);
            }
        }
    } else {
        for (int64_t k = lane; k < d; k += 32)
            if (real) s = fma(X[i * d + k], w[k], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (mode == 1) sl = static_cast<T>(scal[S_XLT]);
    if (lane != 0) return;
    if (mode == 0) {
        const T f = s + add;
        if (out) out[row] = f;
        if (labels) labels[row] = f >= T(0) ? 1 : -1;
    } else {
        const T sp = static_cast<T>(scal[S_SP]);
        const T vl = sl - sp * invC;                       // u_{m-1} = -sum p
        const T v = s + (i < m - 1 ? p[i] : T(0)) * invC;  // u_i = p_i
        out[row] = (i < m - 1) ? v - vl : T(0);
    }
}

// Circulant multi-GPU mode: this rank's partial product over ALL rows, y_i = sum_s Ypart[s][i]
// in fixed slot order (slots this rank did not write were zeroed); reduce-scattered afterwards.
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_slot_sum(const T *__restrict__ Ypart, int nslots, int64_t rows, int64_t m1, T *__restrict__ y, const int *ctrl) {
    // k_finalize's layout: 32-row chunks x 8 slot groups, fixed-order combine (deterministic)
    constexpr int G = kVecThreads / 32;
    __shared__ T grp[G][33];
    if (cg_done(ctrl)) return;
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const int64_t nchunks = (rows + 31) / 32;
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int64_t i = ch * 32 + lane;
        T sg = T(0);
        if (i < rows)
            for (int k = q; k < nslots; k += G) sg += Ypart[static_cast<int64_t>(k) * rows + i];
        grp[q][lane] = sg;
        __syncthreads();
        if (q == 0 && i < rows) {
            T s = T(0);
#pragma unroll
            for (int g = 0; g < G; ++g) s += grp[g][lane];
            y[i] = i < m1 ? s : T(0);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// CG vector kernels on this rank's band (local length nb, rows with global index >= m1 are
// padding and stay 0).  Scalars live in `scal` (double) so no host round trip is needed.

// Slot group q of row i: sum_{k = q, q + 8, ...} Ypart[k][i] in increasing k (the fixed order), with the
// loads issued 8 at a time ahead of the adds (the sum was a chain of dependent L2 round trips: 16 per
// row at C1, ~11 us of the fused CG kernel's 16).  Slot validity (k_matvec_implicit): with NSUB = 2
// column sub-blocks, the odd slot of an in-band column block J below row block R carries nothing.
template <typename T>
__device__ __forceinline__ T slot_group_sum(const T *__restrict__ Ypart, int nslots, int nsub, int band0, int R,
                                            int64_t nb, int64_t i, int q) {
    constexpr int G = kVecThreads / 32, U = 8;
    T sg = T(0);
    for (int k0 = q; k0 < nslots; k0 += G * U) {
        T v[U];
        bool use[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u * G;
            use[u] = k < nslots && !(nsub == 2 && (k & 1) && (k >> 1) >= band0 && (k >> 1) < R);
            v[u] = use[u] ? Ypart[static_cast<int64_t>(k) * nb + i] : T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (use[u]) sg += v[u];
    }
    return sg;
}

// y_i = sum_s Ypart[s][i] (fixed slot order), then pAp = p . y  (mode 0), or for the initial
// / replaced residual (mode 1): r_i = rhs_i - y_i, r.r -> S_DELTA+par (and S_DELTA0 if init);
// par < 0: take the slot from the device iteration counter.
// Layout: a block takes 32-row chunks; thread (row lane r = tid % 32, slot group q = tid / 32) sums
// slots q, q + 8, q + 16, ... of its row (8 independent load streams per row: the slot sum is
// bandwidth-, not latency-bound; C2 cached reads 512 slots), then warp 0 adds the 8 group
// partials in fixed order -- deterministic.
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_finalize(const T *__restrict__ Ypart, int nslots, int nsub, int band0, int64_t nb, int64_t g0, int64_t m1,
               const T *__restrict__ pband, T *__restrict__ y, int mode, const T *__restrict__ yl, T *__restrict__ r,
               T *__restrict__ pout, double *scal, int par, int set_delta0, T *partials, unsigned *counter,
               int write_scalar, const int *ctrl, int pap_slot) {
    constexpr int G = kVecThreads / 32;  // slot groups
    __shared__ T grp[G][33];
    if (cg_done(ctrl)) return;
    if (par < 0) par = (ctrl[C_IT] & 1) ^ 1;  // residual replacement: the slot of delta_{k+1}
    T part = T(0);
    const double ym = scal[S_YM];
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const int64_t nchunks = (nb + 31) / 32;
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int64_t i = ch * 32 + lane;
        // Slot validity (k_matvec_implicit): with NSUB = 2 column sub-blocks, the odd slot of an
        // in-band column block J below this row block R carries nothing (mirrored column sums
        // go to the even slot).  R is uniform over a 32-row chunk.
        const int R = static_cast<int>((g0 + ch * 32) / kTile);
        const T sg = (i < nb) ? slot_group_sum<T>(Ypart, nslots, nsub, band0, R, nb, i, q) : T(0);
        grp[q][lane] = sg;
        __syncthreads();
        if (q == 0 && i < nb) {
            T s = T(0);
#pragma unroll
            for (int g = 0; g < G; ++g) s += grp[g][lane];
            const bool valid = (g0 + i) < m1;
            s = valid ? s : T(0);
            if (mode == 0) {
                y[i] = s;
                part = fma(pband[i], s, part);
            } else {
                // rhs_i = y_i - y_m (Eq. 14)
                const T rhs = valid ? static_cast<T>(static_cast<double>(yl[g0 + i]) - ym) : T(0);
                const T ri = valid ? rhs - s : T(0);
                r[i] = ri;
                if (pout) pout[i] = ri;
                part = fma(ri, ri, part);
            }
        }
        __syncthreads();
    }
    grid_reduce<T>(part, partials, counter, [&](T tot) {
        if (!write_scalar) return;
        if (mode == 0) {
            scal[pap_slot] = scal[pap_slot + S_L] = static_cast<double>(tot);
        } else {
            scal[S_DELTA + par] = scal[S_DELTA + par + S_L] = static_cast<double>(tot);
            if (set_delta0) scal[S_DELTA0] = scal[S_DELTA0 + S_L] = static_cast<double>(tot);
        }
    });
}

// Local partial of a scalar only (multi-rank: the partial is all-reduced by NCCL before use).
// x += a p ; r -= a y ; delta_new = r.r   with a = delta_k / pAp  (Shewchuk)
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_update_xr(T *__restrict__ x, T *__restrict__ r, const T *__restrict__ p, const T *__restrict__ y, int64_t nb,
                double *scal, const int *ctrl, T *partials, unsigned *counter) {
    if (cg_done(ctrl)) return;
    const int par = ctrl[C_IT] & 1;
    const T a = static_cast<T>(scal[S_DELTA + par] / scal[S_PAP]);
    T part = T(0);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        x[i] = fma(a, p[i], x[i]);
        const T ri = fma(-a, y[i], r[i]);
        r[i] = ri;
        part = fma(ri, ri, part);
    }
    grid_reduce<T>(part, partials, counter, [&](T tot) {
        scal[S_DELTA + (par ^ 1)] = scal[S_DELTA + (par ^ 1) + S_L] = static_cast<double>(tot);
        scal[S_ALPHA] = static_cast<double>(a);
    });
}

// p = r + b p  with b = delta_{k+1} / delta_k; the last block then advances the iteration counter
// and evaluates Shewchuk's loop condition (i < imax and delta > eps^2 delta_0) and the
// breakdown test (p.Q~p <= 0 or non-finite).  With fixed > 0 the loop runs exactly
// `fixed` iterations.
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_update_p(T *__restrict__ p, const T *__restrict__ r, int64_t nb, double *scal, int *ctrl,
               unsigned *counter, cudaGraphConditionalHandle loop, int use_loop, T *const *__restrict__ peer_p,
               int npeer, int64_t g0) {
    if (cg_done(ctrl)) {
        if (use_loop && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(loop, 0u);
        return;
    }
    const int par = ctrl[C_IT] & 1;
    const T b = static_cast<T>(scal[S_DELTA + (par ^ 1)] / scal[S_DELTA + par]);
    // npeer > 0 (single-process multi-GPU, PEER transport): the all-gather of p fused into the update --
    // the new band goes straight into every rank's full p (peer_p[q] + g0, NVLink P2P stores; this
    // rank's own buffer is one of them), so no separate exchange of p follows (comm.cu)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const T v = fma(b, p[i], r[i]);
        if (npeer > 0) {
            for (int q = 0; q < npeer; ++q) peer_p[q][g0 + i] = v;
        } else {
            p[i] = v;
        }
    }
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        const int it = ctrl[C_IT] + 1;
        const double pap = scal[S_PAP], dnew = scal[S_DELTA + (par ^ 1)];
        int done = 0;
        if (!(pap > 0.0) || !isfinite(pap) || !isfinite(dnew)) done = 2;
        else if (ctrl[C_FIXED] > 0 ? (it >= ctrl[C_FIXED] || dnew == 0.0) : (dnew <= scal[S_THR])) done = 1;
        else if (it >= ctrl[C_IMAX]) done = 1;
        if (done == 0 && ctrl[C_REPL] > 0 && ctrl[C_FIXED] <= 0) {
            // stagnation guard (R-20, the oracle's rule): a 4x drop of delta below the best
            // resets the window; no such drop within W = 2 max(R, 50) iterations stops the loop
            const int R = ctrl[C_REPL];
            const int W = 2 * (R > 50 ? R : 50);
            double *best = scal + S_BEST;
            if (dnew < 0.25 * *best) {
                *best = dnew;
                ctrl[C_IBEST] = it;
            } else if (it - ctrl[C_IBEST] >= W) {
                done = 3;
            }
        }
        ctrl[C_IT] = it;
        ctrl[C_DONE] = done;
        *counter = 0u;
        // CUDA-graph CG loop (plssvm_cg_loop_t GRAPH): the WHILE node repeats while not done
        if (use_loop) cudaGraphSetConditional(loop, done == 0 ? 1u : 0u);
    }
}

// Block partial of a sum (grid_reduce's first half): warp shuffle tree, then the warps in order.
template <typename T>
__device__ __forceinline__ void block_partial(T v, T *partials) {
    __shared__ T red[kVecThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        T s = T(0);
        for (int w = 0; w < kVecThreads / 32; ++w) s += red[w];
        partials[blockIdx.x] = s;
    }
}
// The total of the block partials in grid_reduce's fixed order (lane-strided, then a shuffle tree),
// computed by every block after a grid barrier: all blocks hold the identical value.
template <typename T>
__device__ __forceinline__ T grid_total(const T *partials) {
    __shared__ T tot;
    if (threadIdx.x < 32) {
        T s = T(0);
        for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += 32) s += ((volatile const T *)partials)[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) tot = s;
    }
    __syncthreads();
    return tot;
}

// One Shewchuk CG iteration after the product, in ONE cooperative launch (single GPU, no residual
// replacement): k_finalize (y = sum of the slots in fixed order, pAp = p.y) | grid barrier |
// k_update_xr (a = delta_k / pAp; x += a p; r -= a y; delta_{k+1} = r.r) | grid barrier | k_update_p
// (b = delta_{k+1} / delta_k; p = r + b p; loop condition and breakdown test).
// The same arithmetic in the same order as the three kernels (same per-thread accumulations, block
// trees and fixed-order grid totals), so the iterates are bit-identical; two launches and their
// gaps per iteration fewer.  Partials: two arrays of gridDim.x (one per reduction).
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_cg_fused(const T *__restrict__ Ypart, int nslots, int nsub, int band0, int64_t nb, int64_t g0, int64_t m1,
               T *__restrict__ x, T *__restrict__ r, T *__restrict__ p, T *__restrict__ y, double *scal, int *ctrl,
               T *partials, cudaGraphConditionalHandle loop, int use_loop) {
    namespace cg = cooperative_groups;
    constexpr int G = kVecThreads / 32;
    __shared__ T grp[G][33];
    if (cg_done(ctrl)) {  // read by every block before the first barrier; written only after the last
        if (use_loop && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(loop, 0u);
        return;
    }
    cg::grid_group grid = cg::this_grid();
    const int par = ctrl[C_IT] & 1;
    // ---- k_finalize (mode 0)
    T part = T(0);
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const int64_t nchunks = (nb + 31) / 32;
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int64_t i = ch * 32 + lane;
        const int R = static_cast<int>((g0 + ch * 32) / kTile);
        const T sg = (i < nb) ? slot_group_sum<T>(Ypart, nslots, nsub, band0, R, nb, i, q) : T(0);
        grp[q][lane] = sg;
        __syncthreads();
        if (q == 0 && i < nb) {
            T s = T(0);
#pragma unroll
            for (int g = 0; g < G; ++g) s += grp[g][lane];
            s = (g0 + i) < m1 ? s : T(0);
            y[i] = s;
            part = fma(p[i], s, part);
        }
        __syncthreads();
    }
    block_partial<T>(part, partials);
    grid.sync();
    const T pap = grid_total<T>(partials);
    // ---- k_update_xr
    const T a = static_cast<T>(scal[S_DELTA + par] / static_cast<double>(pap));
    part = T(0);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        x[i] = fma(a, p[i], x[i]);
        const T ri = fma(-a, y[i], r[i]);
        r[i] = ri;
        part = fma(ri, ri, part);
    }
    block_partial<T>(part, partials + gridDim.x);
    grid.sync();
    const T dnew_t = grid_total<T>(partials + gridDim.x);
    // ---- k_update_p
    const double dnew = static_cast<double>(dnew_t);
    const T b = static_cast<T>(dnew / scal[S_DELTA + par]);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = fma(b, p[i], r[i]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const double papd = static_cast<double>(pap);
        scal[S_PAP] = scal[S_PAP + S_L] = papd;
        scal[S_DELTA + (par ^ 1)] = scal[S_DELTA + (par ^ 1) + S_L] = dnew;
        scal[S_ALPHA] = static_cast<double>(a);
        const int it = ctrl[C_IT] + 1;
        int done = 0;
        if (!(papd > 0.0) || !isfinite(papd) || !isfinite(dnew)) done = 2;
        else if (ctrl[C_FIXED] > 0 ? (it >= ctrl[C_FIXED] || dnew == 0.0) : (dnew <= scal[S_THR])) done = 1;
        else if (it >= ctrl[C_IMAX]) done = 1;
        ctrl[C_IT] = it;
        ctrl[C_DONE] = done;
        if (use_loop) cudaGraphSetConditional(loop, done == 0 ? 1u : 0u);
    }
}

// k_update_p with the all-gather of p fused in through the NCCL device API (one process per GPU,
// NCCL transport, every rank load/store accessible over NVLink, the P2P path
// the paper lacks): p lives in an NCCL symmetric window; each thread stores its new element
// p_i = r_i + b p_i into EVERY rank's window at the same offset (ncclGetLsaPointer, NVLink stores;
// this rank's own copy is one of them), then block b meets block b of every rank in an LSA barrier
// (release / acquire), so when this kernel completes on a rank every rank's band has landed in its
// p.  (A rank writes a peer's p only after that peer's product of the iteration: the scalar all-
// reduces in between order it.)  Then k_update_p's loop condition (last block).  The convergence
// decision is taken from global scalars, so all ranks skip the barrier together once done.
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_update_p_lsa(T *__restrict__ p, const T *__restrict__ r, int64_t nb, double *scal, int *ctrl, unsigned *counter,
                   ncclDevComm dev, ncclWindow_t win, int64_t g0) {
    if (cg_done(ctrl)) return;
    const int par = ctrl[C_IT] & 1;
    const T b = static_cast<T>(scal[S_DELTA + (par ^ 1)] / scal[S_DELTA + par]);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const T v = fma(b, p[i], r[i]);
        const size_t off = static_cast<size_t>(g0 + i) * sizeof(T);
        for (int q = 0; q < dev.lsaSize; ++q) *static_cast<T *>(ncclGetLsaPointer(win, off, q)) = v;
    }
    {
        ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dev, ncclTeamTagLsa(), blockIdx.x);
        bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    }
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        const int it = ctrl[C_IT] + 1;
        const double pap = scal[S_PAP], dnew = scal[S_DELTA + (par ^ 1)];
        int done = 0;
        if (!(pap > 0.0) || !isfinite(pap) || !isfinite(dnew)) done = 2;
        else if (ctrl[C_FIXED] > 0 ? (it >= ctrl[C_FIXED] || dnew == 0.0) : (dnew <= scal[S_THR])) done = 1;
        else if (it >= ctrl[C_IMAX]) done = 1;
        ctrl[C_IT] = it;
        ctrl[C_DONE] = done;
        *counter = 0u;
    }
}

// Entry node of the CUDA-graph CG loop: the WHILE condition = "not done" (k_cg_start's verdict).
__global__ void k_cg_loop_init(cudaGraphConditionalHandle loop, const int *ctrl) {
    cudaGraphSetConditional(loop, ctrl[C_DONE] == 0 ? 1u : 0u);
}

// Chronopoulos-Gear CG (options.cg_variant SINGLE_REDUCTION; Chronopoulos & Gear 1989): the
// product is taken of r instead of p (w = Q~ r), and s = Q~ p is carried by recurrence, so both
// inner products of an iteration, gamma = r.r and delta = w.r, come from ONE reduction point
// (one all-reduce of the pair on several GPUs instead of two).  Mathematically the CG iterates
// of Shewchuk's loop.  Entry: r_i, w_i = Q~ r_i (band), gamma_i, delta_i global.
// Loop condition on gamma_i (same threshold eps^2 delta_0 as the Shewchuk loop), breakdown if
// the p.Q~p equivalent delta_i - beta gamma_i / alpha_{i-1} <= 0; otherwise
//   beta = gamma_i / gamma_{i-1}, alpha = gamma_i / (delta_i - beta gamma_i / alpha_{i-1})
//   p = r + beta p ; s = w + beta s ; x += alpha p ; r -= alpha s ; gamma_{i+1} = r.r (partial)
// Every block takes the same verdict from the same scalars; block 0 records it.
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_cgcg_update(T *__restrict__ x, T *__restrict__ r, T *__restrict__ p, T *__restrict__ s, const T *__restrict__ w,
                  int64_t nb, double *scal, int *ctrl, T *partials, unsigned *counter, cudaGraphConditionalHandle loop,
                  int use_loop) {
    if (cg_done(ctrl)) {
        if (use_loop && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(loop, 0u);
        return;
    }
    const int it = ctrl[C_IT];
    const double g = scal[S_CG_GAMMA], dl = scal[S_CG_DELTA];
    double beta = 0.0, den = dl;
    if (it > 0) {
        beta = g / scal[S_CG_GPREV];
        den = dl - beta * g / scal[S_CG_APREV];
    }
    int done = 0;
    if (ctrl[C_FIXED] > 0 ? (it >= ctrl[C_FIXED] || g == 0.0) : (g <= scal[S_THR])) done = 1;
    else if (it >= ctrl[C_IMAX]) done = 1;
    else if (!(den > 0.0) || !isfinite(den) || !isfinite(g)) done = 2;
    if (done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctrl[C_DONE] = done;
            if (use_loop) cudaGraphSetConditional(loop, 0u);
        }
        return;
    }
    const double alpha = g / den;
    const T a = static_cast<T>(alpha), b = static_cast<T>(beta);
    T part = T(0);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const T pi = fma(b, p[i], r[i]);
        const T si = fma(b, s[i], w[i]);
        p[i] = pi;
        s[i] = si;
        x[i] = fma(a, pi, x[i]);
        const T ri = fma(-a, si, r[i]);
        r[i] = ri;
        part = fma(ri, ri, part);
    }
    grid_reduce<T>(part, partials, counter, [&](T tot) {
        scal[S_CG_GAMMA] = scal[S_CG_GAMMA + S_L] = static_cast<double>(tot);
        scal[S_CG_GPREV] = g;
        scal[S_CG_APREV] = alpha;
        scal[S_ALPHA] = alpha;
        ctrl[C_IT] = it + 1;
    });
}

// Loop entry (after delta_0 is final on every rank): threshold and control block.
__global__ void k_cg_start(double *scal, int *ctrl, double eps2, int imax, int fixed, int repl) {
    const double d0 = scal[S_DELTA0];
    scal[S_BEST] = d0;
    ctrl[C_REPL] = repl;
    ctrl[C_IBEST] = 0;
    scal[S_CG_GAMMA] = d0;  // Chronopoulos-Gear: gamma_0 = r_0.r_0 (global and this rank's partial)
    scal[S_CG_GAMMA + S_L] = scal[S_DELTA0 + S_L];
    scal[S_THR] = eps2 * d0;
    ctrl[C_IT] = 0;
    ctrl[C_IMAX] = imax;
    ctrl[C_FIXED] = fixed;
    ctrl[C_DONE] = (imax <= 0 || (fixed > 0 ? d0 == 0.0 : d0 <= eps2 * d0)) ? 1 : 0;
}

// x = x0 (0 or 1 on valid rows), and, for x0 = 0, r = p = rhs, delta0 = r.r.
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_init(T *__restrict__ x, T *__restrict__ r, T *__restrict__ p, const T *__restrict__ yl, int64_t nb, int64_t g0,
           int64_t m1, T x0, int zero_start, double *scal, T *partials, unsigned *counter, int write_scalar) {
    const double ym = scal[S_YM];
    T part = T(0);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool valid = (g0 + i) < m1;
        x[i] = valid ? x0 : T(0);
        if (zero_start) {
            const T rhs = valid ? static_cast<T>(static_cast<double>(yl[g0 + i]) - ym) : T(0);
            r[i] = rhs;
            p[i] = rhs;
            part = fma(rhs, rhs, part);
        }
    }
    if (zero_start)
        grid_reduce<T>(part, partials, counter, [&](T tot) {
            if (write_scalar) {
                scal[S_DELTA + 0] = scal[S_DELTA + S_L] = static_cast<double>(tot);
                scal[S_DELTA0] = scal[S_DELTA0 + S_L] = static_cast<double>(tot);
            }
        });
}

// Bias (Eq. 15): partial sums sum(x) and <q, x> over the band (two grid reductions).
template <typename T>
__global__ void __launch_bounds__(kVecThreads)
    k_bias_sums(const T *__restrict__ x, const T *__restrict__ q, int64_t nb, int64_t g0, double *scal, int which,
                T *partials, unsigned *counter) {
    T part = T(0);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        part = (which == 0) ? part + x[i] : fma(q[g0 + i], x[i], part);
    grid_reduce<T>(part, partials, counter, [&](T tot) {
        const int sl = which == 0 ? S_SUMX : S_QX;
        scal[sl] = scal[sl + S_L] = static_cast<double>(tot);
    });
}

// b = y_m + Q_mm sum(x) - <q,x> (Eq. 15); alpha = (x_0..x_{m-2}, -sum x).
template <typename T>
__global__ void k_assemble(const T *__restrict__ xfull, int64_t m, double *scal, T *__restrict__ alpha, T *__restrict__ bout) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const T sx = static_cast<T>(scal[S_SUMX]);
    if (i < m - 1) alpha[i] = xfull[i];
    if (i == m - 1) {
        alpha[i] = -sx;
        const T b = static_cast<T>(scal[S_YM]) + static_cast<T>(scal[S_QMM]) * sx - static_cast<T>(scal[S_QX]);
        *bout = b;
        scal[S_B] = static_cast<double>(b);
    }
}

// ---------------------------------------------------------------------------------------
// Predict (Eq. 10): tiles (I over test points Z, J over training points X); the epilogue
// forms alpha_j k(z_i, x_j) and row-reduces into Fpart[J][i] (deterministic slots).
// ldz / ldx: leading dimensions of the two arrays in the engine layout.
template <int KT, typename T>
__global__ void __launch_bounds__(Engine<T>::THREADS, Engine<T>::MIN_BLOCKS)
    k_predict_tiles(const __grid_constant__ Ops<T> ops, int64_t npad, int64_t dpad, const T *__restrict__ nz,
                    const T *__restrict__ nx, const T *__restrict__ alpha, KParams<T> kp, int tilesI,
                    T *__restrict__ Fpart) {
    using E = Engine<T>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    T *smem = align_smem<T>(smem_raw);
    const int I = blockIdx.x % tilesI, Jc = blockIdx.x / tilesI;
    const int64_t row0 = static_cast<int64_t>(I) * kTile, col0 = static_cast<int64_t>(Jc) * E::TN;
    T acc[E::R][E::CC];
    E::contract(ops, static_cast<int>(row0), static_cast<int>(col0), dpad, smem, acc);
    T rs[E::R];
#pragma unroll
    for (int i = 0; i < E::R; ++i) {
        const int64_t gi = row0 + E::row_of(i);
        const T ni = (KT == RBF) ? nz[gi] : T(0);
        T s = T(0);
#pragma unroll
        for (int j = 0; j < E::CC; ++j) {
            const int64_t gj = col0 + E::col_of(j);
            const T nj = (KT == RBF) ? nx[gj] : T(0);
            const T kv = kernel_value<KT, T>(acc[i][j], ni, nj, false, kp);
            s = fma(alpha[gj], kv, s);
        }
        rs[i] = s;
    }
    T *redr = smem;
    E::reduce_rows(rs, redr);
    __syncthreads();
    for (int t = threadIdx.x; t < kTile; t += E::THREADS)
        Fpart[static_cast<int64_t>(Jc) * npad + row0 + t] = E::row_total(redr, t);
}

template <typename T>
__global__ void k_norms(const T *__restrict__ X, int64_t mpad, int64_t dpad, int64_t n, int64_t d, T *__restrict__ nrm,
                        int64_t ld_raw = 0) {
    // ld_raw > 0: X is the caller's row-major n x d array (row stride ld_raw), rows n .. mpad - 1 get 0
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= (ld_raw > 0 ? mpad : n)) return;
    T s = T(0);
    for (int64_t k = lane; k < d; k += 32) {
        const T a = ld_raw > 0 ? (i < n ? X[i * ld_raw + k] : T(0)) : elem(X, i, k, mpad, dpad);
        s = fma(a, a, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) nrm[i] = s;
}

// f_i = sum_J Fpart[J][i] + b ; label = f >= 0 ? +1 : -1
template <typename T>
__global__ void k_predict_finalize(const T *__restrict__ Fpart, int nslots, int64_t npad, int64_t n, T b,
                                   T *__restrict__ f, int32_t *__restrict__ labels) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T s = T(0);
    for (int k = 0; k < nslots; ++k) s += Fpart[static_cast<int64_t>(k) * npad + i];
    const T v = s + b;
    if (f) f[i] = v;
    if (labels) labels[i] = (v >= T(0)) ? 1 : -1;
}

}  // namespace plssvm
