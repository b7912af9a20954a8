// tile_engine.cuh -- the blocked pairwise-contraction engine shared by the three tile kernels
// (implicit Q~p, Q~ precompute, predict).
//
// Paper design it re-derives (§III-C): blocking with padding "at least
// the size of a full block", block-level caching of 2*blocksize points' feature
// slabs in shared memory and thread-level register blocking, over
// the feature-major ("column-major") data layout.
//
// sm_100a realisation: a CTA of 256 threads owns a 128 x 128 tile S = X_I X_J^T (row block I,
// column block J); the contraction over features runs in BK-wide slabs (BK*sizeof(T) = 128 B)
// staged by a 4-deep cp.async ring into shared memory; each thread keeps an 8 x 8 register
// micro-tile (DFMA for fp64, FFMA for fp32).  Thread (ry, rx) owns rows
// ry*VEC + u*16*VEC + v and the same pattern of columns (VEC = 16 B / sizeof(T)), so every
// shared-memory read is a 16-byte LDS.128 and a warp (4 ry x 8 rx) reads 64 B (A) / 128 B (B)
// contiguous bytes per instruction: one wavefront, no bank conflicts.
#pragma once
#include "common.cuh"

namespace plssvm {

template <typename T>
struct Tile {
    static constexpr int BK = 128 / sizeof(T);             // features per slab (16 fp64 / 32 fp32)
    static constexpr int VEC = 16 / sizeof(T);             // elements per 16-byte vector
    static constexpr int STAGES = 4;                       // cp.async ring depth
    static constexpr int SLAB = BK * kTile;                // elements of one operand slab
    static constexpr int SMEM_ELEMS = STAGES * 2 * SLAB;   // A and B rings
    static constexpr size_t SMEM_BYTES = SMEM_ELEMS * sizeof(T);  // 128 KiB
    static constexpr int CPR = kTile * sizeof(T) / 16;     // 16-byte chunks per slab row
    static constexpr int CHUNKS = BK * CPR / kThreads;     // chunks per thread per operand
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Local row (or column) index of the thread's micro-tile element e (0..7): ry*VEC + u*16*VEC + v.
template <typename T>
__device__ __forceinline__ int micro_index(int r, int e) {
    constexpr int VEC = Tile<T>::VEC;
    return r * VEC + (e / VEC) * (16 * VEC) + (e % VEC);
}

__device__ __forceinline__ int thread_ry() { return ((threadIdx.x >> 5) >> 1) * 4 + ((threadIdx.x & 31) >> 3); }
__device__ __forceinline__ int thread_rx() { return ((threadIdx.x >> 5) & 1) * 8 + (threadIdx.x & 7); }

template <typename T>
__device__ __forceinline__ void load_slab(T *sA, T *sB, const T *__restrict__ A, const T *__restrict__ B,
                                          int64_t ld, int64_t k0) {
    using C = Tile<T>;
#pragma unroll
    for (int u = 0; u < C::CHUNKS; ++u) {
        int ch = threadIdx.x + u * kThreads;
        int kr = ch / C::CPR, cc = ch % C::CPR;
        int off = kr * kTile + cc * C::VEC;
        const int64_t g = (k0 + kr) * ld + cc * C::VEC;
        cp_async16(sA + off, A + g);
        cp_async16(sB + off, B + g);
    }
}

// acc[i][j] = sum_k A[k*ld + row_i] * B[k*ld + col_j] over k < dpad, where A/B point at the
// first element of the row / column block in the feature-major array (ld = padded points).
template <typename T>
__device__ __forceinline__ void contract_tile(const T *__restrict__ A, const T *__restrict__ B, int64_t ld,
                                              int64_t dpad, T *smem, T (&acc)[8][8]) {
    using C = Tile<T>;
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    const int ry = thread_ry(), rx = thread_rx();
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = T(0);

    const int nk = static_cast<int>(dpad / C::BK);
#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
        if (s < nk) load_slab<T>(smem + s * 2 * C::SLAB, smem + s * 2 * C::SLAB + C::SLAB, A, B, ld,
                                 static_cast<int64_t>(s) * C::BK);
        cp_async_commit();
    }
    for (int kb = 0; kb < nk; ++kb) {
        cp_async_wait<C::STAGES - 2>();
        __syncthreads();
        const int pf = kb + C::STAGES - 1;
        if (pf < nk) {
            const int st = pf % C::STAGES;
            load_slab<T>(smem + st * 2 * C::SLAB, smem + st * 2 * C::SLAB + C::SLAB, A, B, ld,
                         static_cast<int64_t>(pf) * C::BK);
        }
        cp_async_commit();
        const T *sA = smem + (kb % C::STAGES) * 2 * C::SLAB;
        const T *sB = sA + C::SLAB;
#pragma unroll
        for (int kk = 0; kk < C::BK; ++kk) {
            T a[8], b[8];
#pragma unroll
            for (int u = 0; u < 8 / C::VEC; ++u) {
                V va = *reinterpret_cast<const V *>(sA + kk * kTile + ry * C::VEC + u * 16 * C::VEC);
                V vb = *reinterpret_cast<const V *>(sB + kk * kTile + rx * C::VEC + u * 16 * C::VEC);
                const T *pa = reinterpret_cast<const T *>(&va);
                const T *pb = reinterpret_cast<const T *>(&vb);
#pragma unroll
                for (int v = 0; v < C::VEC; ++v) {
                    a[u * C::VEC + v] = pa[v];
                    b[u * C::VEC + v] = pb[v];
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();  // ring is free for reuse by the epilogue
}

// ---- kernel functions on a contracted value s = <x_i, x_j> -------------------
// RBF uses ||x_i - x_j||^2 = n_i + n_j - 2 s, clamped at 0, with the exact 0 on the diagonal
// (reading R-9).  Poly: integer degree by repeated multiplication (R-6).
template <int KT, typename T>
__device__ __forceinline__ T kernel_value(T s, T ni, T nj, bool diag, const KParams<T> &kp) {
    if constexpr (KT == LINEAR) {
        return s;
    } else if constexpr (KT == POLYNOMIAL) {
        const T base = kp.gamma * s + kp.coef0;
        T r = T(1);
        for (int t = 0; t < kp.degree; ++t) r *= base;
        return r;
    } else {
        T dist = ni + nj - T(2) * s;
        dist = dist > T(0) ? dist : T(0);
        if (diag) dist = T(0);
        if constexpr (sizeof(T) == 4) return expf(-kp.gamma * dist);
        else return exp(-kp.gamma * dist);
    }
}

}  // namespace plssvm
