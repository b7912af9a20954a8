// tile_engine.cuh -- the blocked pairwise-contraction engines shared by the three tile kernels
// (implicit Q~p, Q~ precompute, predict).
//
// Paper design it re-derives (§III-C): blocking with padding "at least
// the size of a full block", block-level caching of 2*blocksize points' feature
// slabs in shared memory and thread-level register blocking.
//
// A CTA owns a 128 x TN tile S = X_I X_J^T (row block I, column block J); the contraction over
// features runs in 128-byte feature slabs staged by a 4-deep cp.async ring.
//
//  * fp64 (Engine<double>): DMMA.8x8x4 tensor-core MMAs (mma.sync m8n8k4 f64; tcgen05 has no
//    f64 kind).  Measured on this B200: DMMA 37.1 TFLOP/s vs DFMA 33.4 (profiles/r01_fp64_peak.txt).
//    The device layout is POINT-major, X[mpad][dpad] (features contiguous), so one 16-byte
//    LDS.128 feeds a thread's A (or B) value for two MMAs: MMA "a" uses feature 2q, MMA "b"
//    feature 2q+1 of each 8-feature group (q = lane % 4; the contraction over k is order-free,
//    A and B use the same permutation).  Smem rows are 128 B with the chunk swizzle
//    c ^ (row & 7), and fragment row rho maps to tile row pi(rho) = (rho >> 1) | ((rho & 1) << 2)
//    so the 8 lanes of each LDS.128 phase hit 8 distinct 16-byte bank groups (no conflicts).
//    4 warps (M) per CTA, warp tile 32 x 64 = 4 x 8 MMA tiles, 64 fp64 accumulators/thread,
//    CTA tile 128 x 64, two CTAs per SM (epilogue of one overlaps the MMAs of the other).
//  * fp32 (Engine<float>): 256 threads, 128 x 128 tile, FFMA register micro-tiles 8 x 8 on the FEATURE-major layout
//    X^T[dpad][mpad] (the paper's column-major layout); thread (ry, rx) owns rows
//    ry*4 + 64u + v, every smem read is one conflict-free LDS.128.
#pragma once
#include <cuda.h>

#include <type_traits>

#include "common.cuh"

namespace plssvm {

// Operands of a tile kernel.  fp64: two TMA descriptors over the point-major array(s) (box
// 16 features x 128 rows for the row operand, 16 x 64 for the column operand, SWIZZLE_128B);
// fp32 (FFMA engine): plain pointers into the feature-major arrays with their leading dimension.
template <typename T>
struct Ops;
template <>
struct Ops<double> {
    CUtensorMap a, b;
};
template <>
struct Ops<float> {
    const float *a, *b;
    int64_t ld;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbarrier_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbarrier_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity));
}
__device__ __forceinline__ void mbarrier_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbarrier_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

template <typename T>
__device__ __forceinline__ T *align_smem(unsigned char *raw) {
    return reinterpret_cast<T *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T>
struct Engine;

// =====================================================================================
// fp64: DMMA engine on the point-major layout X[mpad][ld], ld = dpad.  CTA = 4 warps (128
// threads) owning a 128 x 64 tile (warp tile 32 x 64), two CTAs per SM: while one CTA runs its
// epilogue (kernel function, exp, reductions) the other keeps the tensor pipe busy.
template <>
struct Engine<double> {
    using T = double;
    static constexpr bool kPointMajor = true;
    static constexpr int THREADS = 128;
    static constexpr int MIN_BLOCKS = 2;           // CTAs per SM
    static constexpr int TN = 64;                  // tile columns (rows = kTile = 128)
    static constexpr int NSUB = kTile / TN;        // column sub-blocks per 128-block
    static constexpr int BK = 16;                  // features per slab (128 B per row)
    static constexpr int STAGES = 4;
    static constexpr int SLAB_A = kTile * BK, SLAB_B = TN * BK;
    static constexpr int STAGE = SLAB_A + SLAB_B;
    static constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE * sizeof(T) + 1024;  // 96 KiB + alignment
    static constexpr int R = 4;                    // accumulator rows per thread (m-tiles)
    static constexpr int CC = 16;                  // accumulator columns per thread (8 n-tiles x 2)

    __device__ static __forceinline__ int pi(int r) { return (r >> 1) | ((r & 1) << 2); }
    __device__ static __forceinline__ int wm() { return threadIdx.x >> 5; }
    __device__ static __forceinline__ int lane() { return threadIdx.x & 31; }
    // local tile row of accumulator row index i (0..R-1), local tile col of column index j (0..CC-1)
    __device__ static __forceinline__ int row_of(int i) { return wm() * 32 + i * 8 + pi(lane() >> 2); }
    __device__ static __forceinline__ int col_of(int j) { return (j >> 1) * 8 + pi(2 * (lane() & 3) + (j & 1)); }
    static constexpr uint32_t STAGE_BYTES = uint32_t(STAGE) * sizeof(T);

    __device__ static __forceinline__ void mma(double (&c)[2], double a, double b) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[0]), "+d"(c[1])
                     : "d"(a), "d"(b));
    }

    // acc[i][j] = S[row_of(i)][col_of(j)] = sum_k A[row0 + row][k] B[col0 + col][k].
    // TMA ring: thread 0 issues the two boxes of a slab (SWIZZLE_128B places 16-byte chunk c of
    // row r at c ^ (r & 7), the layout the fragment loads below expect) and completes them on
    // full[stage]; each warp releases a stage with one arrive on empty[stage] (count 4); thread 0
    // refills a stage once all four warps released it.  No block-wide barrier in the loop.
    __device__ static __forceinline__ void contract(const Ops<double> &ops, int row0, int col0, int64_t dpad, T *smem,
                                                    T (&acc)[R][CC]) {
        __shared__ uint64_t full[STAGES], empty[STAGES];
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int j = 0; j < CC; ++j) acc[i][j] = 0.0;
        const int nk = static_cast<int>(dpad / BK);
        if (threadIdx.x == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ops.a)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ops.b)) : "memory");
            for (int s = 0; s < STAGES; ++s) {
                mbarrier_init(&full[s], 1);
                mbarrier_init(&empty[s], THREADS / 32);
            }
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int s = 0; s < STAGES && s < nk; ++s) {
                mbarrier_expect_tx(&full[s], STAGE_BYTES);
                tma_2d(smem + s * STAGE, &ops.a, &full[s], s * BK, row0);
                tma_2d(smem + s * STAGE + SLAB_A, &ops.b, &full[s], s * BK, col0);
            }
        }
        const int ln = lane(), q = ln & 3, prow = pi(ln >> 2);
        const int arow = wm() * 32 + prow, brow = prow;
        for (int kb = 0; kb < nk; ++kb) {
            const int st = kb % STAGES;
            const uint32_t par = (kb / STAGES) & 1;
            mbarrier_wait(&full[st], par);
            const T *sA = smem + st * STAGE;
            const T *sB = sA + SLAB_A;
#pragma unroll
            for (int g = 0; g < BK / 8; ++g) {
                const int c = 4 * g + q;
                double2 a[4], b[8];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) {
                    const int r = arow + mt * 8;  // r & 7 == prow
                    a[mt] = *reinterpret_cast<const double2 *>(sA + r * BK + ((c ^ prow) << 1));
                }
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) {
                    const int r = brow + nt * 8;
                    b[nt] = *reinterpret_cast<const double2 *>(sB + r * BK + ((c ^ prow) << 1));
                }
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) {
                        double(&cc)[2] = *reinterpret_cast<double(*)[2]>(&acc[mt][2 * nt]);
                        mma(cc, a[mt].x, b[nt].x);
                    }
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 8; ++nt) {
                        double(&cc)[2] = *reinterpret_cast<double(*)[2]>(&acc[mt][2 * nt]);
                        mma(cc, a[mt].y, b[nt].y);
                    }
            }
            __syncwarp();
            if (ln == 0) mbarrier_arrive(&empty[st]);
            if (threadIdx.x == 0 && kb + STAGES < nk) {
                mbarrier_wait(&empty[st], par);
                mbarrier_expect_tx(&full[st], STAGE_BYTES);
                tma_2d(smem + st * STAGE, &ops.a, &full[st], (kb + STAGES) * BK, row0);
                tma_2d(smem + st * STAGE + SLAB_A, &ops.b, &full[st], (kb + STAGES) * BK, col0);
            }
        }
        __syncthreads();  // every stage consumed and no TMA in flight: the ring is free for the epilogue
    }

    // Row sums rs[i] (over this thread's columns) -> red[128] : each tile row is owned by one
    // warp and 4 lanes (deterministic shuffle tree).  Scratch: 128 elements.
    __device__ static __forceinline__ void reduce_rows(T (&rs)[R], T *red) {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 1);
            rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 2);
        }
        if ((lane() & 3) == 0) {
#pragma unroll
            for (int i = 0; i < R; ++i) red[row_of(i)] = rs[i];
        }
    }
    __device__ static __forceinline__ T row_total(const T *red, int t) { return red[t]; }
    // Column sums cs[j] (over this thread's rows) -> 4 warps x TN partials.  Scratch: 4*TN.
    __device__ static __forceinline__ void reduce_cols(T (&cs)[CC], T *red) {
#pragma unroll
        for (int j = 0; j < CC; ++j) {
            cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 4);
            cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 8);
            cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 16);
        }
        if ((lane() >> 2) == 0) {
#pragma unroll
            for (int j = 0; j < CC; ++j) red[wm() * TN + col_of(j)] = cs[j];
        }
    }
    __device__ static __forceinline__ T col_total(const T *red, int t) {
        return (red[t] + red[TN + t]) + (red[2 * TN + t] + red[3 * TN + t]);
    }
};

// =====================================================================================
// fp32: FFMA engine on the feature-major layout X^T[dpad][ld], ld = mpad.
template <>
struct Engine<float> {
    using T = float;
    static constexpr bool kPointMajor = false;
    static constexpr int THREADS = kThreads;
    static constexpr int MIN_BLOCKS = 1;
    static constexpr int TN = kTile;
    static constexpr int NSUB = 1;
    static constexpr int BK = 32;
    static constexpr int VEC = 4;
    static constexpr int STAGES = 4;
    static constexpr int SLAB = BK * kTile;
    static constexpr size_t SMEM_BYTES = size_t(STAGES) * 2 * SLAB * sizeof(T) + 1024;  // 128 KiB + alignment
    static constexpr int CPR = kTile * sizeof(T) / 16;  // 16-byte chunks per slab row (32)
    static constexpr int CHUNKS = BK * CPR / kThreads;  // 4
    static constexpr int R = 8, CC = 8;

    __device__ static __forceinline__ int ry() { return ((threadIdx.x >> 5) >> 1) * 4 + ((threadIdx.x & 31) >> 3); }
    __device__ static __forceinline__ int rx() { return ((threadIdx.x >> 5) & 1) * 8 + (threadIdx.x & 7); }
    __device__ static __forceinline__ int micro(int r, int e) { return r * VEC + (e / VEC) * (16 * VEC) + (e % VEC); }
    __device__ static __forceinline__ int row_of(int i) { return micro(ry(), i); }
    __device__ static __forceinline__ int col_of(int j) { return micro(rx(), j); }
    __device__ static __forceinline__ const T *block(const T *X, int64_t row0, int64_t) { return X + row0; }

    __device__ static __forceinline__ void load_slab(T *sA, T *sB, const T *__restrict__ A, const T *__restrict__ B,
                                                     int64_t ld, int64_t k0) {
#pragma unroll
        for (int u = 0; u < CHUNKS; ++u) {
            const int ch = threadIdx.x + u * kThreads;
            const int kr = ch / CPR, cc = ch % CPR;
            const int off = kr * kTile + cc * VEC;
            const int64_t g = (k0 + kr) * ld + cc * VEC;
            cp_async16(sA + off, A + g);
            cp_async16(sB + off, B + g);
        }
    }

    __device__ static __forceinline__ void contract(const Ops<float> &ops, int row0, int col0, int64_t dpad, T *smem,
                                                    T (&acc)[R][CC]) {
        const T *__restrict__ A = ops.a + row0;
        const T *__restrict__ B = ops.b + col0;
        const int64_t ld = ops.ld;
        const int y = ry(), x = rx();
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        const int nk = static_cast<int>(dpad / BK);
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (s < nk) load_slab(smem + s * 2 * SLAB, smem + s * 2 * SLAB + SLAB, A, B, ld, int64_t(s) * BK);
            cp_async_commit();
        }
        for (int kb = 0; kb < nk; ++kb) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            const int pf = kb + STAGES - 1;
            if (pf < nk) {
                const int st = pf % STAGES;
                load_slab(smem + st * 2 * SLAB, smem + st * 2 * SLAB + SLAB, A, B, ld, int64_t(pf) * BK);
            }
            cp_async_commit();
            const T *sA = smem + (kb % STAGES) * 2 * SLAB;
            const T *sB = sA + SLAB;
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                T a[8], b[8];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float4 va = *reinterpret_cast<const float4 *>(sA + kk * kTile + y * VEC + u * 16 * VEC);
                    const float4 vb = *reinterpret_cast<const float4 *>(sB + kk * kTile + x * VEC + u * 16 * VEC);
                    a[u * 4 + 0] = va.x; a[u * 4 + 1] = va.y; a[u * 4 + 2] = va.z; a[u * 4 + 3] = va.w;
                    b[u * 4 + 0] = vb.x; b[u * 4 + 1] = vb.y; b[u * 4 + 2] = vb.z; b[u * 4 + 3] = vb.w;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
        }
        cp_async_wait<0>();
        __syncthreads();
    }

    __device__ static __forceinline__ void reduce_rows(T (&rs)[R], T *red) {
#pragma unroll
        for (int e = 0; e < R; ++e) {
            rs[e] += __shfl_xor_sync(0xffffffffu, rs[e], 1);
            rs[e] += __shfl_xor_sync(0xffffffffu, rs[e], 2);
            rs[e] += __shfl_xor_sync(0xffffffffu, rs[e], 4);
        }
        const int w = threadIdx.x >> 5;
        if ((threadIdx.x & 7) == 0) {
#pragma unroll
            for (int e = 0; e < R; ++e) red[(w & 1) * kTile + row_of(e)] = rs[e];
        }
    }
    __device__ static __forceinline__ T row_total(const T *red, int t) { return red[t] + red[kTile + t]; }
    __device__ static __forceinline__ void reduce_cols(T (&cs)[CC], T *red) {
#pragma unroll
        for (int e = 0; e < CC; ++e) {
            cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], 8);
            cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], 16);
        }
        const int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) < 8) {
#pragma unroll
            for (int e = 0; e < CC; ++e) red[(w >> 1) * kTile + col_of(e)] = cs[e];
        }
    }
    __device__ static __forceinline__ T col_total(const T *red, int t) {
        return (red[t] + red[kTile + t]) + (red[2 * kTile + t] + red[3 * kTile + t]);
    }
};

// ---- kernel functions on a contracted value s = <x_i, x_j> -------------------
// RBF uses ||x_i - x_j||^2 = n_i + n_j - 2 s, clamped at 0, with the exact 0 on the diagonal
// (reading R-9).  Poly: integer degree by repeated multiplication (R-6).
template <int KT, typename T>
__device__ __forceinline__ T kernel_value(T s, T ni, T nj, bool diag, const KParams<T> &kp) {
    if constexpr (KT == LINEAR) {
        return s;
    } else if constexpr (KT == POLYNOMIAL) {
        // integer power by repeated multiplication (R-6).  Degrees 1-4 as a fixed
        // product sequence selected by the (warp-uniform, loop-invariant) degree: no per-entry loop
        // in the unrolled epilogues (the loop cost C3 12 %); b^3 = (b b) b as the oracle's order.
        const T b = kp.gamma * s + kp.coef0;
        const T b2 = b * b;
        const T b3 = b2 * b;
        if (kp.degree <= 4) return kp.degree == 1 ? b : kp.degree == 2 ? b2 : kp.degree == 3 ? b3 : b2 * b2;
        T r = b3;
        for (int t = 3; t < kp.degree; ++t) r *= b;
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
