// tc_engine.cuh -- fp32 implicit Q~p on the 5th-generation tensor cores (tcgen05, kind::tf32)
// with 3xTF32 error compensation.
//
// Same contract as k_matvec_implicit<KT, float> (Eq. 16; symmetric tiles mirrored,
// P:385-389; deterministic Ypart slots), different contraction: S = X_I X_J^T for a 128 x 128
// tile is accumulated in TMEM by tcgen05.mma.cta_group::1.kind::tf32 (M = 128, N = 128, K = 8)
// issued by ONE thread; each fp32 operand is split x = hi + lo (hi = tf32(x), lo = tf32(x - hi),
// precomputed by k_split_tf32) and S = hi.hi^T + hi.lo^T + lo.hi^T (the lo.lo^T term, ~2^-22
// relative, is dropped): fp32-level accuracy (tools/tc_probe.cu: 1.9e-6 relative vs fp64).
//
// The same tile kernel also serves the fp32 cached-mode precompute and predict (TcMode).
// CTA = 6 warps, one CTA per tile, warp-specialised:
//   warp 4 (one lane): TMA producer -- 4 boxes of 128 rows x 128 B (A_hi, A_lo, B_hi, B_lo) per
//                      32-feature slab, SWIZZLE_128B, completion on full[stage] (expect_tx)
//   warp 5 (one lane): TMEM allocation + MMA issuer -- 12 UMMAs per slab, tcgen05.commit frees the
//                      stage (empty[stage]) and, after the last slab, signals the accumulator
//   warps 0-3        : epilogue -- tcgen05.ld 32x32b.x16 (warp w reads TMEM lanes 32w..32w+31 =
//                      tile rows), Q~ entry, row sums (a thread owns a full row), column sums
//                      by a 16-shuffle transpose-reduction per 16-column chunk + smem.
// Shared memory: 3 stages x 64 KiB operand ring (1024-B aligned for the 128-B swizzle).
#pragma once
#include <cuda.h>

#include "kernels.cuh"

namespace plssvm {

struct Tc {
    static constexpr int BK = 32;                              // fp32 features per slab (128 B rows)
    static constexpr int STAGES = 3;
    static constexpr int OPND = kTile * BK;                    // floats per operand tile (16 KiB)
    static constexpr uint32_t STAGE_BYTES = 4 * OPND * 4;      // A_hi, A_lo, B_hi, B_lo
    static constexpr int THREADS = 192;
    static constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_BYTES + 1024 /*align*/ + 4096 /*misc*/;
    // instruction descriptor: D f32, A/B tf32, K-major, N = 128, M = 128 (validated by tc_probe)
    static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
};

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// UMMA shared-memory descriptor, K-major operand in the 128-byte swizzle atom layout:
// start >> 4, LBO unused (0), SBO = 1024 B (8 rows x 128 B), version 1 (sm_100), SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return (uint64_t((saddr >> 4) & 0x3FFFu)) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
        "r"(parity));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes));
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(Tc::IDESC), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t *b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(b)));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Sum of v[0..15] over the 32 lanes of the warp in 16 shuffles: afterwards lane l holds the
// total of column (l >> 1) (lanes 2c and 2c+1 hold the same value).  Fixed order.
__device__ __forceinline__ float transpose_reduce16(const float (&v)[16], int lane) {
    float w8[8], w4[4], w2[2];
    const bool h1 = (lane >> 4) & 1, h2 = (lane >> 3) & 1, h3 = (lane >> 2) & 1, h4 = (lane >> 1) & 1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float send = h1 ? v[i] : v[i + 8];
        const float keep = h1 ? v[i + 8] : v[i];
        w8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float send = h2 ? w8[i] : w8[i + 4];
        const float keep = h2 ? w8[i + 4] : w8[i];
        w4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = h3 ? w4[i] : w4[i + 2];
        const float keep = h3 ? w4[i + 2] : w4[i];
        w2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const float send = h4 ? w2[0] : w2[1];
    const float keep = h4 ? w2[1] : w2[0];
    float w1 = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    return w1 + __shfl_xor_sync(0xffffffffu, w1, 1);
}

// hi/lo split into the point-major padded arrays (zero padding), X[m][d] -> Xhi/Xlo[mpad][dpad].
__global__ void k_split_tf32(const float *__restrict__ X, int64_t m, int64_t d, float *__restrict__ Xhi,
                             float *__restrict__ Xlo, int64_t mpad, int64_t dpad) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= mpad * dpad) return;
    const int64_t i = idx / dpad, k = idx % dpad;
    const float x = (i < m && k < d) ? X[i * d + k] : 0.f;
    uint32_t h, l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    const float hf = __uint_as_float(h);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hf));
    Xhi[idx] = hf;
    Xlo[idx] = __uint_as_float(l);
}

// Epilogue variants of the tcgen05 tile kernel.
enum TcMode : int { TC_MATVEC = 0, TC_PRECOMPUTE = 1, TC_PREDICT = 2 };

// One CTA per 128 x 128 tile (I, J): A = rows I of the A arrays, B = rows J of the B arrays.
//  TC_MATVEC     : Q~ entries -> row sums into Ypart[J] (rows of I) and, for mirrored tiles,
//                  column sums into Ypart[I] (rows of J)                      (same as k_matvec_implicit)
//  TC_PRECOMPUTE : Q~ entries -> the band's tiled cached array Qc (tile and mirrored tile)
//  TC_PREDICT    : alpha_j k(z_i, x_j) -> row sums into Ypart[J] (= Fpart, rows of test block I)
template <int KT, int MODE>
__global__ void __launch_bounds__(Tc::THREADS, 1)
    k_tile_tc(const __grid_constant__ CUtensorMap tma_hi, const __grid_constant__ CUtensorMap tma_lo,
              const __grid_constant__ CUtensorMap tmb_hi, const __grid_constant__ CUtensorMap tmb_lo, int64_t dpad,
              const int2 *__restrict__ tiles, int tilesI, const float *__restrict__ qa, const float *__restrict__ na,
              const float *__restrict__ qb, const float *__restrict__ nb_, const float *__restrict__ p,
              KParams<float> kp, float invC, const double *__restrict__ scal, int64_t m1, int band0, int band1,
              float *__restrict__ Ypart, int64_t band_rows, float *__restrict__ Qc, int T_tiles, const int *ctrl) {
    if (cg_done(ctrl)) return;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float *ring = reinterpret_cast<float *>(base);
    unsigned char *misc = base + size_t(Tc::STAGES) * Tc::STAGE_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(misc);          // [STAGES]
    uint64_t *empty = full + Tc::STAGES;                            // [STAGES]
    uint64_t *accf = empty + Tc::STAGES;                            // [1]
    uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(accf + 1);
    float *colq = reinterpret_cast<float *>(misc + 128);            // [128]
    float *colp = colq + kTile;                                     // [128]  (alpha for predict)
    float *coln = colp + kTile;                                     // [128]
    float *redc = coln + kTile;                                     // [4][128]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int I, J;
    if constexpr (MODE == TC_PREDICT) {
        I = blockIdx.x % tilesI;
        J = blockIdx.x / tilesI;
    } else {
        const int2 tile = tiles[blockIdx.x];
        I = tile.x;
        J = tile.y;
    }
    const int row0 = I * kTile, col0 = J * kTile;
    const int nk = static_cast<int>(dpad / Tc::BK);

    if (warp == 4 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_hi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_lo)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb_hi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb_lo)) : "memory");
        for (int s = 0; s < Tc::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accf, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_addr(tmem_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x < kTile) {
        const int64_t gj = col0 + threadIdx.x;
        colq[threadIdx.x] = (MODE == TC_PREDICT) ? 0.f : qb[gj];
        colp[threadIdx.x] = (MODE == TC_PRECOMPUTE) ? 0.f : p[gj];
        coln[threadIdx.x] = (KT == RBF) ? nb_[gj] : 0.f;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_sh;

    if (warp == 4) {
        if (lane == 0) {  // ---- TMA producer
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % Tc::STAGES;
                if (kb >= Tc::STAGES) mbar_wait(&empty[s], ((kb / Tc::STAGES) - 1) & 1);
                float *st = ring + size_t(s) * 4 * Tc::OPND;
                mbar_expect_tx(&full[s], Tc::STAGE_BYTES);
                const int x = kb * Tc::BK;
                tma_load_2d(st, &tma_hi, &full[s], x, row0);
                tma_load_2d(st + Tc::OPND, &tma_lo, &full[s], x, row0);
                tma_load_2d(st + 2 * Tc::OPND, &tmb_hi, &full[s], x, col0);
                tma_load_2d(st + 3 * Tc::OPND, &tmb_lo, &full[s], x, col0);
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {  // ---- MMA issuer
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % Tc::STAGES;
                mbar_wait(&full[s], (kb / Tc::STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t sa = smem_addr(ring + size_t(s) * 4 * Tc::OPND);
                const uint64_t dah = umma_desc_sw128(sa), dal = umma_desc_sw128(sa + Tc::OPND * 4);
                const uint64_t dbh = umma_desc_sw128(sa + 2 * Tc::OPND * 4), dbl = umma_desc_sw128(sa + 3 * Tc::OPND * 4);
#pragma unroll
                for (int kk = 0; kk < Tc::BK / 8; ++kk) {  // K = 8 tf32 = 32 B per UMMA -> +2 in the descriptor
                    const uint64_t o = uint64_t(kk * 2);
                    umma_tf32(tmem, dah + o, dbh + o, (kb > 0 || kk > 0) ? 1u : 0u);
                    umma_tf32(tmem, dah + o, dbl + o, 1u);
                    umma_tf32(tmem, dal + o, dbh + o, 1u);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(accf);
        }
    } else {  // ---- epilogue warps 0-3: thread = tile row 32w + lane
        const int lr = warp * 32 + lane;
        const int64_t gi = row0 + lr;
        const float qi = (MODE == TC_PREDICT) ? 0.f : qa[gi];
        const float pi = (MODE == TC_MATVEC) ? p[gi] : 0.f;
        const float ni = (KT == RBF) ? na[gi] : 0.f;
        const float Qmm = (MODE == TC_PREDICT) ? 0.f : static_cast<float>(scal[S_QMM]);
        const bool mirrored = (MODE != TC_PREDICT) && (I != J) && (J >= band0) && (J < band1);
        mbar_wait(accf, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        float rs = 0.f;
        float *qrow = nullptr, *qmir = nullptr;
        if constexpr (MODE == TC_PRECOMPUTE) {
            if (T_tiles < 0) {  // packed symmetric layout: ordinal blockIdx.x, no mirror copy
                qrow = Qc + int64_t(blockIdx.x) * (kTile * kTile) + lr * kTile;
            } else {
                qrow = Qc + (int64_t(I - band0) * T_tiles + J) * (kTile * kTile) + lr * kTile;
                if (mirrored) qmir = Qc + (int64_t(J - band0) * T_tiles + I) * (kTile * kTile) + lr;
            }
        }
#pragma unroll 1
        for (int c0 = 0; c0 < kTile; c0 += 16) {
            float v[16];
            tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
            if constexpr (MODE == TC_PREDICT) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int lc = c0 + j;
                    rs = fmaf(colp[lc], kernel_value<KT, float>(v[j], ni, coln[lc], false, kp), rs);
                }
            } else {
                float cs[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int lc = c0 + j;
                    const float qt = qtilde_value<KT, float>(v[j], gi, int64_t(col0 + lc), ni, coln[lc], qi, colq[lc],
                                                             Qmm, invC, m1, kp);
                    if constexpr (MODE == TC_MATVEC) {
                        rs = fmaf(qt, colp[lc], rs);
                        cs[j] = qt * pi;
                    } else {
                        cs[j] = qt;
                    }
                }
                if constexpr (MODE == TC_MATVEC) {
                    if (mirrored) {
                        const float t = transpose_reduce16(cs, lane);
                        if ((lane & 1) == 0) redc[warp * kTile + c0 + (lane >> 1)] = t;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<float4 *>(qrow + c0 + j) = make_float4(cs[j], cs[j + 1], cs[j + 2], cs[j + 3]);
                    if (qmir) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) qmir[(c0 + j) * kTile] = cs[j];  // coalesced over lanes
                    }
                }
            }
        }
        if constexpr (MODE == TC_MATVEC || MODE == TC_PREDICT) {
            const int64_t lrow0 = int64_t(row0) - int64_t(band0) * kTile;
            Ypart[int64_t(J) * band_rows + lrow0 + lr] = rs;
        }
        if constexpr (MODE == TC_MATVEC) {
            if (mirrored) {
                asm volatile("bar.sync 1, 128;");
                const int t = threadIdx.x;
                const int64_t lcol0 = int64_t(col0) - int64_t(band0) * kTile;
                Ypart[int64_t(I) * band_rows + lcol0 + t] =
                    (redc[t] + redc[kTile + t]) + (redc[2 * kTile + t] + redc[3 * kTile + t]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 5) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
    }
}

// =====================================================================================
// Wide variant: 128 x 256 tiles (UMMA N = 256), 16-feature slabs in a 4-stage ring with the
// 64-byte swizzle -- 25 % fewer operand bytes through L2 per useful flop than 128 x 128 (the
// 3xTF32 path is L2-bandwidth bound, profiles/r01_ncu_matvec_c3_tc.txt).  A wide tile
// (I, Jw) covers the two 128-blocks J = 2 Jw + h, h = 0, 1; a half is used iff J >= I and J < T
// (upper triangle; the half below the diagonal of an odd I is computed and dropped), mirrored
// iff J > I.  Slots as in k_tile_tc.  Used for the one-GPU implicit product and for predict.
struct TcW {
    static constexpr int BK = 16;                               // fp32 features per slab (64 B rows)
    static constexpr int STAGES = 4;
    static constexpr int TA = kTile * BK, TB = 2 * kTile * BK;  // floats per A / B operand tile
    static constexpr uint32_t STAGE_BYTES = (2 * TA + 2 * TB) * 4;  // 48 KiB
    static constexpr int THREADS = 192;
    static constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_BYTES + 1024 + 8192;
    static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
};

// K-major operand, 64-byte swizzle atoms (8 rows x 64 B): SBO = 512 B, layout type 4.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
    return (uint64_t((saddr >> 4) & 0x3FFFu)) | (uint64_t(512 >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(4) << 61);
}
__device__ __forceinline__ void umma_tf32_n256(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(TcW::IDESC), "r"(acc));
}

template <int KT, int MODE>
__global__ void __launch_bounds__(TcW::THREADS, 1)
    k_tile_tc_wide(const __grid_constant__ CUtensorMap tma_hi, const __grid_constant__ CUtensorMap tma_lo,
                   const __grid_constant__ CUtensorMap tmb_hi, const __grid_constant__ CUtensorMap tmb_lo, int64_t dpad,
                   const int2 *__restrict__ tiles, int tilesI, int T_tiles, const float *__restrict__ qa,
                   const float *__restrict__ na, const float *__restrict__ qb, const float *__restrict__ nb_,
                   const float *__restrict__ p, KParams<float> kp, float invC, const double *__restrict__ scal,
                   int64_t m1, float *__restrict__ Ypart, int64_t band_rows, const int *ctrl) {
    if (cg_done(ctrl)) return;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float *ring = reinterpret_cast<float *>(base);
    unsigned char *misc = base + size_t(TcW::STAGES) * TcW::STAGE_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(misc);
    uint64_t *empty = full + TcW::STAGES;
    uint64_t *accf = empty + TcW::STAGES;
    uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(accf + 1);
    float *colq = reinterpret_cast<float *>(misc + 128);  // [256]
    float *colp = colq + 2 * kTile;                       // [256] (alpha for predict)
    float *coln = colp + 2 * kTile;                       // [256]
    float *redc = coln + 2 * kTile;                       // [4][256]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int I, Jw;
    if constexpr (MODE == TC_PREDICT) {
        I = blockIdx.x % tilesI;
        Jw = blockIdx.x / tilesI;
    } else {
        const int2 tile = tiles[blockIdx.x];
        I = tile.x;
        Jw = tile.y;
    }
    const int row0 = I * kTile, col0 = Jw * 2 * kTile;
    const int nk = static_cast<int>(dpad / TcW::BK);

    if (warp == 4 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_hi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_lo)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb_hi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb_lo)) : "memory");
        for (int s = 0; s < TcW::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accf, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_addr(tmem_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int c = threadIdx.x; c < 2 * kTile; c += TcW::THREADS) {
        const int64_t gj = col0 + c;
        const bool in = gj < int64_t(T_tiles) * kTile;
        colq[c] = (MODE == TC_PREDICT || !in) ? 0.f : qb[gj];
        colp[c] = in ? p[gj] : 0.f;
        coln[c] = (KT == RBF && in) ? nb_[gj] : 0.f;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_sh;

    if (warp == 4) {
        if (lane == 0) {  // ---- TMA producer
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % TcW::STAGES;
                if (kb >= TcW::STAGES) mbar_wait(&empty[s], ((kb / TcW::STAGES) - 1) & 1);
                float *st = ring + size_t(s) * (2 * TcW::TA + 2 * TcW::TB);
                mbar_expect_tx(&full[s], TcW::STAGE_BYTES);
                const int x = kb * TcW::BK;
                tma_load_2d(st, &tma_hi, &full[s], x, row0);
                tma_load_2d(st + TcW::TA, &tma_lo, &full[s], x, row0);
                tma_load_2d(st + 2 * TcW::TA, &tmb_hi, &full[s], x, col0);
                tma_load_2d(st + 2 * TcW::TA + TcW::TB, &tmb_lo, &full[s], x, col0);
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {  // ---- MMA issuer: 2 K-steps x 3 products per slab
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % TcW::STAGES;
                mbar_wait(&full[s], (kb / TcW::STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t sa = smem_addr(ring + size_t(s) * (2 * TcW::TA + 2 * TcW::TB));
                const uint64_t dah = umma_desc_sw64(sa), dal = umma_desc_sw64(sa + TcW::TA * 4);
                const uint64_t dbh = umma_desc_sw64(sa + 2 * TcW::TA * 4);
                const uint64_t dbl = umma_desc_sw64(sa + (2 * TcW::TA + TcW::TB) * 4);
#pragma unroll
                for (int kk = 0; kk < TcW::BK / 8; ++kk) {
                    const uint64_t o = uint64_t(kk * 2);  // +32 B
                    umma_tf32_n256(tmem, dah + o, dbh + o, (kb > 0 || kk > 0) ? 1u : 0u);
                    umma_tf32_n256(tmem, dah + o, dbl + o, 1u);
                    umma_tf32_n256(tmem, dal + o, dbh + o, 1u);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(accf);
        }
    } else {  // ---- epilogue warps 0-3: thread = tile row 32w + lane, 256 columns (two halves)
        const int lr = warp * 32 + lane;
        const int64_t gi = row0 + lr;
        const float qi = (MODE == TC_PREDICT) ? 0.f : qa[gi];
        const float pi = (MODE == TC_MATVEC) ? p[gi] : 0.f;
        const float ni = (KT == RBF) ? na[gi] : 0.f;
        const float Qmm = (MODE == TC_PREDICT) ? 0.f : static_cast<float>(scal[S_QMM]);
        mbar_wait(accf, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int J = 2 * Jw + h;
            const bool use = (MODE == TC_PREDICT) ? (J < T_tiles) : (J >= I && J < T_tiles);  // warp-uniform
            if (!use) continue;
            const bool mirrored = (MODE == TC_MATVEC) && J > I;
            float rs = 0.f;
#pragma unroll 1
            for (int c0 = h * kTile; c0 < (h + 1) * kTile; c0 += 16) {
                float v[16];
                tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
                if constexpr (MODE == TC_PREDICT) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) rs = fmaf(colp[c0 + j], kernel_value<KT, float>(v[j], ni, coln[c0 + j], false, kp), rs);
                } else {
                    float cs[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int lc = c0 + j;
                        const float qt = qtilde_value<KT, float>(v[j], gi, int64_t(col0 + lc), ni, coln[lc], qi,
                                                                 colq[lc], Qmm, invC, m1, kp);
                        rs = fmaf(qt, colp[lc], rs);
                        cs[j] = qt * pi;
                    }
                    if (mirrored) {
                        const float t = transpose_reduce16(cs, lane);
                        if ((lane & 1) == 0) redc[warp * 2 * kTile + c0 + (lane >> 1)] = t;
                    }
                }
            }
            Ypart[int64_t(J) * band_rows + row0 + lr] = rs;
            if (mirrored) {
                asm volatile("bar.sync 1, 128;");
                const int t = threadIdx.x;
                const int c = h * kTile + t;
                Ypart[int64_t(I) * band_rows + int64_t(J) * kTile + t] =
                    (redc[c] + redc[2 * kTile + c]) + (redc[4 * kTile + c] + redc[6 * kTile + c]);
                asm volatile("bar.sync 1, 128;");  // redc is reused by the next half
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 5) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

}  // namespace plssvm
