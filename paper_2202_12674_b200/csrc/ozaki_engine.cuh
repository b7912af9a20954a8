// ozaki_engine.cuh -- fp64 pairwise contraction on the int8 tensor cores (tcgen05 kind::i8) by
// exact digit splitting (Ozaki scheme): the fp64-accurate S = X_I X_J^T of the implicit Q~p
// (Eq. 16), the cached-mode precompute and the predict (Eq. 10).
//
// Why: a B200 runs fp64 at 37 TFLOP/s (DMMA, profiles/r01_fp64_peak.txt) but int8 MMAs at
// ~4.5 POPS.  Each point x_i is written EXACTLY as
//     x_i = 2^{E_i} * sum_{a=1..S} D_a(x_i) 2^{-7a},   D_a in [-127, 127] (int8 digits),
// E_i = the row's exponent (max_k |x_ik| < 2^{E_i}); the remainder after S digits is < 2^{E_i-7S}.
// Then  x_i . x_j = 2^{E_i+E_j-14} * sum_{l=0..S-1} 2^{-7l} * acc_l,
//       acc_l = sum_{a+b=l} D_a(x_i) . D_b(x_j)       (0-based digit indices a, b)
// keeps every digit product of order <= S-1 (the dropped ones are < S 2^{-7S} relative to
// 2^{E_i+E_j} each: S = 8 gives 1e-16-level products, i.e. fp64 accuracy; SURVEY App. A style
// check in DESIGN.md).  Every acc_l is an EXACT int32 sum (|acc_l| <= S d 127^2 < 2^31 for
// d < 16384), accumulated in TMEM by tcgen05.mma.kind::i8; the combination runs in fp64
// (Horner over l, one rounding per level), so the result is an fp64 dot product with a
// different (shorter) rounding history, not a lower-precision one.
//
// Tile = 128 rows x 64 columns (UMMA M = 128, N = 64): S level accumulators of 64 int32 columns
// each fill the 512-column TMEM (S = 8).  Persistent CTAs (one per SM), warp-specialised:
//   warp 8 (one lane) : TMA producer -- per 32-feature slab ONE 3-D box per operand brings all S
//                       digit planes (32 B x 128 rows x S, SWIZZLE_32B): S x 6 KiB per stage
//   warp 9 (one lane) : TMEM owner + MMA issuer -- S(S+1)/2 UMMAs (K = 32) per slab into the
//                       level accumulators; tcgen05.commit frees the stage / signals the tile
//   warps 0-7         : epilogue -- warp w reads TMEM lanes 32(w%4).. (tile rows) and columns
//                       32(w/4).. of every level (tcgen05.ld 32x32b.x32), Horner-combines them
//                       in fp64, releases the accumulator (the MMA warp starts the next tile),
//                       then applies the kernel function / Eq. 16 corrections and reduces.
// Slot conventions are those of k_matvec_implicit (Engine<double>, TN = 64, NSUB = 2).
#pragma once
#include <cuda.h>

#include "tc_engine.cuh"

namespace plssvm {

enum OzMode : int { OZ_MATVEC = 0, OZ_PRECOMPUTE = 1, OZ_PREDICT = 2 };

template <int S>
struct Oz {
    static constexpr int BK = 32;                                  // int8 features per slab (32 B rows)
    static constexpr int TN = 64;                                  // tile columns (UMMA N)
    static constexpr int NSUB = kTile / TN;                        // = Engine<double>::NSUB
    static constexpr int STAGES = 4;
    static constexpr uint32_t A_PLANE = kTile * BK;                // 4 KiB per digit plane
    static constexpr uint32_t B_PLANE = TN * BK;                   // 2 KiB
    static constexpr uint32_t STAGE_BYTES = S * (A_PLANE + B_PLANE);
    static constexpr int EPI_WARPS = 8;
    static constexpr int THREADS = (EPI_WARPS + 2) * 32;
    static constexpr int PAIRS = S * (S + 1) / 2;
    static constexpr int TMEM_COLS = 512;
    static_assert(S * TN <= TMEM_COLS, "level accumulators must fit TMEM");
    // misc: barriers (256 B) + column data 4 x 64 doubles + row partials 2 x 128 + col partials 4 x 64
    static constexpr size_t MISC = 256 + (4 * TN + 2 * kTile + 4 * TN) * 8;
    static constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_BYTES + 1024 + MISC;
    // instruction descriptor: D s32 (2), A s8 (1), B s8 (1), K-major both, N = 64, M = 128
    static constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(TN >> 3) << 17) | ((128u >> 4) << 24);
};

// K-major operand in 32-byte swizzle atoms (8 rows x 32 B): LBO 1 (unused), SBO = 256 B, type 6.
__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t saddr) {
    return (uint64_t((saddr >> 4) & 0x3FFFu)) | (uint64_t(1) << 16) | (uint64_t(256 >> 4) << 32) | (uint64_t(1) << 46) |
           (uint64_t(6) << 61);
}
template <int S>
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(Oz<S>::IDESC), "r"(acc));
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}

// Sum of v[0..31] over the 32 lanes in 31 shuffles: afterwards lane l holds the total of
// element l.  Fixed order (deterministic).
__device__ __forceinline__ double transpose_reduce32(double (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// Exact digit split of the point-major padded fp64 array Xp[rows][dpad] into S int8 planes
// Dg[S][rows][dpad8] (dpad8 = multiple of 32, zero beyond dpad) and the row scales
// sc_i = 2^{E_i - 7}.  One warp per row; 4 features per lane per step (char4 stores).
template <int S>
__global__ void k_ozaki_split(const double *__restrict__ Xp, int64_t rows, int64_t dpad, int64_t dpad8,
                              int8_t *__restrict__ Dg, double *__restrict__ sc) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= rows) return;
    const double *x = Xp + i * dpad;
    double mx = 0.0;
    for (int64_t k = lane; k < dpad; k += 32) mx = fmax(mx, fabs(x[k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int E = 0;
    if (mx > 0.0) frexp(mx, &E);  // mx = f 2^E, f in [0.5, 1)  =>  |x_ik| < 2^E
    const double inv = ldexp(1.0, -E);
    if (lane == 0) sc[i] = ldexp(1.0, E - 7);
    const int64_t plane = rows * dpad8;
    for (int64_t k0 = 4 * lane; k0 < dpad8; k0 += 128) {
        double u[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) u[v] = (k0 + v < dpad) ? x[k0 + v] * inv : 0.0;  // |u| < 1, exact
#pragma unroll
        for (int a = 0; a < S; ++a) {
            char4 dg;
            signed char *dv = reinterpret_cast<signed char *>(&dg);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                u[v] *= 128.0;                    // exact (power of two)
                const double t = trunc(u[v]);     // |t| <= 127
                u[v] -= t;                        // exact
                dv[v] = static_cast<signed char>(t);
            }
            *reinterpret_cast<char4 *>(Dg + a * plane + i * dpad8 + k0) = dg;
        }
    }
}

// Persistent tile kernel.  Tiles: MATVEC / PRECOMPUTE take the (I, Jc) list of the DMMA engine
// (Jc = 64-column sub-block); PREDICT enumerates tile t -> (t % tilesI, t / tilesI).
//  OZ_MATVEC     : Q~ entries -> row sums Ypart[Jc] (rows of I), mirrored tiles also column sums
//                  Ypart[I * NSUB] (rows of Jc) -- exactly k_matvec_implicit's slots
//  OZ_PRECOMPUTE : Q~ entries -> cached tiled array Qc (packed: ordinal t / NSUB; else band rows,
//                  with the mirrored transposed copy) -- k_precompute's layout
//  OZ_PREDICT    : alpha_j k(z_i, x_j) -> Fpart[Jc][npad]
template <int KT, int S, int MODE>
__global__ void __launch_bounds__(Oz<S>::THREADS, 1)
    k_tile_ozaki(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, int nk,
                 const int2 *__restrict__ tiles, int ntiles, int tilesI, const double *__restrict__ sca,
                 const double *__restrict__ scb, const double *__restrict__ qv, const double *__restrict__ na,
                 const double *__restrict__ nb_, const double *__restrict__ p, KParams<double> kp, double invC,
                 const double *__restrict__ scal, int64_t m1, int band0, int band1, double *__restrict__ Ypart,
                 int64_t band_rows, double *__restrict__ Qc, int T_tiles, const int *ctrl) {
    using O = Oz<S>;
    if (cg_done(ctrl)) return;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *ring = base;
    unsigned char *misc = base + size_t(O::STAGES) * O::STAGE_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(misc);  // [STAGES]
    uint64_t *empty = full + O::STAGES;                   // [STAGES]
    uint64_t *tfull = empty + O::STAGES;                  // accumulators ready
    uint64_t *tempty = tfull + 1;                         // accumulators drained
    uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(tempty + 1);
    double *colsc = reinterpret_cast<double *>(misc + 256);  // [64]
    double *colq = colsc + O::TN;                            // [64]
    double *colp = colq + O::TN;                             // [64] (alpha for predict)
    double *coln = colp + O::TN;                             // [64]
    double *redr = coln + O::TN;                             // [2][128]
    double *redc = redr + 2 * kTile;                         // [4][64]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 8 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb)) : "memory");
        for (int s = 0; s < O::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, O::EPI_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 9) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_sh)),
                     "n"(O::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_sh;

    auto tile_of = [&](int t, int &I, int &Jc) {
        if constexpr (MODE == OZ_PREDICT) {
            I = t % tilesI;
            Jc = t / tilesI;
        } else {
            const int2 tl = tiles[t];
            I = tl.x;
            Jc = tl.y;
        }
    };

    if (warp == 8) {
        if (lane == 0) {  // ---- TMA producer: all S digit planes of a slab in one box per operand
            uint32_t g = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int I, Jc;
                tile_of(t, I, Jc);
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const uint32_t s = g % O::STAGES;
                    if (g >= O::STAGES) mbar_wait(&empty[s], ((g / O::STAGES) - 1) & 1);
                    unsigned char *st = ring + size_t(s) * O::STAGE_BYTES;
                    mbar_expect_tx(&full[s], O::STAGE_BYTES);
                    tma_load_3d(st, &tma, &full[s], kb * O::BK, I * kTile, 0);
                    tma_load_3d(st + S * O::A_PLANE, &tmb, &full[s], kb * O::BK, Jc * O::TN, 0);
                }
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {  // ---- MMA issuer: level l = a + b accumulates D_a(x_I) D_b(x_J)^T
            uint32_t g = 0;
            int n = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
                if (n > 0) {
                    mbar_wait(tempty, (n - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const uint32_t s = g % O::STAGES;
                    mbar_wait(&full[s], (g / O::STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = smem_addr(ring + size_t(s) * O::STAGE_BYTES);
                    const uint32_t sb = sa + S * O::A_PLANE;
#pragma unroll
                    for (int a = 0; a < S; ++a) {
                        const uint64_t da = umma_desc_sw32(sa + a * O::A_PLANE);
#pragma unroll
                        for (int b = 0; b < S - a; ++b) {
                            const uint64_t db = umma_desc_sw32(sb + b * O::B_PLANE);
                            umma_i8<S>(tmem + uint32_t((a + b) * O::TN), da, db, (kb > 0 || a > 0) ? 1u : 0u);
                        }
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(tfull);
            }
        }
    } else {  // ---- epilogue warps 0-7: row 32(w%4) + lane, columns 32(w/4) .. +31
        const int quarter = warp & 3, grp = warp >> 2;
        const int lr = quarter * 32 + lane;
        const int et = threadIdx.x;  // 0..255
        const double Qmm = (MODE == OZ_PREDICT) ? 0.0 : scal[S_QMM];
        int n = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
            int I, Jc;
            tile_of(t, I, Jc);
            const int64_t row0 = int64_t(I) * kTile, col0 = int64_t(Jc) * O::TN;
            const int J = Jc / O::NSUB;
            if (et < O::TN) {  // column data of this tile (the previous tile's readers are done: B3)
                const int64_t gj = col0 + et;
                colsc[et] = scb[gj];
                colq[et] = (MODE == OZ_PREDICT) ? 0.0 : qv[gj];
                colp[et] = (MODE == OZ_PRECOMPUTE) ? 0.0 : p[gj];
                coln[et] = (KT == RBF) ? nb_[gj] : 0.0;
            }
            const int64_t gi = row0 + lr;
            const double sci = sca[gi];
            const double qi = (MODE == OZ_PREDICT) ? 0.0 : qv[gi];
            const double pi = (MODE == OZ_MATVEC) ? p[gi] : 0.0;
            const double ni = (KT == RBF) ? na[gi] : 0.0;
            asm volatile("bar.sync 1, 256;" ::: "memory");  // B1

            // drain: Horner over the levels, highest first:  v = sum_l 2^{-7l} acc_l
            mbar_wait(tfull, n & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t tbase = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(grp * 32);
            double v[32];
            uint32_t r[32];
            tmem_ld32_issue(tbase + uint32_t((S - 1) * O::TN), r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = static_cast<double>(static_cast<int>(r[j]));
#pragma unroll 1
            for (int l = S - 2; l >= 0; --l) {
                tmem_ld32_issue(tbase + uint32_t(l * O::TN), r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = fma(v[j], 0.0078125, static_cast<double>(static_cast<int>(r[j])));
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);  // the MMA warp may overwrite the accumulators now

            double rs = 0.0;
            if constexpr (MODE == OZ_PREDICT) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int lc = grp * 32 + j;
                    const double sv = v[j] * (sci * colsc[lc]);
                    rs = fma(colp[lc], kernel_value<KT, double>(sv, ni, coln[lc], false, kp), rs);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int lc = grp * 32 + j;
                    const double sv = v[j] * (sci * colsc[lc]);
                    v[j] = qtilde_value<KT, double>(sv, gi, col0 + lc, ni, coln[lc], qi, colq[lc], Qmm, invC, m1, kp);
                }
            }
            if constexpr (MODE == OZ_MATVEC) {
                const bool mirrored = (I != J) && (J >= band0) && (J < band1);
#pragma unroll
                for (int j = 0; j < 32; ++j) rs = fma(v[j], colp[grp * 32 + j], rs);
                redr[grp * kTile + lr] = rs;
                if (mirrored) {  // tile-uniform
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] *= pi;
                    redc[quarter * O::TN + grp * 32 + lane] = transpose_reduce32(v, lane);
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");  // B2
                const int64_t lrow0 = row0 - int64_t(band0) * kTile;
                if (et < kTile) Ypart[int64_t(Jc) * band_rows + lrow0 + et] = redr[et] + redr[kTile + et];
                if (mirrored && et >= kTile && et < kTile + O::TN) {
                    const int c = et - kTile;
                    const int64_t lcol0 = col0 - int64_t(band0) * kTile;
                    Ypart[int64_t(I) * O::NSUB * band_rows + lcol0 + c] =
                        (redc[c] + redc[O::TN + c]) + (redc[2 * O::TN + c] + redc[3 * O::TN + c]);
                }
            } else if constexpr (MODE == OZ_PREDICT) {
                redr[grp * kTile + lr] = rs;
                asm volatile("bar.sync 1, 256;" ::: "memory");  // B2
                if (et < kTile) Ypart[int64_t(Jc) * band_rows + row0 + et] = redr[et] + redr[kTile + et];
            } else {  // OZ_PRECOMPUTE: row-major 128 x 128 tiles, this tile is the 64-column half h
                const int h = Jc % O::NSUB;
                double *dst;
                if (T_tiles < 0) dst = Qc + int64_t(t / O::NSUB) * (kTile * kTile) + h * O::TN;
                else dst = Qc + (int64_t(I - band0) * T_tiles + J) * (kTile * kTile) + h * O::TN;
                double *drow = dst + int64_t(lr) * kTile + grp * 32;
#pragma unroll
                for (int j = 0; j < 32; j += 2) *reinterpret_cast<double2 *>(drow + j) = make_double2(v[j], v[j + 1]);
                const bool mirrored = (I != J) && (J >= band0) && (J < band1);
                if (T_tiles >= 0 && mirrored) {  // transposed copy: column lc of this tile = row of tile (J, I)
                    double *mdst = Qc + (int64_t(J - band0) * T_tiles + I) * (kTile * kTile) + int64_t(h * O::TN) * kTile;
#pragma unroll
                    for (int j = 0; j < 32; ++j) mdst[int64_t(grp * 32 + j) * kTile + lr] = v[j];  // coalesced over lanes
                }
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");  // B3: smem partials / column data reusable
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 9) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(O::TMEM_COLS));
    }
}

}  // namespace plssvm
