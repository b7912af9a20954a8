// ozaki_engine.cuh -- fp64 pairwise contraction on the int8 tensor cores (tcgen05 kind::i8) by
// int8 digit splitting (Ozaki scheme): the fp64-accurate S = X_I X_J^T of the implicit Q~p
// (Eq. 16), the cached-mode precompute and the predict (Eq. 10).
//
// Why: a B200 runs fp64 at 37 TFLOP/s (DMMA, profiles/r01_fp64_peak.txt) but int8 MMAs at
// ~4.5 POPS.  Each point x_i is mapped to the integer vector N_i = rn(x_i 2^{54-E_i}) (E_i the
// row's exponent: 2^{E_i-1} <= ||x_i||_inf < 2^{E_i}), a FIXED-POINT representation relative to the
// row maximum: features with |x_ik| >= 2^{E_i-2} are exact, smaller ones are rounded to the grid
// 2^{E_i-54} (|error| <= 2^{E_i-55}).  N_i is written in 7 BALANCED base-256 digits,
//     N_i = sum_{a=0..6} D_a 256^{6-a},   D_a in [-128, 127]  (int8; |N| < 2^54 < the 7-digit range)
// so  x^_i . x^_j = 2^{E_i+E_j-12} * sum_{l=0..12} 2^{-8l} acc_l,   acc_l = sum_{a+b=l} D_a(x_i) . D_b(x_j).
// Levels l <= 6 are kept (28 digit pairs).  Every acc_l is an EXACT int32 sum (|acc_l| <= 7 d 2^14 <
// 2^31 for d <= 16384) accumulated in TMEM by tcgen05.mma.kind::i8; the kept levels are combined in
// exact int64 (V: levels 0-3, W: levels 4-6) and converted with ONE fp64 rounding.  Error of one
// inner product s = x_i.x_j (DESIGN.md §5 derives it):
//     |s~ - s| <= u |s| + 13.04 d u ||x_i||_inf ||x_j||_inf          (u = 2^-53)
// = input rounding (<= d u ||.||inf ||.||inf) + dropped levels 7..12 (<= 12.04 d u ||.||inf ||.||inf)
// + the final rounding.  Against the textbook fp64 dot-product bound in its Cauchy-Schwarz form,
// gamma_d ||x_i||_2 ||x_j||_2 ~ d u ||x_i||_2 ||x_j||_2, this is no larger whenever
// 13.04 rho_i rho_j <= d with rho = ||x||_inf / rms(x) -- AUTO's rule (driver.cu oz_choose).  It is
// NOT the componentwise bound d u sum_k |x_ik x_jk| an fp64 dot satisfies: inner products that are
// small against ||x_i||_inf ||x_j||_inf (orthogonal spikes) lose relative accuracy.
//
// Tile = 128 x 128 per CTA, computed by CTA pairs as 256 x 128 UMMAs (cta_group::2, below).
// The 7 level accumulators of a tile need 7 x 128 int32
// TMEM columns, more than the 512 available, so a tile runs in TWO PASSES over the features:
// pass 0 accumulates levels 0-3 (10 digit pairs, digit planes 0-3), pass 1 levels 4-6 (18
// pairs, planes 0-6), each in <= 4 x 128 TMEM columns.  N = 128 halves the shared-memory operand
// bytes per MMA cycle of an N = 64 tile (the SS-mode UMMA reads A and B from smem each time:
// 128 B/clk at N = 128 = the smem bandwidth, 192 B/clk at N = 64 -- measured: tc pipe 84 %
// busy, imma 46 % with 128 x 64 tiles), at the same L2 traffic per output element.
// Persistent CTA pairs (one CTA per SM), warp-specialised:
//   warp 0 (one lane) : TMA producer -- per pipeline stage (Oz::SLABS consecutive 32-feature slabs)
//                       the pass's pre-swizzled digit planes of the row block and the column half-block
//   warp 1 (one lane) : TMEM owner; in the leader CTA the MMA issuer -- per slab of the stage the pass's digit
//                       pairs (K = 32 UMMAs) into the level accumulators; tcgen05.commit frees the stage /
//                       signals the pass
//   warps 2-3         : idle (warpgroup 0 gives its registers to the epilogue: setmaxnreg 40 / 232)
//   warps 4-11        : epilogue -- warp w reads TMEM lanes 32(w%4).. (tile rows), columns
//                       64((w-4)/4).. of every level (tcgen05.ld 32x32b.x8), combines the levels
//                       in exact int64 (pass 0 -> V, held in registers; pass 1 -> W and the 64
//                       contractions 2^k V + 2^{k-24} W, each term converted exactly in one fp64
//                       operation (scaled_exact), one rounding in their sum),
//                       releases the accumulators after each pass, and only then runs
//                       the kernel function / Eq. 16 corrections and the row / column contributions
//                       -- overlapped with the next pair-tile's MMAs.
// Slot conventions: those of k_matvec_implicit with 128-wide column blocks (NSUB = 1).
#pragma once
#include <cuda.h>

#include "tc_engine.cuh"

namespace plssvm {

enum OzMode : int { OZ_MATVEC = 0, OZ_PRECOMPUTE = 1, OZ_PREDICT = 2 };

// Cycle accounting of k_tile_ozaki (experiment build only, -DPLSSVM_OZ_EXPERIMENTS; read back by
// tools/oz_profile.py through plssvm_exp_oz_profile): per CTA, clock64 cycles spent by
//   [0] the MMA thread waiting for the epilogue to drain the accumulators (tempty)
//   [1] the MMA thread waiting for TMA stages (full)        [2] the MMA thread's whole loop
//   [3] the TMA thread waiting for free stages (empty)
//   [4] epilogue warp 4 waiting for accumulators (tfull)    [5] its pass-0 drain   [6] its pass-1 drain
//   [7] its fp64 work after the release (kernel value, Eq. 16, row / column sums)
#ifdef PLSSVM_OZ_EXPERIMENTS
__device__ unsigned long long g_oz_prof[160][8];
#define OZ_PROF_T0(v) const long long v = clock64()
#define OZ_PROF_ADD(slot, v) atomicAdd(&g_oz_prof[blockIdx.x][slot], static_cast<unsigned long long>(clock64() - (v)))
#else
#define OZ_PROF_T0(v)
#define OZ_PROF_ADD(slot, v)
#endif

// S = 7 (fp64 engine): pass 0 = levels 0..3 (planes 0..3), pass 1 = levels 4..6 (all 7 planes).
// S = 3 (fp32 engine, plssvm.h PLSSVM_FP32_OZAKI): one pass, levels 0..2 (6 digit pairs, planes
// 0..2) -- x rounded to 22 bits below its row maximum, i.e. the fp32 products of the inputs to
// ~2^-22 relative to ||x_i||_inf ||x_j||_inf (the 3xTF32 split carries 21 + 21 bits).
template <int S>
struct Oz {
    static_assert(S == 7 || S == 3, "7 digits (fp64, two passes) or 3 digits (fp32, one pass)");
    static constexpr int NPASS = S == 7 ? 2 : 1;
    static constexpr int BITS = 8 * S - 2;                         // N_i = round(x_i 2^{BITS - E_i})
    static constexpr int SC_SHIFT = S == 7 ? 6 : 14;               // sc_i = 2^{E_i - SC_SHIFT}
    static constexpr int BK = 32;                                  // int8 features per slab (32 B rows)
    static constexpr int TN = 128;                                 // tile columns (UMMA N)
    static constexpr int NSUB = kTile / TN;                        // 1
    static constexpr int LV = S == 7 ? 4 : 3;                      // levels of the last pass (0..LV-1)
    static constexpr int LV0 = S == 7 ? S - LV : LV;               // levels of pass 0
// Pipeline stages: few and LARGE.  The MMA issuer and the TMA producer hand over once per stage (full /
// empty mbarriers, tcgen05.commit), so the number of 32-feature slabs per stage sets how many UMMAs run
// per handshake; A/B (profiles/r02_ab_slabs.txt): fp32 engine 1 slab x 8 stages -> 5 slabs x 2 stages
// (6 -> 30 UMMAs per stage): C3 product 5.81 -> 4.90 ms; fp64 engine 1 slab x 5 stages -> 2 slabs x 2
// stages (pass 1: 18 -> 36 UMMAs, pass 0: 10 -> 20): C1 3.00 -> 2.91 ms.  Two stages of 84 KiB (fp64)
// or 90 KiB (fp32) still cover the L2 -> shared latency: each stage is ~1.5-2.5k MMA cycles.
#ifndef PLSSVM_OZ_STAGES7
#define PLSSVM_OZ_STAGES7 2
#endif
#ifndef PLSSVM_OZ_SLABS7
#define PLSSVM_OZ_SLABS7 2  // fp64 pass 1 (all 7 planes): slabs per stage
#endif
#ifndef PLSSVM_OZ_SLABS7P0
#define PLSSVM_OZ_SLABS7P0 2  // fp64 pass 0 (4 planes): slabs per stage (3: no change)
#endif
#ifndef PLSSVM_OZ_SLABS3
#define PLSSVM_OZ_SLABS3 5  // fp32 engine (3 planes): slabs per stage (4: +1 %)
#endif
#ifndef PLSSVM_OZ_STAGES3
#define PLSSVM_OZ_STAGES3 2
#endif
    static constexpr int STAGES = S == 7 ? PLSSVM_OZ_STAGES7 : PLSSVM_OZ_STAGES3;  // (A/B builds may override)
    static constexpr uint32_t PLANE = kTile * BK;                  // 4 KiB: one A digit plane (B half: 2 KiB)
    // SLABS for the passes that load all S planes (one TMA box per BOXSL slabs: the S planes of consecutive
    // slabs are contiguous), SLABS_P0 for the fp64 engine's 4-plane pass 0 (one box per slab)
    static constexpr int SLABS = S == 7 ? PLSSVM_OZ_SLABS7 : PLSSVM_OZ_SLABS3;
    static constexpr int SLABS_P0 = S == 7 ? PLSSVM_OZ_SLABS7P0 : SLABS;
    // slabs one all-plane TMA box spans (a box dimension is at most 256 rows of 32 B per plane and slab)
    static constexpr int box_slabs(int n) {  // the largest divisor of SLABS whose box fits 256 rows
        return (SLABS % n == 0 && n * S * 32 <= 256) ? n : box_slabs(n - 1);
    }
    static constexpr int BOXSL = box_slabs(SLABS);
    static_assert(SLABS % BOXSL == 0, "the stage's slabs must split into whole boxes");
    static constexpr int LVP = S == 7 ? 4 : 3;  // planes of the fp64 engine's pass 0 (its LV)
    static constexpr uint32_t STAGE_BYTES =
        (SLABS * S > SLABS_P0 * LVP ? SLABS * S : SLABS_P0 * LVP) * (PLANE + PLANE / 2);  // A planes + B halves
#ifndef PLSSVM_OZ_EPI
#define PLSSVM_OZ_EPI 8
#endif
    static constexpr int EPI_WARPS = PLSSVM_OZ_EPI;                  // 8 or 16 epilogue warps
    static constexpr int EPI_THREADS = EPI_WARPS * 32;
    static constexpr int NG = EPI_WARPS / 4;                        // column groups per TMEM lane quarter
    static constexpr int CPT = TN / NG;                             // columns per epilogue thread (64 / 32)
    static constexpr int THREADS = (EPI_WARPS + 4) * 32;             // warpgroup 0: control, then the epilogue
    // setmaxnreg split: the epilogue's increase must come out of what warpgroup 0 releases from the launch
    // allocation (8 warps: 384 x 168 -> 4 x 40 + 8 x 232; 16 warps: 640 x 96 -> 4 x 24 + 16 x 112)
    static constexpr int CTRL_REGS = EPI_WARPS == 8 ? 40 : 24, EPI_REGS = EPI_WARPS == 8 ? 232 : 112;
    static_assert(EPI_WARPS == 8 || EPI_WARPS == 16, "8 or 16 epilogue warps");
    static constexpr int TMEM_COLS = 512;
    static_assert(LV * TN <= TMEM_COLS && LV0 * TN <= TMEM_COLS, "a pass's level accumulators must fit TMEM");
    // misc: barriers (256 B) + column data 4 x 128 doubles + row partials NG x 128 + col partials 4 x 128
    // + the 256-entry exp table + the tile's p / q.p sums (4 warps x 4)
    static constexpr size_t MISC = 256 + (4 * TN + NG * kTile + 4 * TN + 256 + 16) * 8;
    static constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_BYTES + 1024 + MISC;
    // instruction descriptor: D s32 (2), A s8 (1), B s8 (1), K-major both, N = 128, M = 256 (2 SMs)
    static constexpr uint32_t IDESC2 = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(TN >> 3) << 17) | ((256u >> 4) << 24);
};

// Digit planes a pass loads (S = 7: 7 then 4; S = 3: 3).
template <int S>
__host__ __device__ constexpr int oz_planes(int pass) { return (S == 7 && pass == 0) ? Oz<S>::LV : S; }

// K-major operand in 32-byte swizzle atoms (8 rows x 32 B): LBO 1 (unused), SBO = 256 B, type 6.
__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t saddr) {
    return (uint64_t((saddr >> 4) & 0x3FFFu)) | (uint64_t(1) << 16) | (uint64_t(256 >> 4) << 32) | (uint64_t(1) << 46) |
           (uint64_t(6) << 61);
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
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8_issue(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
// Wait with a suspend-time hint (A/B build option PLSSVM_OZ_SLEEP): the waiting thread may stay
// suspended up to the hint (ns) instead of the system-dependent limit before try_wait returns false.
__device__ __forceinline__ void mbar_wait_idle(uint64_t *b, uint32_t parity) {
#ifdef PLSSVM_OZ_SLEEP
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
        "r"(parity), "n"(PLSSVM_OZ_SLEEP));
#else
    mbar_wait(b, parity);
#endif
}

// 2^(j/256), j = 0..255, correctly rounded (tools/gen_exp_table.py: 60-digit Decimal, each value
// checked against its neighbours) -- the table of exp_tab256.
__constant__ double kExp2Tab256[256] = {
    1.0, 1.0027112750502025, 1.0054299011128027, 1.0081558981184175,
    1.0108892860517005, 1.0136300849514894, 1.016378314910953, 1.019133996077738,
    1.0218971486541166, 1.0246677928971357, 1.0274459491187637, 1.030231637686041,
    1.0330248790212284, 1.0358256936019572, 1.0386341019613787, 1.041450124688316,
    1.0442737824274138, 1.0471050958792898, 1.0499440858006872, 1.0527907730046264,
    1.0556451783605572, 1.0585073227945128, 1.061377227289262, 1.0642549128844645,
    1.0671404006768237, 1.0700337118202419, 1.0729348675259756, 1.075843889062791,
    1.0787607977571199, 1.0816856149932152, 1.0846183622133092, 1.0875590609177697,
    1.0905077326652577, 1.0934643990728858, 1.0964290818163769, 1.099401802630222,
    1.102382583307841, 1.1053714457017412, 1.1083684117236787, 1.1113735033448175,
    1.1143867425958924, 1.1174081515673693, 1.1204377524096067, 1.12347556733302,
    1.1265216186082418, 1.129575928566288, 1.1326385195987192, 1.1357094141578055,
    1.1387886347566916, 1.1418762039695616, 1.1449721444318042, 1.148076478840179,
    1.1511892299529827, 1.154310420590216, 1.1574400736337511, 1.1605782120274988,
    1.1637248587775775, 1.1668800369524817, 1.1700437696832502, 1.1732160801636373,
    1.1763969916502812, 1.1795865274628758, 1.182784710984341, 1.1859915656609938,
    1.189207115002721, 1.1924313825831512, 1.1956643920398273, 1.1989061670743806,
    1.202156731452703, 1.2054161090051239, 1.2086843236265816, 1.2119613992768012,
    1.215247359980469, 1.2185422298274085, 1.2218460329727576, 1.2251587936371455,
    1.22848053610687, 1.2318112847340759, 1.2351510639369334, 1.2384998981998165,
    1.241857812073484, 1.245224830175258, 1.2486009771892048, 1.2519862778663162,
    1.255380757024691, 1.2587844395497165, 1.2621973503942507, 1.2656195145788063,
    1.2690509571917332, 1.2724917033894028, 1.275941778396392, 1.2794012075056693,
    1.2828700160787783, 1.2863482295460256, 1.2898358734066657, 1.2933329732290895,
    1.2968395546510096, 1.3003556433796506, 1.3038812651919358, 1.3074164459346773,
    1.3109612115247644, 1.3145155879493546, 1.318079601266064, 1.3216532776031575,
    1.3252366431597413, 1.3288297242059544, 1.3324325470831615, 1.3360451382041458,
    1.339667524053303, 1.3432997311868353, 1.3469417862329458, 1.3505937158920345,
    1.3542555469368927, 1.3579273062129011, 1.3616090206382248, 1.365300717204012,
    1.3690024229745905, 1.3727141650876684, 1.3764359707545302, 1.380167867260238,
    1.383909881963832, 1.387662042298529, 1.3914243757719262, 1.3951969099662003,
    1.3989796725383112, 1.4027726912202048, 1.4065759938190154, 1.4103896082172707,
    1.4142135623730951, 1.4180478843204152, 1.4218926021691656, 1.4257477441054942,
    1.42961333839197, 1.433489413367789, 1.4373759974489824, 1.4412731191286257,
    1.4451808069770467, 1.449099089642035, 1.4530279958490526, 1.4569675544014438,
    1.460917794180647, 1.4648787441464057, 1.4688504333369818, 1.4728328908693675,
    1.4768261459394993, 1.4808302278224719, 1.4848451658727524, 1.488870989524397,
    1.4929077282912648, 1.4969554117672355, 1.5010140696264256, 1.5050837316234065,
    1.5091644275934228, 1.5132561874526098, 1.5173590411982147, 1.5214730189088146,
    1.5255981507445384, 1.529734466947287, 1.533881997840956, 1.5380407738316568,
    1.5422108254079407, 1.5463921831410214, 1.550584877685, 1.5547889397770887,
    1.559004400237837, 1.5632312899713576, 1.567469639965553, 1.5717194812923414,
    1.5759808451078865, 1.5802537626528246, 1.5845382652524937, 1.588834384317164,
    1.593142151342267, 1.597461597908627, 1.6017927556826934, 1.606135656416771,
    1.6104903319492543, 1.6148568142048607, 1.6192351351948637, 1.6236253270173289,
    1.6280274218573478, 1.632441451987275, 1.6368674497669644, 1.6413054476440063,
    1.645755478153965, 1.6502175739206177, 1.6546917676561943, 1.6591780921616162,
    1.6636765803267364, 1.6681872651305825, 1.6727101796415966, 1.6772453570178785,
    1.681792830507429, 1.6863526334483934, 1.6909247992693053, 1.6955093614893326,
    1.7001063537185235, 1.7047158096580513, 1.709337763100463, 1.713972247929926,
    1.718619298122478, 1.723278947746274, 1.7279512309618377, 1.732636182022311,
    1.7373338352737062, 1.7420442251551564, 1.746767386199169, 1.7515033530318782,
    1.7562521603732995, 1.761013843037584, 1.7657884359332727, 1.7705759740635547,
    1.7753764925265212, 1.7801900265154245, 1.785016611318935, 1.789856282321401,
    1.7947090750031072, 1.7995750249405351, 1.804454167806624, 1.809346539371032,
    1.8142521755003989, 1.8191711121586085, 1.8241033854070534, 1.8290490314048973,
    1.8340080864093424, 1.8389805867758937, 1.843966568958626, 1.8489660695104508,
    1.8539791250833855, 1.8590057724288205, 1.864046048397789, 1.8690999899412386,
    1.8741676341103, 1.8792490180565602, 1.8843441790323345, 1.8894531543909392,
    1.8945759815869656, 1.8997126981765553, 1.9048633418176741, 1.9100279502703899,
    1.9152065613971474, 1.9203992131630474, 1.925605943636125, 1.930826790987627,
    1.9360617934922943, 1.9413109895286405, 1.9465744175792332, 1.9518521162309783,
    1.9571441241754002, 1.9624504802089273, 1.9677712232331759, 1.9731063922552343,
    1.978456026387951, 1.9838201648502194, 1.9891988469672663, 1.9945921121709402,
};

// e^t for t <= 0 (the RBF kernel, t = -gamma ||x_i - x_j||^2) given in the scaled form
// tp = t 256/ln2 (the epilogue forms tp = 2 gamma (256/ln2) s + b_i + b_j directly from the inner
// product s and the per-point terms b = -gamma (256/ln2) ||x||^2: no separate distance, multiply
// or Cody-Waite reduction).  tp = n + r', n = 256 k + j, |r'| <= 1/2:
//     e^t = 2^k 2^(j/256) e^{r' L},  L = ln2/256,  e^{r' L} - 1 = r'(C1 + r'(C2 + r'(C3 + r' C4)))
// (C_k = L^k/k!; truncation |r'L|^5/120 < 4e-17).  n by the 1.5 * 2^52 rounding trick; r' = tp - n is
// exact.  ~1 ulp, 9 DP operations.  Precondition tp <= 0 (the caller's clamp); tp < -261000 (t < -706.8:
// e^t < 2e-307, where the exponent shift could leave the normal range) returns 0, tested on the high
// word (a non-positive double below -261000 has the larger unsigned high word; 0xC10FDC40 = -261000.0,
// whose low word is 0) -- an integer compare instead of a DP one.  tab = kExp2Tab256 in smem.
__device__ __forceinline__ double exp_tab256(double tp, const double *__restrict__ tab) {
    constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
    constexpr double C1 = 0.0027076061740622863, C2 = 3.6655655969101062e-06, C3 = 3.3083026805413713e-09,
                     C4 = 2.239395190875157e-12;
    const double kd = tp + kShift;
    const int n = __double2loint(kd);  // round(tp), two's complement
    const double r = tp - (kd - kShift);
    double c = fma(r, C4, C3);
    c = fma(r, c, C2);
    c = fma(r, c, C1);
    const double T = tab[n & 255];
    const double e = fma(T, r * c, T);  // 2^(j/256) e^{r' L}, in [0.997, 2)
    const double v = __hiloint2double(__double2hiint(e) + ((n >> 8) << 20), __double2loint(e));
    return static_cast<unsigned>(__double2hiint(tp)) > 0xC10FDC40u ? 0.0 : v;
}
constexpr double kExpScale256 = 369.3299304675746;  // 256 / ln 2

// Exact int32 -> fp64 without the (slow, XU-pipe) I2F.F64: 2^52 + (r + 2^31) assembled from
// bits, minus 2^52 + 2^31 -- one LOP3 + one DADD.
__device__ __forceinline__ double i2d_exact(uint32_t r) {
    return __hiloint2double(0x43300000, static_cast<int>(r ^ 0x80000000u)) - 4503601774854144.0;
}

// Exact int64 -> fp64 for |v| < 2^53: v = hi 2^32 + lo (lo unsigned), both halves by the bias
// trick, one fma (exact: the sum is representable).  3 DP ops.
__device__ __forceinline__ double i64_to_f64_exact(long long v) {
    const uint32_t hi = static_cast<uint32_t>(static_cast<unsigned long long>(v) >> 32);
    const uint32_t lo = static_cast<uint32_t>(v);
    return fma(i2d_exact(hi), 4294967296.0, __hiloint2double(0x43300000, static_cast<int>(lo)) - 4503599627370496.0);
}

// Level sums combined in INTEGER arithmetic (exact), one conversion per group instead of one per
// level: pass 0 V = acc_0 2^24 + acc_1 2^16 + acc_2 2^8 + acc_3, pass 1 W = acc_4 2^16 + acc_5 2^8 +
// acc_6.  |acc_l| <= (l+1) d 2^14, so |V| <= d 2^38.02 < 2^53 for d <= 16384 (the engine's limit) and
// |W| <= d 2^32.33 -- exactly representable, converted without rounding.
// c + a b for a 32-bit signed level sum a: the level combinations (IMAD.WIDE).  (Written in C++: an
// explicit mad.wide.s32 in PTX was lowered to IMAD.HI + IMAD pairs and made the C1 product 1.7 %
// slower in an A/B run, tools/scripts/ab2.sh.)
__device__ __forceinline__ long long mad_wide(uint32_t a, int b, long long c) {
    return c + static_cast<long long>(static_cast<int>(a)) * b;
}
// The scaled exact conversion 2^k V of an integer |V| < 2^51 in ONE fp64 operation (the digit
// scales are powers of two, so scaling is exact): u = V + 3 2^51 lies in [2^52, 2^53) and is the
// significand of the double 2^k u, whose bits are u + ((1074 + k) << 52); subtracting 2^k 3 2^51
// (exponent 1075 + k, mantissa 0.5) leaves 2^k V exactly.  ub = V + kOzBias (added in the integer
// combination), kb = (1074 + k) << 20 (the exponent term of the high word; 1 <= 1074 + k <= 2045).
// Replaces int64 -> fp64 (3 DP ops) + the scale multiply per group.
constexpr long long kOzBias = 3ll << 51;
__device__ __forceinline__ double scaled_exact(long long ub, int kb) {
    const uint32_t hi = static_cast<uint32_t>(static_cast<unsigned long long>(ub) >> 32) + static_cast<uint32_t>(kb);
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(static_cast<uint32_t>(ub))) -
           __hiloint2double(kb + 0x180000, 0);
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

// AUTO engine check: the largest row "peak" max_k |x_ik| / rms_k(x_ik) over the rows of a
// point-major padded fp64 array (zero rows skipped), as float bits in *peak_bits (atomicMax on
// the bits of a non-negative float orders like the value), and the largest |E_i| of the row
// maxima (2^{E_i-1} <= ||x_i||_inf < 2^{E_i}) in peak_bits[1]: the epilogue's one-operation
// conversions need the digit scales' exponents in range (kOzMaxExp).  The same pass is the input
// validation of the array (driver.cu validate_inputs): a non-finite element sets `bad` in flags[0].
// One warp per row.
template <typename TIN>
__global__ void k_row_peak(const TIN *__restrict__ Xp, int64_t rows, int64_t dpad, int64_t d,
                           unsigned *__restrict__ peak_bits, unsigned *__restrict__ flags, unsigned bad) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= rows) return;
    double mx = 0.0, ss = 0.0;
    bool fin = true;
    for (int64_t k = lane; k < d; k += 32) {
        const double v = static_cast<double>(Xp[i * dpad + k]);
        fin = fin && isfinite(v);
        mx = fmax(mx, fabs(v));
        ss = fma(v, v, ss);
    }
    if (!__all_sync(0xffffffffu, fin)) {
        if (lane == 0) atomicOr(flags, bad);
        return;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if (lane == 0 && mx > 0.0) {
        int E;
        frexp(mx, &E);
        atomicMax(peak_bits + 1, static_cast<unsigned>(E < 0 ? -E : E));
        if (ss > 0.0) {  // (underflowed squares: the exponent check above still applies)
            const float r = static_cast<float>(mx / sqrt(ss / static_cast<double>(d)));
            atomicMax(peak_bits, __float_as_uint(r));
        }
    }
}

// Digit split of the point-major array Xp[rows][dpad] (row stride dpad; rows a multiple of 128, rows
// m_valid .. rows - 1 are padding and read as 0 -- the caller's unpadded X can be split directly): each row is
// rounded to the fixed-point grid 2^{E_i - BITS} of its maximum (exact for |x| >= 2^{E_i-2} with S = 7)
// and written in S balanced base-256 int8 digit planes (plane 0 = most significant), stored
// PRE-SWIZZLED as the shared-memory images the UMMA reads:
//   DA[rows/128][nk][S][128 x 32 B]  (128-point blocks)
// (nk = dpad8 / 32 feature slabs), each 32-byte row in the SWIZZLE_32B pattern (16-byte chunk
// index XOR bit 2 of the row).  A stage of the tile kernel is then ONE contiguous block for the
// row operand, moved by TMA in 128-byte rows with no swizzle (4x fewer, 4x larger requests than
// a 32-byte-row box: the tile kernel was feed-bound with them), and for the column operand (one
// CTA's 64-point half of a 2-SM B tile) the half of every plane's image, [planes][64 x 32 B]: the
// swizzle depends on bit 2 of the row only, so a 64-row half of a 128-row image is itself a valid
// 64-row image.  One layout serves both roles (the digits are written, stored and L2-cached once).
// Row scales sc_i = 2^{E_i - SC_SHIFT} (S = 7: x_i . x_j = sc_i sc_j sum_l 2^{-8l} acc_l;
// S = 3: sc_i sc_j (acc_0 2^16 + acc_1 2^8 + acc_2)).  S = 7: N = rn(x 2^{54-E}), |N| < 2^54 (exact
// for the features within a factor 4 of the row maximum, rounded to 2^{E-54} below); S = 3 rounds the
// (fp32) value to N = rint(x 2^{22-E}), |N| <= 2^22, which three balanced digits hold.  One warp per
// row; 4 features per lane per step.
template <int S, typename TIN>
__global__ void k_ozaki_split(const TIN *__restrict__ Xp, int64_t rows, int64_t m_valid, int64_t dpad, int64_t dpad8,
                              int8_t *__restrict__ DA, double *__restrict__ sc) {
    static_assert(8 * S >= Oz<S>::BITS + 1, "S balanced base-256 digits must hold the split integer");
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= rows) return;
    const TIN *x = Xp + i * dpad;
    const bool real = i < m_valid;  // rows m_valid .. rows - 1: padding, all digits 0
    double mx = 0.0;
    if (real)
        for (int64_t k = lane; k < dpad; k += 32) mx = fmax(mx, fabs(static_cast<double>(x[k])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int E = 0;
    if (mx > 0.0) frexp(mx, &E);  // mx = f 2^E, f in [0.5, 1)  =>  |x_ik| < 2^E
    if (lane == 0) sc[i] = ldexp(1.0, E - Oz<S>::SC_SHIFT);
    const int64_t nk = dpad8 / 32;
    const int r128 = static_cast<int>(i & 127);
    const int flip = (r128 >> 2) & 1;
    for (int64_t k0 = 4 * lane; k0 < dpad8; k0 += 128) {
        long long N[4];
#pragma unroll
        for (int v = 0; v < 4; ++v)  // |N| < 2^{BITS}; exact when x's ulp >= 2^{E-BITS}, else rounded to nearest
            N[v] = (real && k0 + v < dpad) ? __double2ll_rn(ldexp(static_cast<double>(x[k0 + v]), Oz<S>::BITS - E)) : 0ll;
        const int64_t kb = k0 >> 5;
        const int c = static_cast<int>(k0 & 31);
        const int inrow = ((((c >> 4) ^ flip) << 4) | (c & 15));
        int8_t *pa = DA + ((i >> 7) * nk + kb) * (S * 4096) + r128 * 32 + inrow;
#pragma unroll
        for (int a = S - 1; a >= 0; --a) {  // least significant digit first
            char4 dg;
            signed char *dv = reinterpret_cast<signed char *>(&dg);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const signed char dd = static_cast<signed char>(N[v] & 0xFF);  // N = dd (mod 256), dd in [-128, 127]
                N[v] = (N[v] - dd) >> 8;                                       // exact
                dv[v] = dd;
            }
            *reinterpret_cast<char4 *>(pa + a * 4096) = dg;
        }
    }
}

__device__ __forceinline__ void tma_load_2d_2sm(void *dst, const CUtensorMap *map, uint32_t bar_cluster, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y)
        : "memory");
}

// ---- cluster helpers (CTA pair of a cta_group::2 MMA) ----------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA of this CTA's half of a 2-SM operand; completion bytes go to the leader CTA's barrier.
__device__ __forceinline__ void tma_load_3d_2sm(void *dst, const CUtensorMap *map, uint32_t bar_cluster, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y), "r"(z)
        : "memory");
}
template <int S>
__device__ __forceinline__ void umma_i8_2sm(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(Oz<S>::IDESC2), "r"(acc));
}
__device__ __forceinline__ void umma_commit_2sm_mc(uint64_t *bar) {  // arrive on bar in both CTAs of the pair
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_addr(bar)),
        "h"(uint16_t(3))
        : "memory");
}

// Persistent 2-SM tile kernel (cluster of 2 CTAs, tcgen05 cta_group::2).  A CTA pair owns the
// 256 x 128 pair-tile (row blocks I0, I1) x (column block J): CTA rank r stages the digit
// planes of its row block I_r (A, 128 rows) and of HALF the column block (B, rows
// J*128 + 64 r .. +63); the leader's single MMA thread issues M = 256, N = 128 UMMAs that read A
// and B from both CTAs' shared memory and accumulate each CTA's 128 rows in its own TMEM.  Per SM
// the MMA reads 6 KiB of operands per 64-cycle UMMA instead of 8 (A 4 KiB + half of B), and the
// pair loads each B plane once -- the 1-SM kernel was bound by shared-memory bandwidth
// (operand reads + TMA writes ~1.3x the 128 B/clk an SM has).
// Pair-tiles: MATVEC / PRECOMPUTE take a list of int4 (I0, I1, J, use): CTA rank r computes the
// tile (I_r, J); use bit r = that tile is one of this rank's (others are computed and dropped).  The
// two row blocks need not be adjacent: a tile (I, J) with I > J is the mirror of the stored (J, I)
// and the MATVEC epilogue's row and column sums treat both orientations alike (driver.cu
// oz_pair_tiles_matvec uses that to pair every tile of the triangle, no dropped half);
// PREDICT enumerates t -> (2 (t % pairsI) + r, t / pairsI).
//  OZ_MATVEC     : Q~ entries -> row sums Ypart[J] (rows of I), mirrored tiles also column sums
//                  Ypart[I] (rows of J) -- k_matvec_implicit's slots with 128-wide blocks
//  OZ_PRECOMPUTE : Q~ entries -> cached tiled array Qc (packed: ordinal pk[2 t + r]; else band
//                  rows, with the mirrored transposed copy) -- k_precompute's layout
//  OZ_PREDICT    : alpha_j k(z_i, x_j) -> Fpart[J][npad]
// ta4/ta8: maps over the pre-swizzled row-operand digits DA (boxes of 4 / 8 planes of a 128-point
// slab block, 128-byte rows); tb4/tb8: 3-D maps over the SAME digits selecting one 64-point half of a
// block (driver.cu make_tmap_digit_halves).
// T: the value type of the epilogue and of q, norms, p, the products and Q~ (double with S = 7,
// float with S = 3); the digit scales are fp64 either way.
template <int KT, int S, int MODE, typename T>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Oz<S>::THREADS, 1)
    k_tile_ozaki(const __grid_constant__ CUtensorMap ta4, const __grid_constant__ CUtensorMap ta8,
                 const __grid_constant__ CUtensorMap tb4, const __grid_constant__ CUtensorMap tb8, int nk,
                 const int4 *__restrict__ tiles, const int *__restrict__ pk, int ntiles, int rowsI,
                 const double *__restrict__ sca, const double *__restrict__ scb, const T *__restrict__ qv,
                 const T *__restrict__ na, const T *__restrict__ nb_, const T *__restrict__ p, KParams<T> kp, T invC,
                 const double *__restrict__ scal, int64_t m1, int band0, int band1, T *__restrict__ Ypart,
                 int64_t band_rows, T *__restrict__ Qc, int T_tiles, const int *ctrl, int dbg) {
    static_assert((S == 7) == std::is_same<T, double>::value, "S = 7 computes fp64, S = 3 fp32");
    using O = Oz<S>;
    constexpr int TN = O::TN, LV = O::LV;
    if (cg_done(ctrl)) return;  // uniform across the cluster
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // (The integer round trip makes the epilogue's smem pointers generic: its column data, table and
    // partials are read with generic LD.  Deriving them from smem_raw by pointer arithmetic turns them into
    // LDS, which made predict 5 % and the C2 product 2 % SLOWER in an A/B run (profiles/r02_ab_epilogue_lean.txt).)
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *ring = base;
    unsigned char *misc = base + size_t(O::STAGES) * O::STAGE_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(misc);  // [STAGES] (leader's are used)
    uint64_t *empty = full + O::STAGES;                   // [STAGES] (each CTA's own)
    uint64_t *tfull = empty + O::STAGES;                  // a pass's accumulators ready (each CTA)
    uint64_t *tempty = tfull + 1;                         // a pass's accumulators drained (leader: 16 warps)
    uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(tempty + 1);
    double *colsc = reinterpret_cast<double *>(misc + 256);  // [128] 8-byte slots: colk, the column exponent terms
    int *colk = reinterpret_cast<int *>(colsc);              // [128] e_j << 20 (scaled_exact)
    T *colq = reinterpret_cast<T *>(colsc + TN);             // [128] (8-byte slots for either T)
    T *colp = reinterpret_cast<T *>(colsc + 2 * TN);         // [128] (alpha for predict)
    T *coln = reinterpret_cast<T *>(colsc + 3 * TN);         // [128]
    T *redr = reinterpret_cast<T *>(colsc + 4 * TN);         // [NG][128]
    T *redc = reinterpret_cast<T *>(colsc + 4 * TN + O::NG * kTile);  // [4][128]
    double *etab = colsc + 8 * TN + O::NG * kTile;           // [256] 2^(j/256) (fp64 RBF, exp_tab256)
    T *psum = reinterpret_cast<T *>(etab + 256);             // [4][4] MATVEC: per warp sum p_j, q_j p_j, p_i, q_i p_i

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta4)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta8)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb4)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb8)) : "memory");
        for (int s = 0; s < O::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 2 * O::EPI_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_sh)),
                     "n"(O::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_sh;
    const uint32_t full0 = mapa_shared(smem_addr(full), 0);     // leader's full[0] (cluster window)
    const uint32_t tempty0 = mapa_shared(smem_addr(tempty), 0);  // leader's tempty

    // pair-tile t -> this CTA's row block, the column block, use bits
    auto tile_of = [&](int t, int &I, int &J, int &use) {
        if constexpr (MODE == OZ_PREDICT) {
            const int pairsI = (rowsI + 1) / 2;
            const int I0 = 2 * (t % pairsI);
            I = I0 + int(rank);
            J = t / pairsI;
            use = (I0 + 1 < rowsI) ? 3 : 1;
        } else {
            const int4 tl = tiles[t];
            I = rank ? tl.y : tl.x;
            J = tl.z;
            use = tl.w;
        }
    };

    // Register split by warpgroup: the control warps need few, the epilogue keeps a pass's 64
    // fp64 contractions in registers (so the accumulators are released before the fp64 work).
    // (each role branch starts with its setmaxnreg, so the allocator sees the new budget)
    if (warp == 0) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(O::CTRL_REGS));
        if (lane == 0) {  // ---- TMA producer (both CTAs): this CTA's A block and B half
            uint32_t g = 0;
            for (int t = pair; t < ntiles; t += npairs) {
                int I, J, use;
                tile_of(t, I, J, use);
#pragma unroll 1
                for (int pass = 0; pass < O::NPASS; ++pass) {
                    const int np = oz_planes<S>(pass);
                    const int sl = (np == S) ? O::SLABS : O::SLABS_P0;  // slabs per stage in this pass
                    for (int kb = 0; kb < nk; kb += sl, ++g) {
                        const uint32_t s = g % O::STAGES;
                        if (g >= O::STAGES) {
                            OZ_PROF_T0(t0);
                            mbar_wait_idle(&empty[s], ((g / O::STAGES) - 1) & 1);
                            OZ_PROF_ADD(3, t0);
                        }
                        unsigned char *st = ring + size_t(s) * O::STAGE_BYTES;
                        if (dbg & 2) {  // experiment: no data movement
                            if (leader) mbar_arrive(&full[s]);
                            continue;
                        }
                        // both CTAs' bytes: the boxes of the stage's slabs that exist (all-plane boxes span BOXSL
                        // slabs; a box reaching past the block's last slab reads the next block's digits, which no
                        // MMA uses)
                        const int rem = sl < nk - kb ? sl : nk - kb;
                        const int nsl = (np == S) ? (rem + O::BOXSL - 1) / O::BOXSL * O::BOXSL : rem;
                        if (leader) mbar_expect_tx(&full[s], 2u * nsl * np * (O::PLANE + O::PLANE / 2));
                        const uint32_t fb = full0 + s * 8;
                        // pre-swizzled blocks: A (row block I_r, slab kb) = np x 4 KiB at 128-B row
                        // (I * nk + kb) * S * 32; B = half r of block J: rows 16 r .. 16 r + 15 of the
                        // planes (J * nk + kb) * S + a, a < np
                        if (np == S) {  // all planes: boxes spanning BOXSL consecutive slabs each
#pragma unroll
                            for (int h = 0; h < nsl; h += O::BOXSL) {
                                tma_load_2d_2sm(st + h * np * O::PLANE, &ta8, fb, 0, (I * nk + kb + h) * (S * 32));
                                tma_load_3d_2sm(st + sl * np * O::PLANE + h * np * (O::PLANE / 2), &tb8, fb, 0,
                                                16 * int(rank), (J * nk + kb + h) * S);
                            }
                        } else {
                            for (int h = 0; h < nsl; ++h) {  // the first np planes of each slab
                                tma_load_2d_2sm(st + h * np * O::PLANE, &ta4, fb, 0, (I * nk + kb + h) * (S * 32));
                                tma_load_3d_2sm(st + sl * np * O::PLANE + h * np * (O::PLANE / 2), &tb4, fb, 0,
                                                16 * int(rank), (J * nk + kb + h) * S);
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(O::CTRL_REGS));
        if (leader && lane == 0) {  // ---- MMA issuer (leader only): level l = a + b
            uint32_t g = 0, e = 0;  // e: accumulator events (two per pair-tile)
            OZ_PROF_T0(tloop);
            for (int t = pair; t < ntiles; t += npairs) {
#pragma unroll 1
                for (int pass = 0; pass < O::NPASS; ++pass, ++e) {
                    if (e > 0) {  // both CTAs' epilogues have drained the previous pass
                        OZ_PROF_T0(t0);
                        mbar_wait(tempty, (e - 1) & 1);
                        OZ_PROF_ADD(0, t0);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                    }
                    const int np = oz_planes<S>(pass);
                    const int sl = (np == S) ? O::SLABS : O::SLABS_P0;
                    for (int kb0 = 0; kb0 < nk; kb0 += sl, ++g) {
                        const uint32_t s = g % O::STAGES;
                        {
                            OZ_PROF_T0(t0);
                            mbar_wait(&full[s], (g / O::STAGES) & 1);
                            OZ_PROF_ADD(1, t0);
                        }
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        const uint32_t sa0 = smem_addr(ring + size_t(s) * O::STAGE_BYTES);
                        const uint32_t sb0 = sa0 + sl * np * O::PLANE;
                        constexpr int kMaxSl = O::SLABS > O::SLABS_P0 ? O::SLABS : O::SLABS_P0;
#pragma unroll
                        for (int h = 0; h < kMaxSl; ++h) {
                        const int kb = kb0 + h;
                        if (kMaxSl > 1 && (h >= sl || kb >= nk)) break;
                        const uint32_t sa = sa0 + h * np * O::PLANE, sb = sb0 + h * np * (O::PLANE / 2);
                        if (dbg & 4) {  // experiment: data movement only
                        } else if (S == 7 && pass == 1) {  // levels 4..6 (18 pairs), TMEM column block l - 4
#pragma unroll
                            for (int a = 0; a < S; ++a)
#pragma unroll
                                for (int b = 0; b < S; ++b) {
                                    const int l = a + b;
                                    if (l < LV || l >= S) continue;  // compile-time after unrolling
                                    // the first MMA into level l (at kb = 0) is the one with a = 0
                                    umma_i8_2sm<S>(tmem + uint32_t((l - LV) * TN), umma_desc_sw32(sa + a * O::PLANE),
                                                   umma_desc_sw32(sb + b * (O::PLANE / 2)), (kb > 0 || a > 0) ? 1u : 0u);
                                }
                        } else {  // levels 0..LV-1 (S = 7: 10 pairs; S = 3: 6 pairs)
#pragma unroll
                            for (int a = 0; a < LV; ++a)
#pragma unroll
                                for (int b = 0; a + b < LV; ++b)
                                    umma_i8_2sm<S>(tmem + uint32_t((a + b) * TN), umma_desc_sw32(sa + a * O::PLANE),
                                                   umma_desc_sw32(sb + b * (O::PLANE / 2)), (kb > 0 || a > 0) ? 1u : 0u);
                        }
                        }  // slabs of the stage
                        umma_commit_2sm_mc(&empty[s]);  // frees stage s in both CTAs
                    }
                    umma_commit_2sm_mc(tfull);  // this pass's accumulators ready in both CTAs
                }
            }
            OZ_PROF_ADD(2, tloop);
        }
    } else if (warp < 4) {  // idle warps 2-3
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(O::CTRL_REGS));
    } else {  // ---- epilogue warps 4.. (both CTAs): row 32(w%4) + lane, columns CPT((w-4)/4) .. + CPT - 1
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(O::EPI_REGS));
        constexpr bool kTabExp = KT == RBF && S == 7;
        constexpr int CPT = O::CPT, NG = O::NG;
        if (kTabExp && threadIdx.x - 128 < 256) etab[threadIdx.x - 128] = kExp2Tab256[threadIdx.x - 128];  // read after B1
        // fp64 RBF: tp = a2 s + b_i + b_j = (256/ln2) (-gamma) (n_i + n_j - 2 s) (exp_tab256)
        const double gK = kTabExp ? -static_cast<double>(kp.gamma) * kExpScale256 : 0.0, a2 = -2.0 * gK;
        const int quarter = warp & 3, grp = (warp - 4) >> 2;
        const int lr = quarter * 32 + lane;
        const int et = threadIdx.x - 128;  // 0 .. EPI_THREADS - 1
        const T Qmm = (MODE == OZ_PREDICT) ? T(0) : static_cast<T>(scal[S_QMM]);
        uint32_t e = 0;
        for (int t = pair; t < ntiles; t += npairs) {
            int I, J, use;
            tile_of(t, I, J, use);
            const bool used = (use >> rank) & 1;  // CTA-uniform
            const int64_t row0 = int64_t(I) * kTile, col0 = int64_t(J) * TN;
            if (et < TN) {  // column data of this tile (the previous tile's readers are done: B3)
                const int64_t gj = col0 + et;
                colk[et] = ((__double2hiint(scb[gj]) >> 20) - 1023) << 20;  // scb = 2^{e_j}
                colq[et] = (MODE == OZ_PREDICT) ? T(0) : qv[gj];
                colp[et] = (MODE == OZ_PRECOMPUTE) ? T(0) : p[gj];
                coln[et] = (KT == RBF) ? (kTabExp ? T(gK * nb_[gj]) : nb_[gj]) : T(0);  // fp64 RBF: b_j
            }
            const int64_t gi = row0 + lr;
            // row exponent term of the scaled conversions (sca = 2^{e_i}): kb = rkb + colk[j] = (1074 + k) << 20
            // with k = e_i + e_j - 24 (S = 7: the unit of V, level 3) or e_i + e_j (S = 3)
            const int rkb = (1074 - (S == 7 ? 24 : 0) + (used ? (__double2hiint(sca[gi]) >> 20) - 1023 : 0)) << 20;
            // |V| < 2^51 (the one-operation conversion) needs d8 <= 8096; wider points convert V in pass 0
            const bool bigd = S == 7 && nk * Oz<S>::BK > 8096;
            const T qi = (MODE == OZ_PREDICT || !used) ? T(0) : qv[gi];
            const T pi = (MODE == OZ_MATVEC && used) ? p[gi] : T(0);
            const T ni = (KT == RBF && used) ? (kTabExp ? T(gK * na[gi]) : na[gi]) : T(0);  // fp64 RBF: b_i
            const T cqi = Qmm - qi;  // Eq. 16 row constant
            // this thread's diagonal entry (gi == gj: a diagonal tile, column lr): local column index
            // jd in 0 .. CPT - 1, else -1 -- one compare with a constant per entry
            const int jd = (MODE != OZ_PREDICT && I == J && lr >= grp * CPT && lr < grp * CPT + CPT) ? lr - grp * CPT : -1;
            if constexpr (MODE == OZ_MATVEC) {
                // Eq. 16 by rows: sum_j Q~_ij p_j = sum_j k_ij p_j + (Q_mm - q_i) sum_j p_j - sum_j q_j p_j
                // (+ p_i / C on the diagonal), likewise for the mirrored column sums -- the entries
                // need only the kernel value; the per-tile sums come from warps 4-7 (et = lr there)
                if (et < TN) {
                    const T pj = p[col0 + et];
                    T v[4] = {pj, qv[col0 + et] * pj, pi, qi * pi};
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                        for (int u = 0; u < 4; ++u) v[u] += __shfl_xor_sync(0xffffffffu, v[u], o);
                    if (lane == 0)
#pragma unroll
                        for (int u = 0; u < 4; ++u) psum[(et >> 5) * 4 + u] = v[u];
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(O::EPI_THREADS) : "memory");  // B1

            // S = 7, pass 0 (levels 0-3): V = 2^24 sum_{l<4} 2^{-8l} acc_l, an exact int64 (|V| < d 2^38 <
            // 2^53) held EXACTLY as fp64 in sv (64 columns in registers), accumulators released.  Pass 1
            // (levels 4-6): W = 2^16 sum_{l<3} 2^{-8l} acc_{4+l}, exact int64 -> exact fp64, and the
            // contraction is ONE fp64 rounding of the kept digit products: sv = (V + 2^-24 W) sc_i sc_j
            // (DESIGN.md §5 error bound).  Then the accumulators are released and the Q~ entry / kernel
            // value and its row and column contributions run under the next pair-tile's MMAs.
            // S = 3: the single pass, V = acc_0 2^16 + acc_1 2^8 + acc_2.
            const uint32_t tbase = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(grp * CPT);
            const bool mirrored = used && (MODE != OZ_PREDICT) && (I != J) && (J >= band0) && (J < band1);
            T rs = T(0);
            T *qdst = nullptr, *qmir = nullptr;
            if constexpr (MODE == OZ_PRECOMPUTE) {
                if (used) {
                    qdst = ((T_tiles < 0) ? Qc + int64_t(pk[2 * t + int(rank)]) * (kTile * kTile)
                                          : Qc + (int64_t(I - band0) * T_tiles + J) * (kTile * kTile)) +
                           int64_t(lr) * kTile + grp * CPT;
                    if (T_tiles >= 0 && mirrored) qmir = Qc + (int64_t(J - band0) * T_tiles + I) * (kTile * kTile) + lr;
                }
            }
            // the thread's 64 entries, one 64-bit register pair each: S = 7 the pass-0 V + 3 2^51, then the
            // fp64 contractions' bits; S = 3 V + 3 2^51, then the fp32 contractions' bits (one array for
            // both stages keeps the epilogue within the kernel's register budget)
            long long sv[CPT];
            auto sval = [&](int k) -> T {
                if constexpr (S == 7) return __longlong_as_double(sv[k]);
                else return __int_as_float(static_cast<int>(sv[k]));
            };
            const bool prof = warp == 4 && lane == 0;
            (void)prof;
            if constexpr (S == 7) {
                {
                    OZ_PROF_T0(t0);
                    mbar_wait_idle(tfull, e & 1);
                    if (prof) OZ_PROF_ADD(4, t0);
                }
                OZ_PROF_T0(tdr0);
                asm volatile("tcgen05.fence::after_thread_sync;");
                ++e;
                // Levels 0-2 first: pass 1 accumulates levels 4-6 into TMEM columns 0 .. 3 TN - 1 only, so
                // the MMA may start pass 1 as soon as those are read; level 3 (columns 3 TN ..) is read
                // after the release, under pass 1's MMAs -- the critical drain reads 3 levels, not 4.
                if (!(dbg & 1)) {
#pragma unroll
                    for (int c = 0; c < CPT / 8; ++c) {
                        uint32_t r0[8], r1[8], r2[8];
                        tmem_ld8_issue(tbase + uint32_t(2 * TN + c * 8), r2);
                        tmem_ld8_issue(tbase + uint32_t(1 * TN + c * 8), r1);
                        tmem_ld8_issue(tbase + uint32_t(c * 8), r0);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 8; ++j)  // V + 3 2^51 without level 3, exact in int64
                            sv[c * 8 + j] = mad_wide(r0[j], 1 << 24, mad_wide(r1[j], 1 << 16, mad_wide(r2[j], 1 << 8, kOzBias)));
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty0);  // the MMA may start pass 1
                if (prof) OZ_PROF_ADD(5, tdr0);
                if (!(dbg & 1)) {
#pragma unroll
                    for (int c = 0; c < CPT / 8; ++c) {
                        uint32_t r3[8];
                        tmem_ld8_issue(tbase + uint32_t(3 * TN + c * 8), r3);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            // V + 3 2^51, exact in int64; held as bits until pass 1 knows the scale
                            const long long Vb = mad_wide(r3[j], 1, sv[c * 8 + j]);
                            sv[c * 8 + j] = bigd ? __double_as_longlong(i64_to_f64_exact(Vb - kOzBias)) : Vb;
                        }
                    }
                }
            }
            {
                OZ_PROF_T0(t0);
                mbar_wait_idle(tfull, e & 1);
                if (prof) OZ_PROF_ADD(4, t0);
            }
            OZ_PROF_T0(tdr1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            ++e;
            if constexpr (S == 3) {
                // fp32 engine (one pass, no second TMEM buffer): the drain only combines the levels
                // (V + 3 2^51, exact int64), the accumulators are released, and the conversions run
                // under the next pair-tile's MMAs (the MMA waited ~8 % of its loop for drains, C3)
                if (!(dbg & 1)) {
#pragma unroll
                    for (int c = 0; c < CPT / 8; ++c) {
                        uint32_t r0[8], r1[8], r2[8];
                        tmem_ld8_issue(tbase + uint32_t(2 * TN + c * 8), r2);
                        tmem_ld8_issue(tbase + uint32_t(1 * TN + c * 8), r1);
                        tmem_ld8_issue(tbase + uint32_t(c * 8), r0);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 8; ++j)  // S = 3: x_i.x_j = 2^k V, |V| < d 2^30.01 < 2^51
                            sv[c * 8 + j] = mad_wide(r0[j], 1 << 16, mad_wide(r1[j], 1 << 8, mad_wide(r2[j], 1, kOzBias)));
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty0);  // the next pair-tile's MMAs may start
                if (!(dbg & 1)) {
#pragma unroll
                    for (int k = 0; k < CPT; ++k)  // then one rounding to fp32
                        sv[k] = static_cast<uint32_t>(__float_as_int(static_cast<float>(scaled_exact(sv[k], rkb + colk[grp * CPT + k]))));
                }
            } else {
                if (!(dbg & 1)) {
#pragma unroll
                    for (int c = 0; c < CPT / 8; ++c) {
                        uint32_t r0[8], r1[8], r2[8];
                        tmem_ld8_issue(tbase + uint32_t(2 * TN + c * 8), r2);
                        tmem_ld8_issue(tbase + uint32_t(1 * TN + c * 8), r1);
                        tmem_ld8_issue(tbase + uint32_t(c * 8), r0);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int kb = rkb + colk[grp * CPT + c * 8 + j];
                            // x_i.x_j = 2^k V + 2^{k-24} W (level 4 is 2^-32 below level 0, W carries 2^16
                            // of it), both terms exact: ONE rounding in their sum
                            const long long Wb = mad_wide(r0[j], 1 << 16, mad_wide(r1[j], 1 << 8, mad_wide(r2[j], 1, kOzBias)));
                            const double dw = scaled_exact(Wb, kb - (24 << 20));
                            sv[c * 8 + j] = __double_as_longlong(
                                bigd ? fma(__longlong_as_double(sv[c * 8 + j]), __hiloint2double(kb - (51 << 20), 0), dw)  // x 2^k
                                     : scaled_exact(sv[c * 8 + j], kb) + dw);
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty0);  // the next pair-tile's MMAs may start
            }
            if (prof) OZ_PROF_ADD(6, tdr1);
            OZ_PROF_T0(twork);
            if (!(dbg & 1)) {
#pragma unroll
                for (int c = 0; c < CPT / 8; ++c) {  // 8-column chunks of this thread's 64 columns
                    T w[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int lc = grp * CPT + c * 8 + j;
                        const int64_t gj = col0 + lc;
                        const bool diag = (c * 8 + j) == jd;  // gi == gj
                        T kv;
                        if constexpr (kTabExp) {  // kernel_value's RBF (distance clamped at 0, exactly 0 on
                            // the diagonal, R-9) in the scaled exponent form of exp_tab256: tp > 0 (a rounded
                            // distance below 0) and the diagonal give +0.0, by masking both words with
                            // (sign of tp) & (not diagonal) -- integer ops instead of fmin and selects
                            double tp = fma(a2, sval(c * 8 + j), ni + coln[lc]);
                            const int th = __double2hiint(tp);
                            const int keep = (th >> 31) & (diag ? 0 : -1);
                            tp = __hiloint2double(th & keep, __double2loint(tp) & keep);
                            kv = exp_tab256(tp, etab);
#ifdef PLSSVM_OZ_EPI_TAX  // experiment (A/B only, results perturbed by <= 1e-300): a second exp per entry,
                          // to measure what epilogue instructions cost at the power cap
                            kv = fma(1e-300, exp_tab256(tp * 0.999, etab), kv);
#endif
                        } else {
                            kv = kernel_value<KT, T>(sval(c * 8 + j), ni, coln[lc], diag, kp);
                        }
                        if constexpr (MODE == OZ_PREDICT) {
                            rs = fma(colp[lc], kv, rs);
                        } else if constexpr (MODE == OZ_MATVEC) {
                            w[j] = kv;  // Eq. 16's other terms per row / column at the end (p = 0 on padding)
                        } else {  // qtilde_value (Eq. 16) with the row constant Q_mm - q_i hoisted
                            const T v = (kv + (diag ? invC : T(0))) - colq[lc] + cqi;
                            w[j] = (gi < m1 && gj < m1) ? v : T(0);
                        }
                    }
                    if constexpr (MODE == OZ_MATVEC) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            rs = fma(w[j], colp[grp * CPT + c * 8 + j], rs);
                            w[j] *= pi;
                        }
                        if (mirrored) {  // CTA-uniform: column sums over the warp's 32 rows
                            // transpose-reduce 8 values over 32 lanes: lanes l with (l & 3) == 0 end
                            // with column 4 b4 + 2 b3 + b2 (b_k = bit k of l); fixed order
#pragma unroll
                            for (int o = 16, n = 4; o >= 4; o >>= 1, n >>= 1) {
                                const bool up = (lane & o) != 0;
#pragma unroll
                                for (int i = 0; i < n; ++i) {
                                    const T send = up ? w[i] : w[i + n];
                                    const T keep = up ? w[i + n] : w[i];
                                    w[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                                }
                            }
                            T tot = w[0] + __shfl_xor_sync(0xffffffffu, w[0], 2);
                            tot += __shfl_xor_sync(0xffffffffu, tot, 1);
                            if ((lane & 3) == 0) {
                                const int cc = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                                redc[quarter * TN + grp * CPT + c * 8 + cc] = tot;
                            }
                        }
                    } else if constexpr (MODE == OZ_PRECOMPUTE) {
                        if (qdst) {
#pragma unroll
                            for (int j = 0; j < 8; j += 2) {
                                if constexpr (sizeof(T) == 8)
                                    *reinterpret_cast<double2 *>(qdst + c * 8 + j) = make_double2(w[j], w[j + 1]);
                                else
                                    *reinterpret_cast<float2 *>(qdst + c * 8 + j) = make_float2(w[j], w[j + 1]);
                            }
                        }
                        if (qmir) {  // transposed copy: column lc of this tile = row lc of tile (J, I)
#pragma unroll
                            for (int j = 0; j < 8; ++j) qmir[int64_t(grp * CPT + c * 8 + j) * kTile] = w[j];  // coalesced
                        }
                    }
                }
            }

            if constexpr (MODE == OZ_MATVEC) {
                redr[grp * kTile + lr] = rs;
                asm volatile("bar.sync 1, %0;" ::"n"(O::EPI_THREADS) : "memory");  // B2
                auto rowsum = [&](int row) {  // the column groups' partials in fixed order
                    if constexpr (NG == 2) return redr[row] + redr[kTile + row];
                    else return (redr[row] + redr[kTile + row]) + (redr[2 * kTile + row] + redr[3 * kTile + row]);
                };
                if (used) {
                    const int64_t lrow0 = row0 - int64_t(band0) * kTile;
                    auto tsum = [&](int u) { return (psum[u] + psum[4 + u]) + (psum[8 + u] + psum[12 + u]); };
                    if (et < kTile) {  // row et (= this thread's lr): + (Q_mm - q_i) sum p_J - sum (q p)_J
                        const T corr = fma(cqi, tsum(0), -tsum(1)) + ((I == J) ? invC * pi : T(0));
                        Ypart[int64_t(J) * band_rows + lrow0 + et] = rowsum(et) + corr;
                    } else if (mirrored && et < 2 * kTile) {
                        const int cidx = et - kTile;
                        const int64_t lcol0 = col0 - int64_t(band0) * kTile;
                        const T corr = fma(Qmm - colq[cidx], tsum(2), -tsum(3));
                        Ypart[int64_t(I) * band_rows + lcol0 + cidx] =
                            ((redc[cidx] + redc[TN + cidx]) + (redc[2 * TN + cidx] + redc[3 * TN + cidx])) + corr;
                    }
                }
            } else if constexpr (MODE == OZ_PREDICT) {
                redr[grp * kTile + lr] = rs;
                asm volatile("bar.sync 1, %0;" ::"n"(O::EPI_THREADS) : "memory");  // B2
                if (used && et < kTile) {
                    const T fs = NG == 2 ? redr[et] + redr[kTile + et]
                                         : (redr[et] + redr[kTile + et]) + (redr[2 * kTile + et] + redr[3 * kTile + et]);
                    Ypart[int64_t(J) * band_rows + row0 + et] = fs;
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(O::EPI_THREADS) : "memory");  // B3: smem partials / column data reusable
            if (prof) OZ_PROF_ADD(7, twork);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // no more MMAs into either CTA's TMEM, no more remote arrives
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(O::TMEM_COLS));
    }
}

}  // namespace plssvm
