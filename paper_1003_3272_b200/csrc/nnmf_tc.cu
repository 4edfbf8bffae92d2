// nnmf_tc.cu -- tensor-core (tcgen05, kind::f16) path of the NNMF MM
// iteration for large fp32 problems, ranks 17..128 on rank tiles of 64
// (BASELINE config 4) and 128 (see Tc<RK> below).
// Reference: nnmf_objective / nnmf_update_v / nnmf_update_w (nnmf.py:75-110)
// and the V-then-W step of _FrobeniusNnmf (nnmf.py:153-156).
//
// Split products.  The two contractions with X are the whole cost (SURVEY.md
// 8(d): 4mnr of 5.5e11 flops).  Both run on the 5th-gen tensor cores as
// fp32-faithful split products: every fp32 operand x is scaled by a power of
// two 2^e (exact) so the largest |x 2^e| lies in [2^14, 2^15), then split
// into two fp16 values hi = rn(x 2^e), lo = rn(x 2^e - hi) -- 22 significant
// bits.  x w ~ hi_x hi_w + hi_x lo_w + lo_x hi_w, accumulated in fp32 in TMEM
// and scaled back by 2^-(e_x + e_w) in fp64.  fp16 and not 3xTF32: a
// single-CTA tcgen05.mma costs ~110-175 cycles per 32 bytes of K of its A
// operand (measured), so the A bytes per X element set the MMA time; tf32
// hi + lo are 8 bytes, fp16 hi + lo are 4.
//
// Pre-split X.  X is constant over a run, so its scaled fp16 hi / lo pair is
// made ONCE per X (presplit_kernel), row-major: the V step reads it K-major,
// the W step as an MN-major operand (4 bytes per element of X in HBM, all read
// per half step,
// as many as the fp32 X itself).  Both kernels stream [X_hi | X_lo] tiles
// from TMA straight into SS MMAs.
//
// Objective.  f(V, W) = sum_ij (x_ij - v_i . w_j)^2 is an EXPLICIT residual
// (the Gram-trace identity sum x^2 - 2<V, X W^T> +
// <V^T V, W W^T> cancels catastrophically in fp32 when ||X||^2 / f is large),
// evaluated inside the V step's X stream with no extra HBM traffic:
//   * per 128 x 64 X stage the MMA warp also issues R0 = V_h W_hi (4 MMAs,
//     N = 64, B = the W_hi half of the W chunk already in shared memory read
//     as an MN-major operand), V_h = fp16 of V scaled per row by 2^ev_i;
//   * eight residual warps read R0 from TMEM and the X stage from shared
//     memory and accumulate F0 = sum (x - v_h.w_hi)^2 (fp32 squares of 16
//     terms folded into fp64);
//   * the rest is exact algebra the update epilogue adds per row from what it
//     holds (Q = X W^T, V G_W, V, and X_hi.W_lo in its own accumulator
//     columns): the W_lo part of the residual,
//       -2 <v_h, X W_lo^T> + v_h (2 W_hi W_lo^T + W_lo W_lo^T) v_h^T
//     (X W_lo^T ~ X_hi.W_lo: the X_lo.W_lo product is ~2^-24 relative; the
//     Gram G_c from gram3_kernel), and V's rounding E = V - V_h,
//       -2 <(X - V W) W^T, E> - sum_i e_i G_W e_i^T.
//     E is ~2^-12 V and W_lo ~2^-12 W, so these terms are small next to f;
//     F0 is a sum of squares (no cancellation).  tests/test_nnmf_tc_gpu.py
//     and tests/test_nnmf_c4_gpu.py check f against fp64 residuals on
//     well-fit data (||X||^2 / f ~ 1e4) and at C4.  (The CTA-pair form keeps
//     R' = V_h [W_hi | W_lo], N = 128, and only the E terms.)
//
//   nnmf_vstep_tc  (persistent, one CTA per SM, 14 warps, one 128-row tile
//                  per pass, two accumulator sets so pass p's epilogue
//                  overlaps pass p + 1's MMAs)
//     warp 0     TMA: V_h tile per pass; per 64-column stage the W chunk
//                [W_hi ; W_lo] and the X stage [X_hi | X_lo]
//     warp 1     per stage 4 x (SS MMA N = 128 X_hi.[W_hi; W_lo] + SS MMA
//                N = 64 X_lo.W_hi) into Q (3 x 64 columns), then 4 x SS MMA
//                N = 64 V_h.W_hi into a residual buffer
//     warps 2-9  residual (two groups of 4 alternate stages)
//     warps 10-13 epilogue: V' = V * Q / (V G_W + 1e-300), max(V'), the
//                correction terms above
//   nnmf_vprep     V' -> V'^T hi / lo fp16 [64][m] (scaled): the W-step B operand
//   nnmf_wstep_tc  P^T = X^T V' (M = 128 columns of X, N = 64, K = rows),
//                split-K over row ranges; per-split partials reduced in fixed
//                order -> deterministic.
//
// HBM roofline: each kernel streams X once (m n 4 bytes) -> two passes per
// iteration; tensor work 3 x 2mnr per kernel plus 2 x 2mnr for R'.
#include <cuda_fp16.h>

#include "mmk_common.cuh"
#include "nnmf_tc.h"
#include "tc_common.cuh"

namespace {

using namespace mmk;

constexpr int R = 64;            // rank of the tensor-core path
constexpr int BM = 128;          // UMMA M: rows of X (V step) / columns of X (W step)
constexpr int BK = 64;           // K per stage (one 128-byte fp16 operand row)
constexpr uint32_t SXH = BM * BK * 2;       // 16 KB  fp16 X tile [128 x 64]
constexpr uint32_t SX = 2 * SXH;            // 32 KB  X stage [X_hi | X_lo]
constexpr uint32_t SOP = R * BK * 2;        //  8 KB  fp16 operand chunk hi; same again for lo
constexpr uint32_t SGW = R * R * 4;         // 16 KB  G_W (fp32) for the V-step epilogue
constexpr int XST = 4;                      // W step X ring (128 KB in flight per SM)
#ifndef MMK_TC_XSTV
#define MMK_TC_XSTV 4
#endif
constexpr int XSTV = MMK_TC_XSTV;           // V step X ring
#ifndef MMK_TC_GW_SMEM
#define MMK_TC_GW_SMEM 1
#endif
#ifndef MMK_TC_OST
#define MMK_TC_OST 3
#endif
#ifndef MMK_TC_XS128   // rank-128 tile: X ring / operand ring depths (224 KB of smem)
#define MMK_TC_XS128 4
#endif
#ifndef MMK_TC_OST128
#define MMK_TC_OST128 2
#endif
#ifndef MMK_TC_DEFER_R0
#define MMK_TC_DEFER_R0 0
#endif
constexpr int OST = MMK_TC_OST;             // operand ring (V step: one W chunk per X stage,
                                            // held until the residual MMAs finish)
constexpr int NRES = 8;                     // residual warps (two groups of 4)
constexpr int kVThreads = 32 * (2 + NRES + 4);   // TMA, MMA, residual x8, epilogue x4
constexpr int kWThreads = 32 * (2 + 4);          // TMA, MMA, epilogue x4
constexpr uint32_t SVH = BM * R * 2;        // 16 KB  V_h tile [128 rows x 64 ranks]
constexpr uint32_t SMEM_V = XSTV * SX + OST * 2 * SOP + 2 * SVH + (MMK_TC_GW_SMEM ? SGW : 0) + 1024;
// pair form: half-size operand slots and G_W read through L1 leave room for a
// deeper X ring
#ifndef MMK_TC_XSTV2
#define MMK_TC_XSTV2 4   // even: see Tc::XS
#endif
constexpr int XSTV2 = MMK_TC_XSTV2;
constexpr int XSMAX = XSTV2 > XSTV ? XSTV2 : XSTV;
constexpr uint32_t SMEM_V2 = XSTV2 * SX + OST * SOP + 2 * SVH + 1024;
constexpr int OSTW = 3;                     // W step operand ring (a V'^T chunk feeds CB stages)
constexpr uint32_t SMEM_W = XST * SX + OSTW * 2 * SOP + 1024;
static_assert(SMEM_V + 2048 <= 232448, "dynamic + static shared memory per CTA");
static_assert(SMEM_V2 + 2048 <= 232448, "dynamic + static shared memory per CTA (pair)");
constexpr int ACC = 2 * R;                  // accumulator columns: [X.Wh | X.Wl] (N = 128)
constexpr int CB = 2;                       // W step: 128-column blocks per item
constexpr int TM_COLS = 512;
// V step TMEM, single CTA: two Q sets of [X_hi.W_hi | X_hi.W_lo | X_lo.W_hi]
// (3 x 64 columns) and two residual buffers R0 = V_h.W_hi (64 columns); CTA
// pair: two Q sets of 128 columns and two R' = V_h.[W_hi | W_lo] buffers of 128
constexpr int NRB = 2;
constexpr uint32_t QW1 = 3 * R, RW1 = R;        // single CTA
constexpr uint32_t QW2 = ACC, RW2 = ACC;        // CTA pair
static_assert(2 * QW1 + NRB * RW1 <= TM_COLS, "V-step TMEM budget (single CTA)");
static_assert(2 * QW2 + NRB * RW2 <= TM_COLS, "V-step TMEM budget (pair)");
static_assert(2 * CB * ACC <= TM_COLS, "W step: two accumulator sets");

// Rank tiles of the tensor-core path: RK = 64 (ranks 17..64, the layout
// above) and RK = 128 (ranks 65..128, zero-padded to 128).  At RK = 128 a
// single-CTA Q set [hh | hl | lh] is 384 TMEM columns, so the V step keeps ONE
// Q set (its epilogue copies Q out to a global scratch and releases the set
// before the V' arithmetic) beside the two 64-column residual buffers, one
// V_h tile buffer (32 KB) and a 3-deep X ring; the W step takes one 128-column
// block per item (accumulator [X.V_hi | X.V_lo] = 256 columns, two sets).
template <int RK>
struct Tc {
    static constexpr uint32_t SOP = RK * BK * 2;     // fp16 operand chunk [RK x 64] (hi; lo again)
    static constexpr uint32_t SVH = BM * RK * 2;     // V_h tile [128 rows x RK ranks]
    static constexpr int ACC = 2 * RK;               // [X.B_hi | X.B_lo] accumulator columns
    static constexpr int NQ = RK == 64 ? 2 : 1;      // V step: Q accumulator sets
    static constexpr int NVB = RK == 64 ? 2 : 1;     // V step: V_h tile buffers
    // V step X ring (single CTA): EVEN, because the two residual groups take
    // alternate stages -- with an odd depth a group's next use of a slot can
    // come two phases after its previous one (the other group's stage in
    // between), and its parity wait would pass on the stale phase
    static constexpr int XS = RK == 64 ? XSTV : MMK_TC_XS128;
    static constexpr int OST = RK == 64 ? MMK_TC_OST : MMK_TC_OST128;   // V step operand ring
    static constexpr bool GWS = RK == 64 && MMK_TC_GW_SMEM;   // G_W staged in smem
    static constexpr uint32_t QW = 3 * RK;           // single-CTA Q set [hh | hl | lh]
    static constexpr uint32_t SMEM_V =
        XS * SX + OST * 2 * SOP + NVB * SVH + (GWS ? SGW : 0) + 1024;
    static_assert(XS % 2 == 0, "the residual groups alternate stages: even X ring");
    static constexpr int CB = RK == 64 ? 2 : 1;      // W step: 128-column blocks per item
    static constexpr uint32_t SMEM_W = XST * SX + OSTW * 2 * SOP + 1024;
    static_assert(NQ * QW + NRB * BK <= TM_COLS, "V-step TMEM budget");
    static_assert(2 * CB * ACC <= TM_COLS, "W-step TMEM budget");
    static_assert(SMEM_V + 2048 <= 232448 && SMEM_W + 2048 <= 232448, "shared memory per CTA");
    static_assert(OST <= ::OST, "VBars holds up to OST operand slots");
};
static_assert(Tc<64>::SMEM_V == SMEM_V && Tc<64>::SMEM_W == SMEM_W, "rank-64 layout");

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// power-of-two exponent e with max * 2^e in [2^14, 2^15) (0 for max == 0)
__host__ __device__ inline int scale_exp(float mx) {
    if (!(mx > 0.f)) return 0;
    int E;
    frexpf(mx, &E);   // mx = f 2^E, f in [0.5, 1)
    int e = 15 - E;
    return e < -120 ? -120 : (e > 120 ? 120 : e);
}

// fp16 hi / lo of an already-scaled value, packed pairwise (even K in the
// low half of the 32-bit word)
__device__ __forceinline__ void split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

// kind::f16 instruction descriptor: fp16 A/B, fp32 D; b_mn = 1 for an
// MN-major B operand
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int b_mn = 0) {
    return (1u << 4) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

// One 64-column stage of Q += X W^T with A = [X_hi | X_lo] (two 128-row x
// 64-K fp16 tiles, 128B swizzle) and the operand chunk [B_hi ; B_lo] stacked
// along N (64 + 64 rows, K-major): per K16 step an SS MMA with N = 128 gives
// D[:, 0:64] += X_hi.B_hi, D[:, 64:128] += X_hi.B_lo, and one with N = 64
// adds X_lo.B_hi into d_lo (its own 64 columns: the epilogue needs X_hi.B_lo
// alone for the objective's W_lo correction).  The epilogue sums the parts.
// Issued warp-converged (every lane calls it; one elected lane issues)
template <int RK>
__device__ __forceinline__ void issue_split_stage_e(uint32_t d, uint32_t d_lo, const uint8_t* xs,
                                                    const uint8_t* bhl, bool first) {
    const uint64_t db0 = tc::sdesc_sw128(bhl, 16, 1024);
    const uint64_t ah = tc::sdesc_sw128(xs, 16, 1024);
    const uint64_t al = tc::sdesc_sw128(xs + SXH, 16, 1024);
    constexpr uint32_t id_hi = idesc_f16(BM, 2 * RK);
    constexpr uint32_t id_lo = idesc_f16(BM, RK);
#pragma unroll
    for (int ks = 0; ks < BK / 16; ++ks) {
        const uint32_t acc = (first && ks == 0) ? 0u : 1u;
        tc::mma_f16ss_e(d, ah + ks * 2, db0 + ks * 2, id_hi, acc);
        tc::mma_f16ss_e(d_lo, al + ks * 2, db0 + ks * 2, id_lo, acc);
    }
}

// W-step stage with A MN-major: the X stage holds [X_hi | X_lo] as row-major
// tiles of the pre-split X (K = 64 rows of X, M = 128 columns, the columns
// contiguous: two 64-column boxes per half, 128B swizzle), read as A = X^T
// directly -- no transposed copy of X.  LBO = the second 64-column box, SBO =
// the next 8 rows; a K16 step advances 16 rows (2048 bytes).
constexpr uint32_t SXB = BK * 64 * 2;   // 8 KB: one [64 rows x 64 columns] fp16 box
template <int RK>
__device__ __forceinline__ void issue_split_stage_mn(uint32_t d, const uint8_t* xs,
                                                     const uint8_t* bhl, bool first) {
    const uint64_t db0 = tc::sdesc_sw128(bhl, 16, 1024);
    const uint64_t ah = tc::sdesc_sw128(xs, SXB, 1024);
    const uint64_t al = tc::sdesc_sw128(xs + SXH, SXB, 1024);
    constexpr uint32_t id_hi = idesc_f16(BM, 2 * RK) | (1u << 15);   // A MN-major
    constexpr uint32_t id_lo = idesc_f16(BM, RK) | (1u << 15);
#pragma unroll
    for (int ks = 0; ks < BK / 16; ++ks) {
        const uint32_t acc = (first && ks == 0) ? 0u : 1u;
        tc::mma_f16ss(d, ah + ks * (2048 >> 4), db0 + ks * 2, id_hi, acc);
        tc::mma_f16ss(d, al + ks * (2048 >> 4), db0 + ks * 2, id_lo, 1);
    }
}

// The same stage for a CTA pair (cta_group::2, M = 256, issued by the
// leader): A = each CTA's own [X_hi | X_lo] stage (same offset), B = this
// CTA's half of the W chunk (leader [W_hi], peer [W_lo]: N = 128 split
// between the pair); per K16 step X_hi.[W_hi ; W_lo] and X_lo.[W_hi ; W_lo].
__device__ __forceinline__ void issue_split_stage_pair(uint32_t d, const uint8_t* xs,
                                                       const uint8_t* bh, bool first) {
    const uint64_t db0 = tc::sdesc_sw128(bh, 16, 1024);
    const uint64_t ah = tc::sdesc_sw128(xs, 16, 1024);
    const uint64_t al = tc::sdesc_sw128(xs + SXH, 16, 1024);
    constexpr uint32_t id = idesc_f16(2 * BM, ACC);
#pragma unroll
    for (int ks = 0; ks < BK / 16; ++ks) {
        const uint32_t acc = (first && ks == 0) ? 0u : 1u;
        tc::mma_f16ss_pair_e(d, ah + ks * 2, db0 + ks * 2, id, acc);
        tc::mma_f16ss_pair_e(d, al + ks * 2, db0 + ks * 2, id, 1);
    }
}

// Pipeline trace of CTA 0 (timing studies only: -DMMK_TC_TRACE, never in
// the product build): clock64 per stage at 8 points, see TRACE_AT below
#ifdef MMK_TC_TRACE
__device__ unsigned long long g_tctrace[8][4096];
#define TRACE_AT(what, it)                                                       \
    do {                                                                         \
        if (blockIdx.x == 0 && (it) < 4096) g_tctrace[what][it] = clock64();     \
    } while (0)
#else
#define TRACE_AT(what, it) \
    do {                   \
    } while (0)
#endif

// Scales shared by the kernels of one iteration (device, in the workspace):
// exponents of X (cached with sum x^2), W and V'; maxima as float bits.
struct Scales {
    int ex, ew, ev, pad_;
    unsigned int wmax_bits, vmax_bits, pad2_, pad3_;
};

// ---------------------------------------------------------------------------
// V step.  mX / mX2: fp16 hi / lo maps of the pre-split X (m x n); mWh / mWl:
// W_hi / W_lo (64 x n).  part[b] = this CTA's share of f(V, W); the V'
// maximum goes to sc->vmax_bits.
//
// Pipeline per 64-column stage `it` of a 128-row tile (pass p = tile):
//   TMA      V_h tile of the pass (split_v_kernel's fp16 V, per-row scale);
//            per stage the W chunk [W_hi ; W_lo] -> operand slot it % OST and
//            the X stage [X_hi | X_lo] -> slot it % XSTV
//   MMA      Q(it) += X_hi [W_hi ; W_lo] + X_lo W_hi (8 SS MMAs), commit ->
//            xempty; R'(it) = V_h [W_hi | W_lo] (4 SS MMAs N = 128, B = the W
//            chunk read MN-major: rows = ranks = K, W_hi and W_lo two 64-column
//            atoms), commit -> rfull, oempty
//   residual group (it % 2) reads its rows of X(it) into registers as soon
//            as the stage lands (release -> xempty), then R'(it) from TMEM
//   epilogue V' of the tile from Q (two accumulator sets: pass p's epilogue
//            overlaps pass p + 1)
// Measured at C4 (scripts/vstep_time.py, profiles/r02/README.md): 1.69 ms,
// against ~1.3 ms for the same kernel without the residual.  Variant builds
// put ~0.26 ms on the R' MMAs and ~0.17 ms on the residual warps' X reads;
// ncu shows no unit saturated (tensor pipe 42 %, tensor-core smem reads 51 %,
// L1 55 %): per stage the MMA warp waits ~230 cycles for an R' buffer (two
// fit in TMEM beside the two Q sets) and ~260 for X (a 4-deep ring fills the
// 227 KB of shared memory).  The CTA-pair form below issues its 12 MMAs in
// ~360 cycles instead of ~570 but is slower end to end (1.82 ms): the extra
// X_lo.W_lo products raise power (lower clocks) and every stage crosses the
// pair twice (forwarded X completion, remote rempty arrivals).
struct VBars {
    uint64_t xfull[XSMAX], xempty[XSMAX], ofull[OST], oempty[OST];
    uint64_t pxfull[XSMAX];             // pair, leader: the peer's X stage landed (forwarded)
    uint64_t vfull[2], vempty[2];       // V_h tiles of a pass (TMA -> MMA)
    uint64_t dfull[2], dempty[2];       // Q accumulator sets: MMA -> epilogue
    uint64_t rfull[NRB], rempty[NRB];   // residual buffers: MMA -> residual warps
};

// per-row exponent of V_h: max_k |v_ik| * 2^ev in [2^14, 2^15)
template <int RK>
__device__ __forceinline__ int row_exp(const float4* vr) {
    float mx = 0.f;
#pragma unroll
    for (int l4 = 0; l4 < RK / 4; ++l4) {
        const float4 v = vr[l4];
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    return scale_exp(mx);
}

// PAIR (the default at C4): the kernel runs as CTA pairs (clusters of 2).
// Pair q takes the 256-row units q, q + G/2, ...; CTA rank r of the pair
// owns the 128-row tile 2u + r of unit u (its X stages, its V_h tile, its
// TMEM lanes of Q and R').  Only the leader's MMA warp issues, with
// tcgen05.mma.cta_group::2 (M = 256, one instruction for both tiles): a pair
// MMA runs at the full tensor rate (64 cycles at N = 128, measured) where a
// single-CTA M = 128 one costs ~110-175 cycles whatever N is, and with the
// residual MMAs the single-CTA form is tensor-issue bound (12 MMAs per stage).
// B (N = 128) is split between the pair: the W chunk's [W_hi] rows in the
// leader's operand slot, [W_lo] at the same offset in the peer's -- read
// K-major for Q and MN-major for R'.  Q's second MMA per K16 step is
// X_lo.[W_hi ; W_lo] (N = 128: a pair MMA cannot split an N = 64 W_hi between
// the CTAs), which adds the X_lo.W_lo product the single-CTA form omits.
// Both CTAs' TMA loads complete on the LEADER's full barriers; commits are
// multicast to the barriers of both CTAs; the epilogue and residual warps of
// both CTAs arrive on the leader's dempty / rempty (cluster address).  The
// residual warps read their X stage after the stage's R' commit (which the
// MMA could only issue once the stage had landed: the peer never sees its own
// xfull complete).
template <bool PAIR, int RK>
__global__ void __launch_bounds__(kVThreads, 1)
nnmf_vstep_tc(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mX2,
              const __grid_constant__ CUtensorMap mWh, const __grid_constant__ CUtensorMap mWl,
              const __grid_constant__ CUtensorMap mVh, const float* __restrict__ V,
              const float* __restrict__ GWf, const float* __restrict__ Gc,
              float* __restrict__ Vout, Scales* sc, int m, int n,
              double* __restrict__ part, float* __restrict__ Qs) {
    using C = Tc<RK>;
    static_assert(!PAIR || RK == 64, "the CTA-pair form is rank-64 only");
    constexpr uint32_t SOPK = C::SOP, SVHK = C::SVH;
    constexpr uint32_t OSLOT = PAIR ? SOP : 2 * SOPK;  // operand slot: pair = this CTA's half
    constexpr uint32_t QW = PAIR ? QW2 : C::QW, RW = PAIR ? RW2 : RW1;
    constexpr int NQ = PAIR ? 2 : C::NQ, NVB = PAIR ? 2 : C::NVB;
    constexpr uint32_t TM_RES = NQ * QW;               // residual buffers after the Q sets
    constexpr int NARR = PAIR ? 8 : 4;                 // arrivals on dempty / rempty
    constexpr int XS = PAIR ? XSTV2 : C::XS;           // X ring depth
    constexpr int OSL = PAIR ? OST : C::OST;           // operand ring depth
    static_assert(XS % 2 == 0, "the residual groups alternate stages: even X ring");
    static_assert(XS <= XSMAX && OSL <= OST, "VBars sizes");
    constexpr bool GWS = !PAIR && C::GWS;              // G_W staged in smem
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = align1024(smem_raw);
    uint8_t* xring = base;
    uint8_t* oring = base + XS * SX;
    uint8_t* vbuf = oring + OSL * OSLOT;
    float* gws = reinterpret_cast<float*>(vbuf + NVB * SVHK);
    __shared__ VBars B;
    __shared__ uint32_t tmem_base;
    __shared__ double red[kVThreads / 32];
    __shared__ float vmx[kVThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (m + BM - 1) / BM, nk = (n + BK - 1) / BK;
    const int rank = PAIR ? (int)tc::cluster_rank() : 0;
    const int G = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
    const int me = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
    const int units = PAIR ? (ntiles + 1) / 2 : ntiles;
    const int mine = units > me ? (units - 1 - me) / G + 1 : 0;
    auto tile_of = [&](int p) { return PAIR ? 2 * (me + p * G) + rank : me + p * G; };
    // G_W rounded to fp32 (gram_sum_kernel), staged for the denominator rows
    if (GWS)
        for (int i = threadIdx.x; i < R * R / 4; i += kVThreads)
            reinterpret_cast<float4*>(gws)[i] = __ldg(reinterpret_cast<const float4*>(GWf) + i);
    if (threadIdx.x == 0) {
        for (int s = 0; s < XS; ++s) {
            tc::mbar_init(&B.xfull[s], 1);
            tc::mbar_init(&B.xempty[s], 5);   // the residual group's 4 warps + the Q MMAs' commit
            tc::mbar_init(&B.pxfull[s], 1);   // pair: the peer's forwarder
        }
        for (int s = 0; s < OSL; ++s) {
            tc::mbar_init(&B.ofull[s], 1);
            tc::mbar_init(&B.oempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&B.vfull[b], 1);
            tc::mbar_init(&B.vempty[b], 1);
            tc::mbar_init(&B.dfull[b], 1);
            tc::mbar_init(&B.dempty[b], NARR);   // epilogue warps (of both CTAs)
        }
        for (int b = 0; b < NRB; ++b) {
            tc::mbar_init(&B.rfull[b], 1);
            tc::mbar_init(&B.rempty[b], NARR);   // the residual group(s) that read it
        }
        tc::fence_barrier_init();
        tc::tma_prefetch(&mX);
        tc::tma_prefetch(&mX2);
        tc::tma_prefetch(&mWh);
        tc::tma_prefetch(&mWl);
        tc::tma_prefetch(&mVh);
    }
    if (warp == 1) {
        if constexpr (PAIR)
            tc::tmem_alloc_pair<TM_COLS>(&tmem_base);
        else
            tc::tmem_alloc<TM_COLS>(&tmem_base);
    }
    tc::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) tc::cluster_sync();   // barriers initialised, TMEM allocated in both
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    // the leader's copy of a barrier (pair: TMA completions and the peer's
    // consumer arrivals are counted there)
    auto lead = [](uint64_t* bar) { return tc::map_to_rank(bar, 0); };
    auto arrive_lead = [&](uint64_t* bar) {
        if (PAIR && rank != 0)
            tc::mbar_arrive_cluster(lead(bar));
        else
            tc::mbar_arrive(bar);
    };
    double acc = 0.0;   // residual warps: F'; epilogue warps: the correction terms
    float vmax = 0.f;
    if (warp == 0) {
        if (lane == 0) {   // TMA producer
            int it = 0;
            for (int p = 0; p < mine; ++p) {
                const int tile = tile_of(p), vb = p % NVB;
                tc::mbar_wait(&B.vempty[vb], ((p / NVB) & 1) ^ 1);
                if constexpr (PAIR) {
                    if (rank == 0) tc::mbar_expect_tx(&B.vfull[vb], 2 * SVH);
                    tc::tma_load_2d_pair(vbuf + vb * SVH, &mVh, lead(&B.vfull[vb]), 0, tile * BM);
                } else {
                    // [128 rows x RK ranks] as RK / 64 column atoms of 128-byte rows
                    tc::mbar_expect_tx(&B.vfull[vb], SVHK);
#pragma unroll
                    for (int a = 0; a < RK / 64; ++a)
                        tc::tma_load_2d(vbuf + vb * SVHK + a * (SVHK / (RK / 64)), &mVh,
                                        &B.vfull[vb], 64 * a, tile * BM);
                }
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int os = it % OSL, xs = it % XS;
                    tc::mbar_wait(&B.oempty[os], ((it / OSL) & 1) ^ 1);
                    if constexpr (PAIR) {   // this CTA's half of [W_hi ; W_lo]
                        if (rank == 0) tc::mbar_expect_tx(&B.ofull[os], 2 * SOP);
                        tc::tma_load_2d_pair(oring + os * OSLOT, rank == 0 ? &mWh : &mWl,
                                             lead(&B.ofull[os]), kb * BK, 0);
                    } else {
                        tc::mbar_expect_tx(&B.ofull[os], 2 * SOPK);
                        tc::tma_load_2d(oring + os * OSLOT, &mWh, &B.ofull[os], kb * BK, 0);
                        tc::tma_load_2d(oring + os * OSLOT + SOPK, &mWl, &B.ofull[os], kb * BK, 0);
                    }
                    tc::mbar_wait(&B.xempty[xs], ((it / XS) & 1) ^ 1);
                    TRACE_AT(0, it);
                    // own X stage -> own xfull (pair: the peer's forwarder
                    // passes its completion on to the leader's pxfull)
                    tc::mbar_expect_tx(&B.xfull[xs], SX);
                    tc::tma_load_2d(xring + xs * SX, &mX, &B.xfull[xs], kb * BK, tile * BM);
                    tc::tma_load_2d(xring + xs * SX + SXH, &mX2, &B.xfull[xs], kb * BK, tile * BM);
                }
            }
        }
    } else if (warp == 1) {
        if (!PAIR || rank == 0) {   // MMA issuer: the whole warp, one elected lane issues
            // R' = V_h [W_hi | W_lo] (pair, N = 128) or R0 = V_h W_hi (single, N = 64)
            constexpr uint32_t id_res = idesc_f16(PAIR ? 2 * BM : BM, RW, 1);
            int it = 0;
            for (int p = 0; p < mine; ++p) {
                const int b = p % NQ, vb = p % NVB;
                tc::mbar_wait(&B.dempty[b], ((p / NQ) & 1) ^ 1);
                tc::mbar_wait(&B.vfull[vb], (p / NVB) & 1);
                tc::tc_fence_after();
                const uint64_t va = tc::sdesc_sw128(vbuf + vb * SVHK, 16, 1024);
                // R0 MMAs of stage s (after its Q MMAs, or -- DEFER -- after the
                // Q MMAs of stage s + 1 of the same tile, so a late residual
                // buffer does not hold back the Q stream that frees X slots)
                auto issue_r0 = [&](int s_it) {
                    const int os = s_it % OSL, rb = s_it % NRB;
                    tc::mbar_wait(&B.rempty[rb], ((s_it / NRB) & 1) ^ 1);
                    if (lane == 0) TRACE_AT(3, s_it);
                    tc::tc_fence_after();
                    const uint8_t* ob = oring + os * OSLOT;
                    const uint64_t wr = tc::sdesc_sw128(ob, PAIR ? SOP : SOPK, 1024);   // MN-major
                    const uint32_t dr = tmem + TM_RES + rb * RW;
#pragma unroll
                    for (int ks = 0; ks < RK / 16; ++ks) {
                        // K16 step ks of V_h: column atom ks / 4 (16 KB apart), 32 bytes in
                        const uint64_t vk = va + (ks >> 2) * ((SVHK / (RK / 64)) >> 4) + (ks & 3) * 2;
                        if constexpr (PAIR)
                            tc::mma_f16ss_pair_e(dr, vk, wr + ks * (2048 >> 4), id_res,
                                                 ks ? 1u : 0u);
                        else
                            tc::mma_f16ss_e(dr, vk, wr + ks * (2048 >> 4), id_res, ks ? 1u : 0u);
                    }
                    if constexpr (PAIR) {
                        tc::mma_commit_pair_e(&B.rfull[rb]);
                        tc::mma_commit_pair_e(&B.oempty[os]);
                    } else {
                        tc::mma_commit_e(&B.rfull[rb]);
                        tc::mma_commit_e(&B.oempty[os]);
                    }
                    if (lane == 0) TRACE_AT(4, s_it);
                };
                constexpr bool DEFER = !PAIR && MMK_TC_DEFER_R0;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int os = it % OSL, xs = it % XS;
                    tc::mbar_wait(&B.ofull[os], (it / OSL) & 1);
                    tc::mbar_wait(&B.xfull[xs], (it / XS) & 1);
                    if constexpr (PAIR) tc::mbar_wait(&B.pxfull[xs], (it / XS) & 1);
                    if (lane == 0) TRACE_AT(1, it);
                    tc::tc_fence_after();
                    const uint8_t* ob = oring + os * OSLOT;
                    if constexpr (PAIR)
                        issue_split_stage_pair(tmem + b * QW, xring + xs * SX, ob, kb == 0);
                    else
                        issue_split_stage_e<RK>(tmem + b * QW, tmem + b * QW + C::ACC,
                                                xring + xs * SX, ob, kb == 0);
                    if (lane == 0) TRACE_AT(2, it);
                    if constexpr (PAIR)
                        tc::mma_commit_pair_e(&B.xempty[xs]);
                    else
                        tc::mma_commit_e(&B.xempty[xs]);
                    if constexpr (DEFER) {
                        if (kb > 0) issue_r0(it - 1);
                    } else {
                        issue_r0(it);
                    }
                }
                if constexpr (DEFER) issue_r0(it - 1);
                if constexpr (PAIR) {
                    tc::mma_commit_pair_e(&B.dfull[b]);
                    tc::mma_commit_pair_e(&B.vempty[vb]);
                } else {
                    tc::mma_commit_e(&B.dfull[b]);
                    tc::mma_commit_e(&B.vempty[vb]);
                }
            }
        } else if (lane == 0) {
            // the peer's forwarder: each of its X stages landed -> the leader's pxfull
            const int total = mine * nk;
            for (int it = 0; it < total; ++it) {
                const int xs = it % XS;
                tc::mbar_wait(&B.xfull[xs], (it / XS) & 1);
                tc::mbar_arrive_cluster(lead(&B.pxfull[xs]));
            }
        }
    } else if (warp < 2 + NRES) {
        // residual group g takes the stages with it % 2 == g; thread = row
        // `quarter * 32 + lane` of the tile.  X-scaled units: d 2^ex = x_s -
        // R' 2^(ex - ev_i - ew) (powers of two, exact), squares of 16 terms in
        // fp32 (packed fp32x2) folded into fp64, times 2^-2ex at the end
        const int g = (warp - 2) >> 2, quarter = warp & 3, r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const int ex = sc->ex, ew = sc->ew;
        int it = 0;
        for (int p = 0; p < mine; ++p) {
            const long long row = (long long)tile_of(p) * BM + r;
            int ke = ex - (row < m ? row_exp<RK>(reinterpret_cast<const float4*>(V + row * RK)) : 0) -
                     ew;
            ke = ke < -126 ? -126 : (ke > 127 ? 127 : ke);
            const float nk2 = -exp2f((float)ke);
            const float2 nkk = make_float2(nk2, nk2);
            for (int kb = 0; kb < nk; ++kb, ++it) {
                if ((it & 1) != g) continue;
                // this row's 64 X values of the stage into registers, then release
                // the slot (its other user is the Q MMA, which commits on xempty)
                const int xs = it % XS;
                const int rb = it % NRB;
                const uint32_t rcol = (uint32_t)(rb * RW);
                const uint32_t rph = (uint32_t)((it / NRB) & 1);
                tc::mbar_wait(&B.xfull[xs], (it / XS) & 1);
                if (r == 0) TRACE_AT(5, it);
                const uint32_t xh = tc::smem_u32(xring + xs * SX) + r * 128;
                uint4 hv[8], lv[8];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    hv[cc] = tc::lds128(xh + ((cc ^ (r & 7)) * 16));
                    lv[cc] = tc::lds128(xh + SXH + ((cc ^ (r & 7)) * 16));
                }
                // the slot's next writer is the TMA (async proxy): order these
                // generic-proxy reads before it
                tc::fence_async_smem();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&B.xempty[xs]);
                tc::mbar_wait(&B.rfull[rb], rph);
                if (r == 0) TRACE_AT(6, it);
                tc::tc_fence_after();
                // R' in 8-column chunks, the load of chunk q + 1 in flight while
                // chunk q is consumed (one TMEM round trip exposed per stage)
                // pair: R' = V_h [W_hi | W_lo] (hi and lo halves summed here);
                // single CTA: R0 = V_h W_hi (the W_lo part enters exactly in the
                // epilogue through X_hi.W_lo and the Grams W_hi W_lo^T, W_lo W_lo^T)
                uint32_t th[2][8], tl[2][8];
                const uint32_t tr0 = tmem + TM_RES + rcol + lane_off;
                if constexpr (PAIR) {
                    tc::tmem_ld8x2_nw(tr0, tr0 + R, th[0], tl[0]);
                    tc::tmem_wait_ld8x2(th[0], tl[0]);
                } else {
                    tc::tmem_ld8_nw(tr0, th[0]);
                    tc::tmem_wait_ld8(th[0]);
                }
                float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < 8; ++q) {   // columns 8q .. 8q + 7
                    if (q < 7) {
                        if constexpr (PAIR)
                            tc::tmem_ld8x2_nw(tr0 + 8 * (q + 1), tr0 + R + 8 * (q + 1),
                                              th[(q + 1) & 1], tl[(q + 1) & 1]);
                        else
                            tc::tmem_ld8_nw(tr0 + 8 * (q + 1), th[(q + 1) & 1]);
                    }
                    if (!(q & 1)) s2 = make_float2(0.f, 0.f);
                    const uint4 hq = hv[q], lq = lv[q];
                    const uint32_t hw[4] = {hq.x, hq.y, hq.z, hq.w};
                    const uint32_t lw[4] = {lq.x, lq.y, lq.z, lq.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 xs2 = __fadd2_rn(
                            __half22float2(*reinterpret_cast<const __half2*>(&hw[e])),
                            __half22float2(*reinterpret_cast<const __half2*>(&lw[e])));
                        float2 rr = make_float2(__uint_as_float(th[q & 1][2 * e]),
                                                __uint_as_float(th[q & 1][2 * e + 1]));
                        if constexpr (PAIR)
                            rr = __fadd2_rn(rr, make_float2(__uint_as_float(tl[q & 1][2 * e]),
                                                            __uint_as_float(tl[q & 1][2 * e + 1])));
                        const float2 d = __ffma2_rn(rr, nkk, xs2);
                        s2 = __ffma2_rn(d, d, s2);
                    }
                    if (q & 1) acc += (double)(s2.x + s2.y);   // 16 terms per fold
                    if (q < 7) {
                        if constexpr (PAIR)
                            tc::tmem_wait_ld8x2(th[(q + 1) & 1], tl[(q + 1) & 1]);
                        else
                            tc::tmem_wait_ld8(th[(q + 1) & 1]);
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (r == 0) TRACE_AT(7, it);
                if (lane == 0) arrive_lead(&B.rempty[rb]);
            }
        }
        acc *= exp2(-2.0 * ex);
    } else {
        // epilogue: thread = row.  V' = V Q / (V G_W + 1e-300) with the row
        // of V G_W formed here (fp32, l ascending), plus the correction terms
        // -2 (Q - V G_W)_ik e_ik - e_ik (e G_W)_ik of f (fp64) for V's fp16
        // rounding E = V - V_h.  Single CTA: the residual warps summed
        // (x - v_h . w_hi)^2, so the W_lo part of the residual is added here
        // exactly, per row i and rank k:
        //   v_h,ik ((v_h,i G_c)_k - 2 (X W_lo^T)_ik),  G_c = 2 W_hi W_lo^T + W_lo W_lo^T
        // with X W_lo^T = the X_hi.W_lo accumulator (the X_lo.W_lo product, ~2^-24
        // relative, is left out) and G_c from gram3_kernel
        const int quarter = warp & 3;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const double qscale = exp2(-(double)(sc->ex + sc->ew));
        const uint32_t gws_s = tc::smem_u32(gws);
        for (int p = 0; p < mine; ++p) {
            const int b = p % NQ;
            tc::mbar_wait(&B.dfull[b], (p / NQ) & 1);
            tc::tc_fence_after();
            const long long row = (long long)tile_of(p) * BM + quarter * 32 + lane;
            const uint32_t ta = tmem + b * QW + lane_off;
            // Q part h (32 columns): q = X.W_hi (+ X_lo.W_hi), q2 = X_hi.W_lo
            auto load_q = [&](int h, float* q, float* q2) {
                tc::tmem_ld32(ta + h * 32, q);   // warp-collective: before any row guard
                tc::tmem_ld32(ta + RK + h * 32, q2);
                if constexpr (!PAIR) {   // + X_lo.W_hi (its own columns)
                    float q3[32];
                    tc::tmem_ld32(ta + 2 * RK + h * 32, q3);
#pragma unroll
                    for (int i = 0; i < 32; ++i) q[i] += q3[i];
                }
            };
            if constexpr (NQ == 1) {
                // one Q set (RK = 128): copy it out as [q | q2] rows of the
                // scratch and hand the set back to the MMA warp; the V'
                // arithmetic is vfinish_kernel's (G_W and G_c staged in its
                // shared memory -- here they would not fit beside the rings)
                float4* qrow = reinterpret_cast<float4*>(Qs + (row < m ? row : 0) * (2 * RK));
#pragma unroll 1
                for (int h = 0; h < RK / 32; ++h) {
                    float q[32], q2[32];
                    load_q(h, q, q2);
                    if (row < m) {
#pragma unroll
                        for (int k4 = 0; k4 < 8; ++k4) {
                            qrow[h * 8 + k4] = make_float4(q[4 * k4], q[4 * k4 + 1], q[4 * k4 + 2],
                                                           q[4 * k4 + 3]);
                            qrow[RK / 4 + h * 8 + k4] = make_float4(q2[4 * k4], q2[4 * k4 + 1],
                                                                    q2[4 * k4 + 2], q2[4 * k4 + 3]);
                        }
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_lead(&B.dempty[b]);
                continue;
            }
            const float4* vr = reinterpret_cast<const float4*>(V + (row < m ? row : 0) * RK);
            const int ev = row < m ? row_exp<RK>(vr) : 0;
            const float vs = exp2f((float)ev), vsi = exp2f(-(float)ev);
#pragma unroll 1
            for (int h = 0; h < RK / 32; ++h) {
                float q[32], q2[32];
                load_q(h, q, q2);
                if (row >= m) continue;
                float4* o = reinterpret_cast<float4*>(Vout + row * RK + h * 32);
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                    // columns h*32 + hh*8 .. +8: (V G_W) and (E G_W) in fp32
                    float den[8], eg[8], gcg[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) den[c] = eg[c] = gcg[c] = 0.f;
#pragma unroll 2
                    for (int l4 = 0; l4 < RK / 4; ++l4) {
                        const float4 vv = vr[l4];
                        const float va[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float el = va[e] - __half2float(__float2half_rn(va[e] * vs)) * vsi;
                            const uint32_t g4 =
                                gws_s + 4u * (uint32_t)((4 * l4 + e) * RK + h * 32 + hh * 8);
#pragma unroll
                            for (int c4 = 0; c4 < 2; ++c4) {
                                const float4 gg =
                                    GWS ? tc::lds128f(g4 + 16u * c4)
                                        : __ldg(reinterpret_cast<const float4*>(GWf) +
                                                (((4 * l4 + e) * RK + h * 32 + hh * 8) / 4 + c4));
                                den[4 * c4] = fmaf(va[e], gg.x, den[4 * c4]);
                                den[4 * c4 + 1] = fmaf(va[e], gg.y, den[4 * c4 + 1]);
                                den[4 * c4 + 2] = fmaf(va[e], gg.z, den[4 * c4 + 2]);
                                den[4 * c4 + 3] = fmaf(va[e], gg.w, den[4 * c4 + 3]);
                                eg[4 * c4] = fmaf(el, gg.x, eg[4 * c4]);
                                eg[4 * c4 + 1] = fmaf(el, gg.y, eg[4 * c4 + 1]);
                                eg[4 * c4 + 2] = fmaf(el, gg.z, eg[4 * c4 + 2]);
                                eg[4 * c4 + 3] = fmaf(el, gg.w, eg[4 * c4 + 3]);
                                if constexpr (!PAIR) {   // v_h G_c, G_c = 2 W_hi W_lo^T + W_lo W_lo^T
                                    const float vh = va[e] - el;
                                    const int gi = ((4 * l4 + e) * RK + h * 32 + hh * 8) / 4 + c4;
                                    const float4 gc = __ldg(reinterpret_cast<const float4*>(Gc) + gi);
                                    gcg[4 * c4] = fmaf(vh, gc.x, gcg[4 * c4]);
                                    gcg[4 * c4 + 1] = fmaf(vh, gc.y, gcg[4 * c4 + 1]);
                                    gcg[4 * c4 + 2] = fmaf(vh, gc.z, gcg[4 * c4 + 2]);
                                    gcg[4 * c4 + 3] = fmaf(vh, gc.w, gcg[4 * c4 + 3]);
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int kq = 0; kq < 2; ++kq) {
                        const int k4 = h * 8 + hh * 2 + kq;   // float4 index in the row
                        const float4 vv = vr[k4];
                        const float va[4] = {vv.x, vv.y, vv.z, vv.w};
                        float nv[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int c = 4 * kq + i, kk = hh * 8 + c;   // column within the half
                            const double vk = (double)va[i];
                            const double qk = ((double)q[kk] + (double)q2[kk]) * qscale;
                            const double dk = (double)den[c];
                            const double ek =
                                (double)(va[i] - __half2float(__float2half_rn(va[i] * vs)) * vsi);
                            acc = fma(-2.0 * (qk - dk), ek, acc);
                            acc = fma(-ek, (double)eg[c], acc);
                            if constexpr (!PAIR) {
                                const double vhk = vk - ek;
                                acc = fma(vhk, (double)gcg[c] - 2.0 * (double)q2[kk] * qscale, acc);
                            }
                            nv[i] = (float)(vk * (qk / (dk + kDenomGuard)));
                            vmax = fmaxf(vmax, nv[i]);
                        }
                        o[hh * 2 + kq] = make_float4(nv[0], nv[1], nv[2], nv[3]);
                    }
                }
            }
            if constexpr (NQ == 2) {
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_lead(&B.dempty[b]);
            }
        }
    }
    // per-CTA share of f (residual + correction terms, fixed warp order) and max(V')
    acc = warp_sum(acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    if (lane == 0) {
        red[warp] = acc;
        vmx[warp] = vmax;
    }
    tc::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        double c = 0.0;
        float mx = 0.f;
        for (int w = 2; w < kVThreads / 32; ++w) {
            c += red[w];
            mx = fmaxf(mx, vmx[w]);
        }
        part[blockIdx.x] = c;
        atomicMax(&sc->vmax_bits, __float_as_uint(mx));   // V' >= 0: bit order = value order
    }
    if constexpr (PAIR) {
        tc::cluster_sync();   // both CTAs done with the pair's TMEM
        if (warp == 1) tc::tmem_free_pair<TM_COLS>(tmem);
    } else {
        if (warp == 1) tc::tmem_free<TM_COLS>(tmem);
    }
}

// V (m x RK fp32) -> V_h = rn(V_i 2^ev_i) fp16 row-major (the A operand of
// the residual MMAs), ev_i = scale_exp(max_k |v_ik|); RK / 4 threads per row
template <int RK>
__global__ void __launch_bounds__(256)
split_v_kernel(const float* __restrict__ V, __half* __restrict__ Vh, long long m) {
    constexpr int TPR = RK / 4;   // threads per row (16 or 32)
    const long long t = (long long)blockIdx.x * 256 + threadIdx.x;
    const long long row = t / TPR;
    const int c4 = (int)(t % TPR);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < m) v = reinterpret_cast<const float4*>(V + row * RK)[c4];
    float mx = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (row >= m) return;
    const float s = exp2f((float)scale_exp(mx));
    const __half2 a = __floats2half2_rn(v.x * s, v.y * s);
    const __half2 b = __floats2half2_rn(v.z * s, v.w * s);
    uint2 o;
    o.x = *reinterpret_cast<const uint32_t*>(&a);
    o.y = *reinterpret_cast<const uint32_t*>(&b);
    reinterpret_cast<uint2*>(Vh + row * RK)[c4] = o;
}

// RK = 128: the V' arithmetic of the V step (its rank-64 epilogue above, the
// same terms) as a pass over the [q | q2] rows the V step copied out.  Block
// (x, y) takes the 64 columns y * 64 .. of every 256-row tile x, x + gridDim.x,
// ...: that half of G_W and G_c (fp32, 64 KB) and the tile of V (coalesced
// load, 133 KB) are staged in shared memory.  Two threads per row -- lanes l
// and l + 16 of a warp -- split the rank sums by parity of the rank index and
// combine them with one shuffle per 8-column chunk; the V rows are padded to a
// stride of 2 (mod 32) words so the two halves read even / odd banks, and the
// G reads are broadcasts (two rows of G per warp load).  V' = V Q / (V G_W +
// 1e-300), the correction terms of f for V's fp16 rounding and the W_lo part
// of the residual -> part[y gridDim.x + x] (fixed order), max V' ->
// sc->vmax_bits.
constexpr int kVfinThreads = 512;
constexpr int kVfinRows = kVfinThreads / 2;
constexpr int kVfinCols = 64;
template <int RK>
constexpr uint32_t vfinish_smem() {
    return (2 * RK * kVfinCols + kVfinRows * (RK + 2)) * 4;
}
template <int RK>
__global__ void __launch_bounds__(kVfinThreads, 1)
vfinish_kernel(const float* __restrict__ Qs, const float* __restrict__ V,
               const float* __restrict__ GWf, const float* __restrict__ Gc,
               float* __restrict__ Vout, Scales* sc, long long m, double* __restrict__ part) {
    constexpr int ROWS = kVfinRows, NC = kVfinCols, VS = RK + 2;
    extern __shared__ __align__(16) float fsm[];
    float* vt = fsm + 2 * RK * NC;   // [ROWS][RK + 2]
    const int cb = (int)blockIdx.y * NC;   // first column of this block's half
    for (int i = threadIdx.x; i < RK * NC / 4; i += kVfinThreads) {
        const int l = i / (NC / 4), c4 = (i % (NC / 4)) * 4;
        reinterpret_cast<float4*>(fsm)[i] =
            __ldg(reinterpret_cast<const float4*>(GWf + (long long)l * RK + cb + c4));
        reinterpret_cast<float4*>(fsm + RK * NC)[i] =
            __ldg(reinterpret_cast<const float4*>(Gc + (long long)l * RK + cb + c4));
    }
    const uint32_t gw_s = tc::smem_u32(fsm), gc_s = tc::smem_u32(fsm + RK * NC);
    const double qscale = exp2(-(double)(sc->ex + sc->ew));
    const int lane = threadIdx.x & 31, h = lane >> 4;           // rank parity of this thread
    const int rl = (threadIdx.x >> 5) * 16 + (lane & 15);        // row in the tile
    double acc = 0.0;
    float vmax = 0.f;
    for (long long r0 = (long long)blockIdx.x * ROWS; r0 < m; r0 += (long long)gridDim.x * ROWS) {
        __syncthreads();   // the previous tile's readers are done (and G is staged)
        for (int i = threadIdx.x; i < ROWS * (RK / 4); i += kVfinThreads) {
            const int rr = i / (RK / 4), c4 = (i % (RK / 4)) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r0 + rr < m) v = __ldg(reinterpret_cast<const float4*>(V + (r0 + rr) * RK + c4));
            float* d = vt + rr * VS + c4;
            d[0] = v.x, d[1] = v.y, d[2] = v.z, d[3] = v.w;
        }
        __syncthreads();
        const long long row = r0 + rl;
        const bool valid = row < m;   // rows past m: zeros, no output (shuffles stay converged)
        const float* vrow = vt + rl * VS;
        float mx = 0.f;
#pragma unroll 8
        for (int k = h; k < RK; k += 2) mx = fmaxf(mx, fabsf(vrow[k]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const int ev = scale_exp(mx);
        const float vs = exp2f((float)ev), vsi = exp2f(-(float)ev);
        const float4* qrow = reinterpret_cast<const float4*>(Qs + (valid ? row : 0) * (2 * RK));
        float4* o = reinterpret_cast<float4*>(Vout + (valid ? row : 0) * RK);
#pragma unroll 1
        for (int c0 = 0; c0 < NC; c0 += 8) {   // this pass's 8 columns (of the half)
            // column pairs (c, c + 1) as packed fp32x2 FMAs; ranks l = 2 i + h
            float2 den2[4], eg2[4], gcg2[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) den2[c] = eg2[c] = gcg2[c] = make_float2(0.f, 0.f);
#pragma unroll 4
            for (int l = h; l < RK; l += 2) {
                const float va = vrow[l];
                const float el = va - __half2float(__float2half_rn(va * vs)) * vsi;
                const float vh = va - el;
                const float2 va2 = make_float2(va, va), el2 = make_float2(el, el),
                             vh2 = make_float2(vh, vh);
                const uint32_t off = 4u * (uint32_t)(l * NC + c0);
#pragma unroll
                for (int c4 = 0; c4 < 2; ++c4) {
                    const float4 gg = tc::lds128f(gw_s + off + 16u * c4);
                    const float4 gc = tc::lds128f(gc_s + off + 16u * c4);
                    const float2 g0 = make_float2(gg.x, gg.y), g1 = make_float2(gg.z, gg.w);
                    const float2 h0 = make_float2(gc.x, gc.y), h1 = make_float2(gc.z, gc.w);
                    den2[2 * c4] = __ffma2_rn(va2, g0, den2[2 * c4]);
                    den2[2 * c4 + 1] = __ffma2_rn(va2, g1, den2[2 * c4 + 1]);
                    eg2[2 * c4] = __ffma2_rn(el2, g0, eg2[2 * c4]);
                    eg2[2 * c4 + 1] = __ffma2_rn(el2, g1, eg2[2 * c4 + 1]);
                    gcg2[2 * c4] = __ffma2_rn(vh2, h0, gcg2[2 * c4]);
                    gcg2[2 * c4 + 1] = __ffma2_rn(vh2, h1, gcg2[2 * c4 + 1]);
                }
            }
            // the two rank halves (even + odd, in that order on both lanes)
            float den[8], eg[8], gcg[8];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float2 a[3] = {den2[c], eg2[c], gcg2[c]};
                float2 t[3];
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const float ox = __shfl_xor_sync(0xffffffffu, a[u].x, 16);
                    const float oy = __shfl_xor_sync(0xffffffffu, a[u].y, 16);
                    t[u] = h ? make_float2(ox + a[u].x, oy + a[u].y)
                             : make_float2(a[u].x + ox, a[u].y + oy);
                }
                den[2 * c] = t[0].x, den[2 * c + 1] = t[0].y;
                eg[2 * c] = t[1].x, eg[2 * c + 1] = t[1].y;
                gcg[2 * c] = t[2].x, gcg[2 * c + 1] = t[2].y;
            }
            if (!valid) continue;
            {   // this thread's 4 of the 8 columns: kq = h
                const int kq = h;
                const int k4 = (cb + c0) / 4 + kq;   // float4 index in the row
                const float4 qv = qrow[k4], q2v = qrow[RK / 4 + k4];
                const float qa[4] = {qv.x, qv.y, qv.z, qv.w};
                const float q2a[4] = {q2v.x, q2v.y, q2v.z, q2v.w};
                float nv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int c = 4 * kq + i;
                    const float vf = vrow[4 * k4 + i];
                    const double vk = (double)vf;
                    const double qk = ((double)qa[i] + (double)q2a[i]) * qscale;
                    const double dk = (double)den[c];
                    const double ek = (double)(vf - __half2float(__float2half_rn(vf * vs)) * vsi);
                    acc = fma(-2.0 * (qk - dk), ek, acc);
                    acc = fma(-ek, (double)eg[c], acc);
                    acc = fma(vk - ek, (double)gcg[c] - 2.0 * (double)q2a[i] * qscale, acc);
                    nv[i] = (float)(vk * (qk / (dk + kDenomGuard)));
                    vmax = fmaxf(vmax, nv[i]);
                }
                o[k4] = make_float4(nv[0], nv[1], nv[2], nv[3]);
            }
        }
    }
    // block share of f (fixed order) and max(V')
    __shared__ double red[kVfinThreads / 32];
    __shared__ float vmx[kVfinThreads / 32];
    acc = warp_sum(acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = acc;
        vmx[threadIdx.x >> 5] = vmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double c = 0.0;
        float mx = 0.f;
        for (int w = 0; w < kVfinThreads / 32; ++w) {
            c += red[w];
            mx = fmaxf(mx, vmx[w]);
        }
        part[blockIdx.y * gridDim.x + blockIdx.x] = c;
        atomicMax(&sc->vmax_bits, __float_as_uint(mx));   // V' >= 0: bit order = value order
    }
}

// ---------------------------------------------------------------------------
// W step.  P^T partials: item (row split s, column super-block cs of CB x 128
// columns) D[col][k] = sum_{rows of s} X[row][col] V'[row][k]; the V'^T chunk
// (fp16 hi / lo, K-major along rows) is shared by the CB column blocks of an
// item.  mX / mX2: fp16 hi / lo maps of the row-major pre-split X (m x n,
// [64 rows x 64 columns] boxes; see issue_split_stage_mn).
struct WBars {
    uint64_t xfull[XST], xempty[XST], ofull[OSTW], oempty[OSTW];
    uint64_t dfull[2], dempty[2];
};

template <int RK>
__global__ void __launch_bounds__(kWThreads, 1)
nnmf_wstep_tc(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mX2,
              const __grid_constant__ CUtensorMap mVh, const __grid_constant__ CUtensorMap mVl,
              int m, int n, int splits, int rows_per_split, float* __restrict__ wpart,
              const long long* __restrict__ skip) {
    if (skip && *skip) return;   // the engine's final pass (iteration cap): W half unused
    constexpr int CB = Tc<RK>::CB, ACC = Tc<RK>::ACC;
    constexpr uint32_t SOP = Tc<RK>::SOP;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = align1024(smem_raw);
    uint8_t* xring = base;
    uint8_t* oring = base + XST * SX;
    __shared__ WBars B;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = (int)gridDim.x, me = (int)blockIdx.x;
    const int ncb = (n + BM - 1) / BM;
    const int ncs = (ncb + CB - 1) / CB;
    const int nitems = ncs * splits;
    const int npass = nitems > me ? (nitems - 1 - me) / G + 1 : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < XST; ++s) {
            tc::mbar_init(&B.xfull[s], 1);
            tc::mbar_init(&B.xempty[s], 1);   // MMA commit
        }
        for (int s = 0; s < OSTW; ++s) {
            tc::mbar_init(&B.ofull[s], 1);
            tc::mbar_init(&B.oempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&B.dfull[b], 1);
            tc::mbar_init(&B.dempty[b], 4);
        }
        tc::fence_barrier_init();
        tc::tma_prefetch(&mX);
        tc::tma_prefetch(&mX2);
        tc::tma_prefetch(&mVh);
        tc::tma_prefetch(&mVl);
    }
    if (warp == 1) tc::tmem_alloc<TM_COLS>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    // pass p = item me + p G: (number of column blocks, K-blocks of rows, first row)
    auto pass_of = [&](int p, int& nacc, int& nkb, int& r0) {
        const int item = me + p * G, s = item / ncs, cs = item % ncs;
        r0 = s * rows_per_split;
        int r1 = r0 + rows_per_split;
        if (r1 > m) r1 = m;
        const int left = ncb - cs * CB;
        nacc = left < CB ? left : CB;
        nkb = r1 > r0 ? (r1 - r0 + BK - 1) / BK : 0;
    };
    if (warp == 0) {
        if (lane == 0) {   // TMA producer
            int xit = 0, oit = 0;
            for (int p = 0; p < npass; ++p) {
                int nacc, nkb, r0;
                pass_of(p, nacc, nkb, r0);
                const int col0 = ((me + p * G) % ncs) * CB * BM;
                for (int kb = 0; kb < nkb; ++kb, ++oit) {
                    const int os = oit % OSTW;
                    tc::mbar_wait(&B.oempty[os], ((oit / OSTW) & 1) ^ 1);
                    tc::mbar_expect_tx(&B.ofull[os], 2 * SOP);
                    tc::tma_load_2d(oring + os * 2 * SOP, &mVh, &B.ofull[os], r0 + kb * BK, 0);
                    tc::tma_load_2d(oring + os * 2 * SOP + SOP, &mVl, &B.ofull[os], r0 + kb * BK, 0);
                    for (int j = 0; j < nacc; ++j, ++xit) {
                        const int xs = xit % XST;
                        tc::mbar_wait(&B.xempty[xs], ((xit / XST) & 1) ^ 1);
                        // rows r0 + kb BK .. +64 of columns col0 + j BM .. +128
                        // (two 64-column boxes of X_hi, then of X_lo)
                        tc::mbar_expect_tx(&B.xfull[xs], SX);
                        uint8_t* xd = xring + xs * SX;
                        const int c0 = col0 + j * BM, rr = r0 + kb * BK;
                        tc::tma_load_2d(xd, &mX, &B.xfull[xs], c0, rr);
                        tc::tma_load_2d(xd + SXB, &mX, &B.xfull[xs], c0 + 64, rr);
                        tc::tma_load_2d(xd + SXH, &mX2, &B.xfull[xs], c0, rr);
                        tc::tma_load_2d(xd + SXH + SXB, &mX2, &B.xfull[xs], c0 + 64, rr);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // MMA issuer
            int xit = 0, oit = 0;
            for (int p = 0; p < npass; ++p) {
                int nacc, nkb, r0;
                pass_of(p, nacc, nkb, r0);
                const int b = p & 1;
                tc::mbar_wait(&B.dempty[b], ((p >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                for (int kb = 0; kb < nkb; ++kb, ++oit) {
                    const int os = oit % OSTW;
                    tc::mbar_wait(&B.ofull[os], (oit / OSTW) & 1);
                    for (int j = 0; j < nacc; ++j, ++xit) {
                        const int xs = xit % XST;
                        tc::mbar_wait(&B.xfull[xs], (xit / XST) & 1);
                        tc::tc_fence_after();
                        issue_split_stage_mn<RK>(tmem + (b * CB + j) * ACC, xring + xs * SX,
                                                 oring + os * 2 * SOP, kb == 0);
                        tc::mma_commit(&B.xempty[xs]);
                    }
                    tc::mma_commit(&B.oempty[os]);
                }
                tc::mma_commit(&B.dfull[b]);
            }
        }
    } else {
        // epilogue: thread = column `quarter * 32 + lane` of each block
        const int quarter = warp & 3;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        for (int p = 0; p < npass; ++p) {
            int nacc, nkb, r0;
            pass_of(p, nacc, nkb, r0);
            const int item = me + p * G, s = item / ncs, b = p & 1;
            tc::mbar_wait(&B.dfull[b], (p >> 1) & 1);
            tc::tc_fence_after();
            for (int j = 0; j < nacc; ++j) {
                const long long col = (long long)((item % ncs) * CB + j) * BM + quarter * 32 + lane;
                float4* o = reinterpret_cast<float4*>(wpart + ((long long)s * n + col) * RK);
                const uint32_t ta = tmem + (b * CB + j) * ACC + lane_off;
#pragma unroll 1
                for (int h = 0; h < RK / 32; ++h) {
                    float v[32];
                    if (nkb > 0) {
                        float v2[32];
                        tc::tmem_ld32(ta + h * 32, v);
                        tc::tmem_ld32(ta + RK + h * 32, v2);
#pragma unroll
                        for (int k = 0; k < 32; ++k) v[k] += v2[k];   // scaled units (see wreduce)
                    } else {
#pragma unroll
                        for (int k = 0; k < 32; ++k) v[k] = 0.f;
                    }
                    if (col < n) {
#pragma unroll
                        for (int k4 = 0; k4 < 8; ++k4)
                            o[h * 8 + k4] =
                                make_float4(v[4 * k4], v[4 * k4 + 1], v[4 * k4 + 2], v[4 * k4 + 3]);
                    }
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&B.dempty[b]);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free<TM_COLS>(tmem);
}

// max |x| over X -> the X scale exponent (sc->ex), cached in the workspace
// and keyed by (X, m, n, ldx): X is constant over a run, so after the first
// call this is a no-op launch.
struct XXCache {
    unsigned long long key[4];
    int ex, pad_;
    unsigned long long pkey[4];   // X the pre-split copy was made from (presplit_kernel)
};

__global__ void __launch_bounds__(512)
xmax_kernel(const float* __restrict__ X, long long ldx, long long m, long long n,
            XXCache* cache, float* __restrict__ mpart, unsigned int* counter, Scales* sc) {
    const unsigned long long k0 = reinterpret_cast<unsigned long long>(X);
    if (cache->key[0] == k0 && cache->key[1] == (unsigned long long)m &&
        cache->key[2] == (unsigned long long)n && cache->key[3] == (unsigned long long)ldx) {
        if (blockIdx.x == 0 && threadIdx.x == 0) sc->ex = cache->ex;
        return;   // uniform across the grid: every block exits, the counter is untouched
    }
    __shared__ float sf[32];
    float mx = 0.f;
    // float4 grid-stride over the m x n/4 quads (n % 8 == 0, ldx % 4 == 0,
    // X 16-byte aligned: eligible()); 8 quads in flight per thread
    const long long nq = n / 4, total = m * nq;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + 7 * stride < total; q += 8 * stride) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long t = q + u * stride, row = t / nq, c4 = t - row * nq;
            v[u] = __ldg(reinterpret_cast<const float4*>(X + row * ldx) + c4);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)),
                                 fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
    }
    for (; q < total; q += stride) {
        const long long row = q / nq, c4 = q - row * nq;
        const float4 v = __ldg(reinterpret_cast<const float4*>(X + row * ldx) + c4);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sf[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, sf[w]);
        mpart[blockIdx.x] = mx;
    }
    if (arrive_last(counter, gridDim.x) && threadIdx.x == 0) {
        float g = 0.f;
        for (unsigned int b = 0; b < gridDim.x; ++b) g = fmaxf(g, mpart[b]);
        cache->ex = scale_exp(g);
        sc->ex = cache->ex;
        cache->key[1] = (unsigned long long)m;
        cache->key[2] = (unsigned long long)n;
        cache->key[3] = (unsigned long long)ldx;
        __threadfence();
        cache->key[0] = k0;
    }
}

// Pre-split copy of X: X_hi = rn(x 2^ex), X_lo = rn(x 2^ex - X_hi) in fp16,
// row-major m x n (the V step reads [128 rows x 64 columns] boxes of it, the
// W step [64 rows x 64 columns] boxes as an MN-major operand).  Made once per
// X (keyed like the scale cache; runs after xmax_kernel, whose
// exponent it uses); later launches exit at the key check.  float4 in, 8-byte
// hi / lo out, 4 quads in flight per thread.
__device__ __forceinline__ void split_quad(float4 v, float sc, uint2& h, uint2& l) {
    split_pair(v.x * sc, v.y * sc, h.x, l.x);
    split_pair(v.z * sc, v.w * sc, h.y, l.y);
}
__global__ void __launch_bounds__(256)
presplit_kernel(const float* __restrict__ X, long long ldx, long long m, long long n,
                XXCache* cache, __half* __restrict__ Xh, __half* __restrict__ Xl,
                unsigned int* counter) {
    const unsigned long long k0 = reinterpret_cast<unsigned long long>(X);
    if (cache->pkey[0] == k0 && cache->pkey[1] == (unsigned long long)m &&
        cache->pkey[2] == (unsigned long long)n && cache->pkey[3] == (unsigned long long)ldx)
        return;   // uniform across the grid
    const float sc = exp2f((float)cache->ex);
    const long long nq = n / 4, total = m * nq;
    const long long stride = (long long)gridDim.x * blockDim.x;
    uint2* H = reinterpret_cast<uint2*>(Xh);
    uint2* L = reinterpret_cast<uint2*>(Xl);
    long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + 3 * stride < total; q += 4 * stride) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long t = q + u * stride, row = t / nq, c4 = t - row * nq;
            v[u] = __ldg(reinterpret_cast<const float4*>(X + row * ldx) + c4);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint2 h, l;
            split_quad(v[u], sc, h, l);
            H[q + u * stride] = h;   // quad t of the dense m x n copy
            L[q + u * stride] = l;
        }
    }
    for (; q < total; q += stride) {
        const long long row = q / nq, c4 = q - row * nq;
        uint2 h, l;
        split_quad(__ldg(reinterpret_cast<const float4*>(X + row * ldx) + c4), sc, h, l);
        H[q] = h;
        L[q] = l;
    }
    if (arrive_last(counter, gridDim.x) && threadIdx.x == 0) {
        cache->pkey[1] = (unsigned long long)m;
        cache->pkey[2] = (unsigned long long)n;
        cache->pkey[3] = (unsigned long long)ldx;
        __threadfence();
        cache->pkey[0] = k0;
    }
}

// Gram G = sum_c a_c a_c^T of fp32 vectors a_c of RK components (VEC_ROWS:
// A is RK x len, the vectors are columns of the row-major W; else A is len x
// RK, the rows of V).  A block computes the 64 x 64 quadrant (blockIdx.y / QN,
// blockIdx.y % QN) of G (one quadrant at RK = 64).  Products are formed in
// fp32 and summed 8 at a time in fp32, then folded into fp64 accumulators
// (4 x 4 per thread); each block writes its partial, gram_sum_kernel adds
// the partials in block order.
template <bool VEC_ROWS, int RK>
__global__ void __launch_bounds__(256)
gram32_kernel(const float* __restrict__ A, long long len, long long per_block,
              double* __restrict__ part) {
    constexpr int QN = RK / 64;
    __shared__ __align__(16) float S[QN][32][64 + 4];   // [quadrant half][vector][component]
    const int qi = (int)blockIdx.y / QN, qj = (int)blockIdx.y % QN;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    const long long c_begin = (long long)blockIdx.x * per_block;
    long long c_end = c_begin + per_block;
    if (c_end > len) c_end = len;
    for (long long c0 = c_begin; c0 < c_end; c0 += 32) {
        if (VEC_ROWS) {
            for (int idx = threadIdx.x; idx < 32 * RK; idx += 256) {
                const int a = idx >> 5, cc = idx & 31;
                S[a >> 6][cc][a & 63] = (c0 + cc < c_end) ? A[(long long)a * len + c0 + cc] : 0.f;
            }
        } else {
            for (int idx = threadIdx.x; idx < 32 * (RK / 4); idx += 256) {
                const int cc = idx / (RK / 4), a4 = (idx % (RK / 4)) * 4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (c0 + cc < c_end) v = *reinterpret_cast<const float4*>(A + (c0 + cc) * RK + a4);
                *reinterpret_cast<float4*>(&S[a4 >> 6][cc][a4 & 63]) = v;
            }
        }
        __syncthreads();
#pragma unroll
        for (int k8 = 0; k8 < 32; k8 += 8) {
            float p[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) p[i][j] = 0.f;
#pragma unroll
            for (int kk = k8; kk < k8 + 8; ++kk) {
                const float4 a = *reinterpret_cast<const float4*>(&S[qi][kk][4 * ty]);
                const float4 b = *reinterpret_cast<const float4*>(&S[qj][kk][4 * tx]);
                const float av[4] = {a.x, a.y, a.z, a.w};
                const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) p[i][j] = fmaf(av[i], bv[j], p[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += (double)p[i][j];
        }
        __syncthreads();
    }
    double* pb = part + (long long)blockIdx.x * (RK * RK);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) pb[(64 * qi + 4 * ty + i) * RK + 64 * qj + 4 * tx + j] = acc[i][j];
}

// The W-side Grams of one iteration in one pass over W (RK x len, rows are
// the vectors): G_W = W W^T as gram32_kernel<true>, plus G_c = (2 W_hi +
// W_lo) W_lo^T = 2 W_hi W_lo^T + W_lo W_lo^T of the fp16 split the V-step MMAs
// use (W_hi = rn(w 2^ew) 2^-ew, W_lo = rn(w 2^ew - W_hi 2^ew) 2^-ew, as
// split_w_kernel), the Gram of the objective's W_lo correction.  fp32
// products summed 8 at a time and folded into fp64.  A block computes the
// 64 x 64 quadrant (blockIdx.y / QN, blockIdx.y % QN) of both.  Partials:
// part[b], part[gridDim.x + b].
template <int RK>
__global__ void __launch_bounds__(256)
gram3_kernel(const float* __restrict__ A, long long len, long long per_block,
             const Scales* sc, double* __restrict__ part) {
    constexpr int QN = RK / 64;
    // rows of quadrant row qi (w, 2 w_hi + w_lo) and of quadrant column qj (w, w_lo)
    __shared__ __align__(16) float Sa[32][64 + 4], Sc[32][64 + 4], Sb[32][64 + 4], Sl[32][64 + 4];
    const int qi = (int)blockIdx.y / QN, qj = (int)blockIdx.y % QN;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const float s = exp2f((float)sc->ew), si = exp2f(-(float)sc->ew);
    double acc[2][4][4];
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[g][i][j] = 0.0;
    const long long c_begin = (long long)blockIdx.x * per_block;
    long long c_end = c_begin + per_block;
    if (c_end > len) c_end = len;
    for (long long c0 = c_begin; c0 < c_end; c0 += 32) {
        for (int idx = threadIdx.x; idx < 2 * 32 * 64; idx += 256) {
            const int side = idx >> 11, a = (idx >> 5) & 63, cc = idx & 31;
            const int row = 64 * (side ? qj : qi) + a;
            const float w = (c0 + cc < c_end) ? A[(long long)row * len + c0 + cc] : 0.f;
            const float hi = __half2float(__float2half_rn(w * s));
            const float lo = __half2float(__float2half_rn(w * s - hi));
            if (side) {
                Sb[cc][a] = w;
                Sl[cc][a] = lo * si;
            } else {
                Sa[cc][a] = w;
                Sc[cc][a] = 2.f * (hi * si) + lo * si;
            }
        }
        __syncthreads();
#pragma unroll
        for (int k8 = 0; k8 < 32; k8 += 8) {
            float p[2][4][4];
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) p[g][i][j] = 0.f;
#pragma unroll
            for (int kk = k8; kk < k8 + 8; ++kk) {
                const float4 a = *reinterpret_cast<const float4*>(&Sa[kk][4 * ty]);
                const float4 b = *reinterpret_cast<const float4*>(&Sb[kk][4 * tx]);
                const float4 ac = *reinterpret_cast<const float4*>(&Sc[kk][4 * ty]);
                const float4 bl = *reinterpret_cast<const float4*>(&Sl[kk][4 * tx]);
                const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
                const float acv[4] = {ac.x, ac.y, ac.z, ac.w};
                const float blv[4] = {bl.x, bl.y, bl.z, bl.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        p[0][i][j] = fmaf(av[i], bv[j], p[0][i][j]);
                        p[1][i][j] = fmaf(acv[i], blv[j], p[1][i][j]);
                    }
            }
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[g][i][j] += (double)p[g][i][j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        double* pb = part + ((long long)g * gridDim.x + blockIdx.x) * (RK * RK);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                pb[(64 * qi + 4 * ty + i) * RK + 64 * qj + 4 * tx + j] = acc[g][i][j];
    }
}

// out[e] = sum_b part[b][e] in block order: 8 groups of 128 threads take
// interleaved partials, combined in group order (deterministic)
template <int RK>
__global__ void __launch_bounds__(1024)
gram_sum_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out,
                float* __restrict__ outf, const long long* __restrict__ skip = nullptr) {
    if (skip && *skip) return;
    __shared__ double sm[8][128];
    const int o = blockIdx.x * 128 + (threadIdx.x & 127), g = threadIdx.x >> 7;
    double s = 0.0;
#pragma unroll 4
    for (int b = g; b < nparts; b += 8) s += part[(long long)b * (RK * RK) + o];
    sm[g][threadIdx.x & 127] = s;
    __syncthreads();
    if (g == 0) {
        double t = sm[0][threadIdx.x];
#pragma unroll
        for (int k = 1; k < 8; ++k) t += sm[k][threadIdx.x];
        out[o] = t;
        if (outf) outf[o] = (float)t;   // fp32 copy (G_W for the V-step epilogue)
    }
}

// ---------------------------------------------------------------------------
// max |W| -> sc->ew (last block), and reset the V' maximum for this iteration
__global__ void __launch_bounds__(1024)
wmax_kernel(const float* __restrict__ W, long long len, float* __restrict__ mpart,
            unsigned int* counter, Scales* sc) {
    __shared__ float sf[32];
    float mx = 0.f;
    const long long len4 = len / 4;   // W rows are n % 8 == 0 long (eligible()): len % 4 == 0
    const float4* W4 = reinterpret_cast<const float4*>(W);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < len4;
         t += (long long)gridDim.x * blockDim.x) {
        const float4 v = W4[t];
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sf[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < 32; ++w) mx = fmaxf(mx, sf[w]);
        mpart[blockIdx.x] = mx;
    }
    if (arrive_last(counter, gridDim.x) && threadIdx.x == 0) {
        float g = 0.f;
        for (unsigned int b = 0; b < gridDim.x; ++b) g = fmaxf(g, mpart[b]);
        sc->ew = scale_exp(g);
        sc->wmax_bits = __float_as_uint(g);
        sc->vmax_bits = 0u;
    }
}

// W (64 x n fp32) -> W_hi / W_lo (64 x n fp16), scaled by 2^ew
__global__ void split_w_kernel(const float* __restrict__ W, __half* __restrict__ Wh,
                               __half* __restrict__ Wl, long long len, const Scales* sc) {
    const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (t >= len) return;
    const float s = exp2f((float)sc->ew);
    uint32_t h, l;
    split_pair(W[t] * s, (t + 1 < len ? W[t + 1] : 0.f) * s, h, l);
    if (t + 1 < len) {
        *reinterpret_cast<uint32_t*>(Wh + t) = h;
        *reinterpret_cast<uint32_t*>(Wl + t) = l;
    } else {
        Wh[t] = __ushort_as_half((unsigned short)(h & 0xffffu));
        Wl[t] = __ushort_as_half((unsigned short)(l & 0xffffu));
    }
}

// V' (m x 64 fp32) -> V'^T hi / lo (64 x m fp16), scaled by 2^ev where ev
// comes from max(V') of the V step, AND this block's share of the Gram
// V'^T V' (one read of V' for both).  A block takes the 128-row tiles
// blockIdx.x, + gridDim.x, ...: each tile is loaded once (float4) into a
// transposed copy T (for the 16-byte chunks (8 rows) of both fp16 outputs)
// and a row-major copy S (for the Gram: thread (ty, tx) owns the 4 x 4 block
// (4 ty, 4 tx), fp32 products of 8 rows folded into fp64, as gram32_kernel);
// the block's partial goes to gpart[blockIdx.x] (gram_sum_kernel adds them).
// RK = 128: the transposed split only (GRAM = false; the Gram of V' is
// gram32_kernel's, one more read of V').
constexpr int kVprepBlocks = 2 * kNumSMs;
template <int RK, bool GRAM>
constexpr uint32_t vprep_smem() {
    return (RK * (128 + 4) + (GRAM ? 128 * (RK + 4) : 0)) * 4;
}
template <int RK, bool GRAM>
__global__ void __launch_bounds__(256)
vprep_gram_kernel(const float* __restrict__ V, __half* __restrict__ Vth,
                  __half* __restrict__ Vtl, long long m, Scales* sc, double* __restrict__ gpart,
                  const long long* __restrict__ skip) {
    static_assert(!GRAM || RK == 64, "the fused Gram is rank-64 only");
    constexpr int R = RK;
    if (skip && *skip) return;
    extern __shared__ __align__(16) float vsm[];
    float(*T)[128 + 4] = reinterpret_cast<float(*)[128 + 4]>(vsm);
    float(*S)[R + 4] = reinterpret_cast<float(*)[R + 4]>(vsm + R * (128 + 4));
    const int ev = scale_exp(__uint_as_float(sc->vmax_bits));
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->ev = ev;
    const float s = exp2f((float)ev);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    const long long ntiles = (m + 127) / 128;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long r0 = tile * 128;
        for (int i = threadIdx.x; i < 128 * (R / 4); i += 256) {
            const int rr = i / (R / 4), k4 = (i % (R / 4)) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r0 + rr < m) v = *reinterpret_cast<const float4*>(V + (r0 + rr) * R + k4);
            if (GRAM) *reinterpret_cast<float4*>(&S[rr][k4]) = v;
            T[k4][rr] = v.x * s;
            T[k4 + 1][rr] = v.y * s;
            T[k4 + 2][rr] = v.z * s;
            T[k4 + 3][rr] = v.w * s;
        }
        __syncthreads();
        // chunk c of rank k: rows r0 + 8c .. r0 + 8c + 7 (16 bytes of fp16)
        for (int e = threadIdx.x; e < R * 16; e += 256) {
            const int k = e / 16, c = e % 16;
            const long long row = r0 + 8 * c;
            if (row >= m) continue;
            uint32_t h[4], l[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                split_pair(T[k][8 * c + 2 * q], T[k][8 * c + 2 * q + 1], h[q], l[q]);
            if (row + 8 <= m) {
                *reinterpret_cast<uint4*>(Vth + (long long)k * m + row) = make_uint4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<uint4*>(Vtl + (long long)k * m + row) = make_uint4(l[0], l[1], l[2], l[3]);
            } else {
                for (int q = 0; q < 8 && row + q < m; ++q) {
                    const uint32_t hw = h[q / 2] >> (16 * (q & 1)), lw = l[q / 2] >> (16 * (q & 1));
                    Vth[(long long)k * m + row + q] = __ushort_as_half((unsigned short)(hw & 0xffffu));
                    Vtl[(long long)k * m + row + q] = __ushort_as_half((unsigned short)(lw & 0xffffu));
                }
            }
        }
        // Gram share of the tile's 128 rows (rows past m are zero)
#pragma unroll 1
        for (int k8 = 0; k8 < (GRAM ? 128 : 0); k8 += 8) {
            float p[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) p[i][j] = 0.f;
#pragma unroll
            for (int kk = k8; kk < k8 + 8; ++kk) {
                const float4 a = *reinterpret_cast<const float4*>(&S[kk][4 * ty]);
                const float4 b = *reinterpret_cast<const float4*>(&S[kk][4 * tx]);
                const float av[4] = {a.x, a.y, a.z, a.w};
                const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) p[i][j] = fmaf(av[i], bv[j], p[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += (double)p[i][j];
        }
        __syncthreads();
    }
    if (!GRAM) return;
    double* pb = gpart + (long long)blockIdx.x * (R * R);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) pb[(4 * ty + i) * R + 4 * tx + j] = acc[i][j];
}

// red[k n + j] = sum_s wpart[s][j][k] (fixed split order); a block owns 32
// columns j: coalesced reads of the [32 j][RK k] slab of every split, fp64
// sums, transposed through shared memory for coalesced writes
template <int RK>
__global__ void __launch_bounds__(256)
wreduce_tc_kernel(const float* __restrict__ wpart, int splits, long long n,
                  double* __restrict__ red, const Scales* sc, const long long* __restrict__ skip) {
    constexpr int R = RK, NQ8 = RK / 8;   // slab elements per thread
    if (skip && *skip) return;
    __shared__ double T[R][32 + 1];
    // partials are in the scaled units of the split products: X 2^ex, V' 2^ev
    const double pscale = exp2(-(double)(sc->ex + sc->ev));
    const long long j0 = (long long)blockIdx.x * 32;
    double acc[NQ8];
#pragma unroll
    for (int q = 0; q < NQ8; ++q) acc[q] = 0.0;
    // element e = q * 256 + tid of the slab: j = e / RK, k = e % RK
    for (int sp = 0; sp < splits; ++sp) {
        const float* src = wpart + ((long long)sp * n + j0) * R;
#pragma unroll
        for (int q = 0; q < NQ8; ++q) {
            const int e = q * 256 + threadIdx.x;
            if (j0 + e / R < n) acc[q] += (double)src[e];
        }
    }
#pragma unroll
    for (int q = 0; q < NQ8; ++q) {
        const int e = q * 256 + threadIdx.x;
        T[e % R][e / R] = acc[q] * pscale;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * 32; e += 256) {
        const int k = e / 32, jj = e % 32;
        if (j0 + jj < n) red[(long long)k * n + j0 + jj] = T[k][jj];
    }
}

// f-partial (this rank's rows) = sum of the V step's per-CTA shares in CTA order
__global__ void tc_objective_kernel(const double* __restrict__ part, int nparts,
                                    double* __restrict__ out) {
    __shared__ double sc[32];
    const double f = block_sum_array(part, nparts, sc);
    if (threadIdx.x == 0) *out = f;
}

// rank r < RK on the rank-RK kernels: V (m x r) -> V_RK (m x RK, zero
// columns r..RK-1) and back; the rank-RK reduction buffer's G block -> r x r
__global__ void pad_cols_kernel(const float* __restrict__ src, int r, int rk, long long rows,
                                float* __restrict__ dst) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * rk) return;
    const long long i = t / rk;
    const int k = (int)(t % rk);
    dst[t] = k < r ? src[i * r + k] : 0.f;
}
__global__ void unpad_cols_kernel(const float* __restrict__ src, int r, int rk, long long rows,
                                  float* __restrict__ dst) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * r) return;
    dst[t] = src[(t / r) * rk + t % r];
}
__global__ void unpad_gram_kernel(const double* __restrict__ gk, const double* __restrict__ fk,
                                  int r, int rk, double* __restrict__ g, double* __restrict__ f) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < r * r) g[t] = gk[(t / r) * rk + t % r];
    if (t == 0) *f = *fk;
}

// the rank tile of rank r: 64 for ranks 17..64, 128 for 65..128
inline int rank_tile(long long r) { return r <= 64 ? 64 : 128; }

struct TcPlan {
    int vgrid, wgrid, splits, rows_per_split;
    bool vpair;   // V step as CTA pairs (cta_group::2)
};

// MMK_TC_PAIR=1 runs the rank-64 V step as CTA pairs (cta_group::2; same
// results to rounding -- Q gains the X_lo.W_lo product -- and 8 % slower at
// C4, see the V-step notes above); single CTAs are the default
bool vstep_pair_enabled() {
    static const bool on = [] {
        const char* e = getenv("MMK_TC_PAIR");
        return e && e[0] == '1';
    }();
    return on;
}

TcPlan tc_plan(long long m, long long n, int rk) {
    TcPlan P;
    const int ntiles = (int)((m + BM - 1) / BM);
    P.vpair = rk == 64 && vstep_pair_enabled() && ntiles >= 2;
    if (P.vpair) {
        const int units = (ntiles + 1) / 2;
        P.vgrid = 2 * (units < kNumSMs / 2 ? units : kNumSMs / 2);
    } else {
        P.vgrid = ntiles < kNumSMs ? ntiles : kNumSMs;
    }
    const int cb = rk == 64 ? Tc<64>::CB : Tc<128>::CB;
    const int ncb = (int)((n + BM - 1) / BM);
    const int ncs = (ncb + cb - 1) / cb;
    // split count minimising (wave quantisation loss) + (split-K partial
    // traffic: S fp32 partials of n x rk written and read back, relative to
    // one pass over X); rows per split >= 4 K-blocks
    const int max_splits = (int)((m + 4 * BK - 1) / (4 * BK));
    int best = 1;
    double best_cost = 1e300;
    for (int S = 1; S <= max_splits && S <= 4 * kNumSMs; ++S) {
        const int items = ncs * S;
        const int waves = (items + kNumSMs - 1) / kNumSMs;
        const double eff = (double)items / ((double)waves * kNumSMs);
        const double partial = 2.0 * S * (double)n * rk * 4.0 / ((double)m * n * 4.0);
        const double cost = 1.0 / eff + partial;
        if (cost < best_cost - 1e-12) {
            best_cost = cost;
            best = S;
        }
    }
    long long rps = (m + best - 1) / best;
    rps = (rps + BK - 1) / BK * BK;
    P.rows_per_split = (int)rps;
    P.splits = (int)((m + rps - 1) / rps);
    const int items = ncs * P.splits;
    P.wgrid = items < kNumSMs ? items : kNumSMs;
    return P;
}

constexpr int kGramBlocks = 2 * kNumSMs;

// G = Gram of A (see gram32_kernel) into out (fp64 RK x RK)
template <int RK>
void gram32(const float* A, long long len, bool vec_rows, double* gpart, double* out,
            cudaStream_t st, float* outf = nullptr) {
    long long per = (len + kGramBlocks - 1) / kGramBlocks;
    per = (per + 31) / 32 * 32;
    const int blocks = (int)((len + per - 1) / per);
    const dim3 grid(blocks, (RK / 64) * (RK / 64));
    if (vec_rows)
        MMK_LAUNCH("nnmf_gram32", st,
                   (gram32_kernel<true, RK><<<grid, 256, 0, st>>>(A, len, per, gpart)));
    else
        MMK_LAUNCH("nnmf_gram32", st,
                   (gram32_kernel<false, RK><<<grid, 256, 0, st>>>(A, len, per, gpart)));
    MMK_LAUNCH("nnmf_gram_sum", st,
               (gram_sum_kernel<RK><<<RK * RK / 128, 1024, 0, st>>>(gpart, blocks, out, outf)));
}

// G_W and G_c = 2 W_hi W_lo^T + W_lo W_lo^T (gram3_kernel) -> GW (fp64), GWf, GcF
template <int RK>
void gram3(const float* W, long long len, const Scales* sc, double* gpart, double* GW,
           float* GWf, double* G64, float* GcF, cudaStream_t st) {
    // one wave at RK = 64: the kernel holds two 4 x 4 fp64 accumulator sets
    long long per = (len + kNumSMs - 1) / kNumSMs;
    per = (per + 31) / 32 * 32;
    const int blocks = (int)((len + per - 1) / per);
    const dim3 grid(blocks, (RK / 64) * (RK / 64));
    MMK_LAUNCH("nnmf_gram32", st,
               (gram3_kernel<RK><<<grid, 256, 0, st>>>(W, len, per, sc, gpart)));
    MMK_LAUNCH("nnmf_gram_sum", st,
               (gram_sum_kernel<RK><<<RK * RK / 128, 1024, 0, st>>>(gpart, blocks, GW, GWf)));
    MMK_LAUNCH("nnmf_gram_sum", st,
               (gram_sum_kernel<RK><<<RK * RK / 128, 1024, 0, st>>>(
                   gpart + (long long)blocks * RK * RK, blocks, G64, GcF)));
}

struct TcWs {
    __half *Wh, *Wl, *Vth, *Vtl, *Vh;
    __half *Xh, *Xl;   // pre-split X (row-major)
    float *wpart, *mpart, *GWf;   // GWf: G_W in fp32 (V-step epilogue)
    float* GcF;                   // G_c = 2 W_hi W_lo^T + W_lo W_lo^T in fp32 (V-step epilogue)
    float* Qs;                    // RK = 128: the V step's Q rows [q | q2] (m x 2 RK)
    double* G64;                  // its fp64 sum
    double *part, *gpart;
    XXCache* xx;
    Scales* sc;
    unsigned int* counter;   // [0] xmax, [1] wmax, [2] presplit
};

inline char* c_base(void* p) { return reinterpret_cast<char*>(p); }

// The per-X part first (pre-split copy, scale cache, counters: what
// prepare_x touches, independent of the rank tile), then the rank-RK part
size_t tc_layout(long long m, long long n, int rk, void* base, TcWs* L) {
    const TcPlan P = tc_plan(m, n, rk);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    const size_t xe = (size_t)m * n;
    size_t oXh = take(2 * xe), oXl = take(2 * xe);
    size_t oP = take(8 * (size_t)kNumSMs * 3);   // V-step partials (+ vfinish's at RK = 128)
    size_t oM = take(4 * (size_t)kNumSMs * 8);   // [0, 4*148) xmax, then wmax
    size_t oC = take(sizeof(XXCache) + sizeof(Scales) + 64);
    size_t oWh = take(2 * (size_t)rk * n), oWl = take(2 * (size_t)rk * n);
    size_t oVh = take(2 * (size_t)rk * m), oVl = take(2 * (size_t)rk * m);
    size_t oVr = take(2 * (size_t)rk * m);
    size_t oWp = take(4 * (size_t)P.splits * n * rk);
    size_t oGP = take(8 * (size_t)rk * rk * kGramBlocks * 2);   // gram3: two Grams
    size_t oGF = take(4 * (size_t)rk * rk);
    size_t oGS = take(4 * (size_t)rk * rk), oG64 = take(8 * (size_t)rk * rk);
    size_t oQs = take(rk == 128 ? 4 * (size_t)m * 2 * rk : 0);
    if (base && L) {
        char* c = c_base(base);
        L->Xh = (__half*)(c + oXh);
        L->Xl = (__half*)(c + oXl);
        L->mpart = (float*)(c + oM);
        L->xx = (XXCache*)(c + oC);
        L->sc = (Scales*)(c + oC + sizeof(XXCache));
        L->counter = (unsigned int*)(c + oC + sizeof(XXCache) + sizeof(Scales));
        L->Wh = (__half*)(c + oWh);
        L->Wl = (__half*)(c + oWl);
        L->Vth = (__half*)(c + oVh);
        L->Vtl = (__half*)(c + oVl);
        L->Vh = (__half*)(c + oVr);
        L->wpart = (float*)(c + oWp);
        L->part = (double*)(c + oP);
        L->gpart = (double*)(c + oGP);
        L->GWf = (float*)(c + oGF);
        L->GcF = (float*)(c + oGS);
        L->G64 = (double*)(c + oG64);
        L->Qs = (float*)(c + oQs);
    }
    return off;
}

thread_local bool t_x_prepared = false;   // set while an engine captures its loop
// set while an engine captures its loop: ctl[MMK_CTL_LAST], read by the W-half
// kernels at run time (they exit when the pass only needs its objective)
thread_local const long long* t_last_flag = nullptr;

}  // namespace

namespace mmk_tc {

// The tensor-core path needs the pre-split copy of X (4 bytes per element)
// next to X itself; shapes whose copy would pass 96 GiB take the SIMT path.
bool shape_ok(int dtype, long long m, long long n, long long r) {
    // ranks 17..128: ranks below the rank tile (64 or 128) run on its kernels
    // with V and W zero-padded (exact: a zero component stays zero and adds
    // nothing)
    if (dtype != MMK_F32 || r < 17 || r > 128) return false;
    if ((n & 7) || (m & 7) || m < BM || n < BM) return false;
    if (m > 0x7fffffffLL || n > 0x7fffffffLL) return false;
    // the pre-split copy, plus at the 128-rank tile the V step's Q rows
    // (m x 256 fp32)
    const double q_rows = r > 64 ? 1024.0 * (double)m : 0.0;
    return 4.0 * (double)m * (double)n + q_rows <= 96.0 * (1ull << 30);
}

bool eligible(int dtype, long long m, long long n, long long r, long long ldx, const void* X) {
    if (!shape_ok(dtype, m, n, r)) return false;
    // 16-byte rows for the pre-split pass (ldx % 4) and a 16-byte aligned X
    if ((ldx & 3) || (reinterpret_cast<uintptr_t>(X) & 15)) return false;
    const char* env = getenv("MMK_NNMF_TC");
    if (env && env[0] == '0') return false;
    return true;
}

// rank < RK: the zero-padded operands after the rank-RK region
struct PadWs {
    float *Vp, *Vpo, *Wp;
    double *redp, *GWp;
};
size_t pad_layout(long long m, long long n, int rk, void* base, PadWs* L) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    const size_t oV = take(4 * (size_t)m * rk), oVo = take(4 * (size_t)m * rk);
    const size_t oW = take(4 * (size_t)rk * n);
    const size_t oRed = take(8 * ((size_t)rk * n + rk * rk + 2)), oG = take(8 * (size_t)rk * rk);
    if (base && L) {
        char* c = reinterpret_cast<char*>(base);
        L->Vp = (float*)(c + oV);
        L->Vpo = (float*)(c + oVo);
        L->Wp = (float*)(c + oW);
        L->redp = (double*)(c + oRed);
        L->GWp = (double*)(c + oG);
    }
    return off;
}

size_t ws_bytes(long long m, long long n, long long r) {
    const int rk = rank_tile(r);
    const size_t core = (tc_layout(m, n, rk, nullptr, nullptr) + 255) & ~size_t(255);
    return core + (r < rk ? pad_layout(m, n, rk, nullptr, nullptr) : 0);
}

void set_x_prepared(bool on) { t_x_prepared = on; }
void set_last_flag(const int64_t* p) { t_last_flag = reinterpret_cast<const long long*>(p); }
const long long* last_flag() { return t_last_flag; }

// [begin, end) of the pre-split copy of X inside the tensor-core workspace:
// it is always written (presplit_kernel, keyed in the zeroed header) before
// it is read, so a workspace need not be zero-filled there
void presplit_span(long long m, long long n, size_t* begin, size_t* end) {
    TcWs L;
    char* const base = reinterpret_cast<char*>(uintptr_t(1) << 20);   // any non-null base
    tc_layout(m, n, 64, base, &L);   // the per-X part does not depend on the rank tile
    *begin = (size_t)(reinterpret_cast<char*>(L.Xh) - base);
    *end = *begin + 2 * 2 * (size_t)m * (size_t)n;   // X_hi, X_lo (adjacent, 256-aligned)
}

int prepare_x(const float* X, long long ldx, long long m, long long n, void* tcws,
              cudaStream_t st) {
    TcWs L;
    tc_layout(m, n, 64, tcws, &L);   // per-X part only (rank-independent offsets)
    MMK_LAUNCH("nnmf_xmax_cached", st,
               (xmax_kernel<<<4 * kNumSMs, 512, 0, st>>>(X, ldx, m, n, L.xx, L.mpart, L.counter,
                                                         L.sc)));
    MMK_LAUNCH("nnmf_presplit_cached", st,
               (presplit_kernel<<<8 * kNumSMs, 256, 0, st>>>(X, ldx, m, n, L.xx, L.Xh, L.Xl,
                                                             L.counter + 2)));
    MMK_CHECK_LAUNCH("nnmf_prepare_x");
    return MMK_OK;
}

// Phase A of one iteration on the tensor cores at the rank tile RK; writes
// V_out and red = [P | G_V' | f-partial].
template <int RK>
static int iter_a_rk(const float* X, long long ldx, const float* V, const float* W,
                     float* V_out, long long m, long long n, void* tcws, double* GW, double* red,
                     cudaStream_t st) {
    using C = Tc<RK>;
    constexpr bool VGRAM = RK == 64;   // V'^T V' fused into vprep_gram_kernel
    TcWs L;
    tc_layout(m, n, RK, tcws, &L);
    const TcPlan P = tc_plan(m, n, RK);
    if (mmk_host::first_on_device(reinterpret_cast<const void*>(nnmf_wstep_tc<RK>))) {
        cudaFuncSetAttribute(nnmf_vstep_tc<false, RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::SMEM_V);
        if constexpr (RK == 64)
            cudaFuncSetAttribute(nnmf_vstep_tc<true, 64>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_V2);
        cudaFuncSetAttribute(nnmf_wstep_tc<RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::SMEM_W);
        cudaFuncSetAttribute(vprep_gram_kernel<RK, VGRAM>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, vprep_smem<RK, VGRAM>());
        if constexpr (RK == 128)
            cudaFuncSetAttribute(vfinish_kernel<RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 vfinish_smem<RK>());
    }
    CUtensorMap mX, mX2, mWh, mWl, mVr, mXt, mXt2, mVh, mVl;
    int rc;
    if ((rc = mmk_host::make_map_f16(&mX, L.Xh, m, n, n, BM))) return rc;
    if ((rc = mmk_host::make_map_f16(&mX2, L.Xl, m, n, n, BM))) return rc;
    // the W step reads the same row-major copy in [64 rows x 64 columns] boxes
    if ((rc = mmk_host::make_map_f16(&mXt, L.Xh, m, n, n, BK))) return rc;
    if ((rc = mmk_host::make_map_f16(&mXt2, L.Xl, m, n, n, BK))) return rc;
    if ((rc = mmk_host::make_map_f16(&mVr, L.Vh, m, RK, RK, BM))) return rc;
    if ((rc = mmk_host::make_map_f16(&mWh, L.Wh, RK, n, n, RK))) return rc;
    if ((rc = mmk_host::make_map_f16(&mWl, L.Wl, RK, n, n, RK))) return rc;
    if ((rc = mmk_host::make_map_f16(&mVh, L.Vth, RK, m, m, RK))) return rc;
    if ((rc = mmk_host::make_map_f16(&mVl, L.Vtl, RK, m, m, RK))) return rc;
    const long long rn = (long long)RK * n;
    if (!t_x_prepared) {
        int prc = prepare_x(X, ldx, m, n, tcws, st);
        if (prc) return prc;
    }
    MMK_LAUNCH("nnmf_wmax", st,
               (wmax_kernel<<<kNumSMs, 1024, 0, st>>>(W, rn, L.mpart + 4 * kNumSMs,
                                                     L.counter + 1, L.sc)));
    MMK_LAUNCH("nnmf_split_w", st,
               (split_w_kernel<<<ceil_div((rn + 1) / 2, 256), 256, 0, st>>>(W, L.Wh, L.Wl, rn,
                                                                            L.sc)));
    gram3<RK>(W, n, L.sc, L.gpart, GW, L.GWf, L.G64, L.GcF, st);
    MMK_LAUNCH("nnmf_split_v", st,
               (split_v_kernel<RK><<<ceil_div(m * (RK / 4), 256), 256, 0, st>>>(V, L.Vh, m)));
    if constexpr (RK == 64) {
        if (P.vpair) {
            // clusters of 2 CTAs (one TPC): the pair's MMAs run as cta_group::2
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(P.vgrid);
            cfg.blockDim = dim3(kVThreads);
            cfg.dynamicSmemBytes = SMEM_V2;
            cfg.stream = st;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            MMK_LAUNCH("nnmf_vstep_tc", st,
                       (void)cudaLaunchKernelEx(&cfg, nnmf_vstep_tc<true, 64>, mX, mX2, mWh, mWl,
                                                mVr, V, (const float*)L.GWf, (const float*)L.GcF,
                                                V_out, L.sc, (int)m, (int)n, L.part,
                                                (float*)nullptr));
        }
    }
    if (!P.vpair) {
        MMK_LAUNCH("nnmf_vstep_tc", st,
                   (nnmf_vstep_tc<false, RK><<<P.vgrid, kVThreads, C::SMEM_V, st>>>(
                       mX, mX2, mWh, mWl, mVr, V, L.GWf, L.GcF, V_out, L.sc, (int)m, (int)n,
                       L.part, L.Qs)));
    }
    MMK_CHECK_LAUNCH("nnmf_vstep_tc");
    int nparts = P.vgrid;
    if constexpr (RK == 128) {   // the V' arithmetic (G_W, G_c in shared memory)
        MMK_LAUNCH("nnmf_vfinish_tc", st,
                   (vfinish_kernel<RK><<<dim3(kNumSMs, RK / kVfinCols), kVfinThreads,
                                         vfinish_smem<RK>(), st>>>(
                       L.Qs, V, L.GWf, L.GcF, V_out, L.sc, m, L.part + P.vgrid)));
        MMK_CHECK_LAUNCH("nnmf_vfinish_tc");
        nparts += kNumSMs * (RK / kVfinCols);
    }
    MMK_LAUNCH("nnmf_objective_tc", st,
               (tc_objective_kernel<<<1, 256, 0, st>>>(L.part, nparts,
                                                        red + rn + (long long)RK * RK)));
    {   // V'^T hi / lo for the W step and the Gram V'^T V' -> red (one read of V' at RK = 64)
        const int vb = (int)(ceil_div(m, 128) < kVprepBlocks ? ceil_div(m, 128) : kVprepBlocks);
        MMK_LAUNCH("nnmf_vprep_gram", st,
                   (vprep_gram_kernel<RK, VGRAM><<<vb, 256, vprep_smem<RK, VGRAM>(), st>>>(
                       V_out, L.Vth, L.Vtl, m, L.sc, L.gpart, t_last_flag)));
        if constexpr (VGRAM)
            MMK_LAUNCH("nnmf_gram_sum", st,
                       (gram_sum_kernel<RK><<<RK * RK / 128, 1024, 0, st>>>(
                           L.gpart, vb, red + rn, nullptr, t_last_flag)));
        else
            gram32<RK>(V_out, m, false, L.gpart, red + rn, st);
    }
    MMK_LAUNCH("nnmf_wstep_tc", st,
               (nnmf_wstep_tc<RK><<<P.wgrid, kWThreads, C::SMEM_W, st>>>(
                   mXt, mXt2, mVh, mVl, (int)m, (int)n, P.splits, P.rows_per_split, L.wpart,
                   t_last_flag)));
    MMK_CHECK_LAUNCH("nnmf_wstep_tc");
    MMK_LAUNCH("nnmf_wreduce_tc", st,
               (wreduce_tc_kernel<RK><<<ceil_div(n, 32), 256, 0, st>>>(L.wpart, P.splits, n, red,
                                                                        L.sc, t_last_flag)));
    MMK_CHECK_LAUNCH("nnmf_tc_iter_a");
    return MMK_OK;
}

// Phase A of one iteration on the tensor cores (any rank 17..128)
int iter_a(const float* X, long long ldx, const float* V, const float* W, float* V_out,
           long long m, long long n, long long r, void* tcws, double* GW, double* red,
           cudaStream_t st) {
    const int rk = rank_tile(r);
    if (r == rk)
        return rk == 64 ? iter_a_rk<64>(X, ldx, V, W, V_out, m, n, tcws, GW, red, st)
                        : iter_a_rk<128>(X, ldx, V, W, V_out, m, n, tcws, GW, red, st);
    PadWs Pd;
    pad_layout(m, n, rk,
               reinterpret_cast<char*>(tcws) +
                   ((tc_layout(m, n, rk, nullptr, nullptr) + 255) & ~size_t(255)),
               &Pd);
    MMK_LAUNCH("nnmf_pad_v", st,
               (pad_cols_kernel<<<ceil_div(m * rk, 256), 256, 0, st>>>(V, (int)r, rk, m, Pd.Vp)));
    cudaMemcpyAsync(Pd.Wp, W, sizeof(float) * r * n, cudaMemcpyDeviceToDevice, st);
    cudaMemsetAsync(Pd.Wp + r * n, 0, sizeof(float) * (rk - r) * n, st);
    int rc = rk == 64
                 ? iter_a_rk<64>(X, ldx, Pd.Vp, Pd.Wp, Pd.Vpo, m, n, tcws, Pd.GWp, Pd.redp, st)
                 : iter_a_rk<128>(X, ldx, Pd.Vp, Pd.Wp, Pd.Vpo, m, n, tcws, Pd.GWp, Pd.redp, st);
    if (rc) return rc;
    MMK_LAUNCH("nnmf_unpad_v", st,
               (unpad_cols_kernel<<<ceil_div(m * r, 256), 256, 0, st>>>(Pd.Vpo, (int)r, rk, m,
                                                                         V_out)));
    // [P (r n) | G (r r) | f]: the first r rows of P are the padded P's
    cudaMemcpyAsync(red, Pd.redp, sizeof(double) * r * n, cudaMemcpyDeviceToDevice, st);
    MMK_LAUNCH("nnmf_unpad_gram", st,
               (unpad_gram_kernel<<<ceil_div(r * r, 256), 256, 0, st>>>(
                   Pd.redp + (long long)rk * n, Pd.redp + (long long)rk * n + rk * rk, (int)r, rk,
                   red + r * n, red + r * n + r * r)));
    (void)GW;
    MMK_CHECK_LAUNCH("nnmf_tc_iter_a_padded");
    return MMK_OK;
}

}  // namespace mmk_tc

#ifdef MMK_TC_TRACE
extern "C" int mmk_tc_trace_read(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, g_tctrace, sizeof(g_tctrace));
}
#endif
