// nnmf_tc.cu -- tensor-core (tcgen05, kind::tf32, 3xTF32) path of the NNMF
// MM iteration for large fp32 problems with rank 64 (BASELINE config 4).
//
// The two contractions with X are the whole cost (4mnr of
// 5.5e11 flops); both run on the 5th-gen tensor cores in split-precision
// "3xTF32": every fp32 operand is split into tf32 hi + lo (hi = round-to-
// nearest tf32, lo = exact remainder) and a*b ~ hi*hi + hi*lo + lo*hi,
// accumulated in fp32 in TMEM -- fp32-faithful products.
// The O((m+n) r^2) Gram side stays in fp64 on the CUDA cores.
//
//   nnmf_vstep_tc  (persistent, one CTA per SM, 10 warps)
//     warp 0   TMA producer: X tile [128 rows x 32 cols] + W_hi/W_lo chunks
//              [64 x 32] per stage (128-byte swizzle, K-major), 4 stages
//     warps 2-5 split X in shared memory into hi (in place) / lo, and
//              accumulate sum x^2 (fp64) for the objective
//     warp 1   one thread issues 12 tcgen05.mma (M128 N64 K8) per stage into
//              a double-buffered fp32 accumulator Q = X W^T in TMEM
//     warps 6-9 epilogue: tcgen05.ld Q rows, V' = V * Q / (V G_W + 1e-300),
//              <V, Q> (fp64); writes V' and its tf32 split for the W step
//   nnmf_wstep_tc  P^T = X^T V' (M = 128 columns of X, N = 64, K = rows),
//              split-K over row ranges; both operands MN-major (32-byte-atom
//              128B swizzle, the only MN-major tf32 layout); per-split
//              partials reduced in fixed order -> deterministic.
//
// Objective f(V, W) = sum x^2 - 2 <V, X W^T> + <V^T V, W W^T> in fp64: every
// term is a by-product of the pass (no extra X traffic).  Its conditioning
// is ||X||^2 / f times the 3xTF32 accumulation error;
// tests/test_nnmf_tc_gpu.py checks it against the explicit residual.
//
// HBM roofline: each kernel streams X once (m n 4 bytes) -> two passes per
// iteration; tensor work 3 x 2mnr per kernel.
#include "mmk_common.cuh"
#include "nnmf_tc.h"
#include "tc_common.cuh"

namespace {

using namespace mmk;

constexpr int R = 64;            // rank of the tensor-core path (UMMA N)
constexpr int BM = 128;          // UMMA M: rows of X (V step) / columns of X (W step)
constexpr int BK = 32;           // K per stage: one 128-byte row of fp32
constexpr int NCONV = 8;         // split warps: groups of 4 take X stages round-robin
constexpr int NGROUP = NCONV / 4;
constexpr int kThreads = 32 * (2 + NCONV + 4);   // TMA, MMA, split x8, epilogue x4
constexpr uint32_t SX = BM * BK * 4;        // 16 KB  raw X tile (the hi operand)
constexpr uint32_t SOP = R * BK * 4;        //  8 KB  W (or V') chunk hi; same again for lo
constexpr int XST = 8;                      // X ring (128 KB in flight per SM)
constexpr int OST = 4;                      // operand (W / V' chunk) ring
constexpr uint32_t SMEM = XST * SX + OST * 2 * SOP + 1024;
constexpr int NA = 4;                       // TMEM A-operand buffers [X_hi | X_lo] (64 cols)
constexpr int ACC = 2 * R;                  // accumulator columns: [X.Wh | X.Wl] (N = 128)
constexpr int TMAX = 2;                     // accumulators per pass (V step: row tiles)
constexpr int CB = 2;                       // W step: 128-column blocks per item
constexpr int TM_COLS = 512;
constexpr uint32_t TM_A = TMAX * ACC;       // A buffers after the accumulators

// experiment switches (MMK_TC_DBG, timing studies only; results are wrong
// when set): 1 skip the lo MMAs, 2 skip the tf32 split, 4 skip all MMAs
__constant__ int c_dbg = 0;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// 3xTF32 split of an X value: hi = x with its 13 low mantissa bits cleared
// (what the tensor core reads of a tf32 operand), lo = x - hi exactly.
__device__ __forceinline__ void tf32_hilo(float x, float& hi, float& lo) {
    hi = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
    lo = x - hi;
}

struct Bars {
    uint64_t xfull[XST], xempty[XST], ofull[OST], oempty[OST], afull[NA], aempty[NA];
    uint64_t dfull, dempty;
};

__device__ __forceinline__ void init_bars(Bars& B) {
    for (int s = 0; s < XST; ++s) {
        tc::mbar_init(&B.xfull[s], 1);
        tc::mbar_init(&B.xempty[s], 128);   // released by the split warps
    }
    for (int s = 0; s < OST; ++s) {
        tc::mbar_init(&B.ofull[s], 1);
        tc::mbar_init(&B.oempty[s], 1);
    }
    for (int b = 0; b < NA; ++b) {
        tc::mbar_init(&B.afull[b], 128);
        tc::mbar_init(&B.aempty[b], 1);
    }
    tc::mbar_init(&B.dfull, 1);
    tc::mbar_init(&B.dempty, 128);
    tc::fence_barrier_init();
}

// One stage of 3xTF32, both MMAs with A from TMEM (buffer a = [X_hi | X_lo],
// 32 + 32 columns, written by the split warps) so the tensor core reads only
// the B operand from shared memory.  The operand chunk holds [B_hi ; B_lo]
// stacked along N (64 + 64 rows): per K-step a TS MMA with N = 128 gives
// D[:, 0:64] += X_hi.B_hi and D[:, 64:128] += X_hi.B_lo, and a TS MMA with
// N = 64 adds X_lo.B_hi into D[:, 0:64].  The epilogue sums the two halves:
// X_hi B_hi + X_hi B_lo + X_lo B_hi.
template <bool MN>
__device__ __forceinline__ void issue_stage(uint32_t d, uint32_t a, const uint8_t* bhl,
                                            bool first) {
    constexpr uint32_t id_lo = tc::idesc_tf32(BM, R, 0, MN ? 1 : 0);
    constexpr uint32_t id_hi = tc::idesc_tf32(BM, ACC, 0, MN ? 1 : 0);
    // descriptors advance by their 16-byte start-address field only
    const uint64_t db0 = MN ? tc::sdesc_sw128_32b(bhl, 4096, 512) : tc::sdesc_sw128(bhl, 16, 1024);
    constexpr uint64_t step = MN ? (1024 >> 4) : (32 >> 4);
    const int dbg = c_dbg;
    if (dbg & 4) return;
#pragma unroll
    for (int ks = 0; ks < BK / 8; ++ks) {
        const uint32_t acc = (first && ks == 0) ? 0u : 1u;
        tc::mma_tf32_ts(d, a + ks * 8, db0 + ks * step, id_hi, acc);
        if (!(dbg & 1)) tc::mma_tf32_ts(d, a + 32 + ks * 8, db0 + ks * step, id_lo, 1);
    }
}

// Work of one CTA pass: `nacc` accumulators (row tiles or column blocks),
// `nkb` K-blocks; stage (kb, j) streams X block j of K-block kb while the
// operand chunk of kb is shared by all j.
struct Pass {
    int nacc, nkb;
};

// An X stage from shared memory into registers: V step (MN = false) reads
// row `lane` of the 128B-swizzled K-major tile; W step (MN = true) reads
// column `lane` of box `quarter` of the 32-byte-atom swizzled MN-major tile.
template <bool MN>
__device__ __forceinline__ void read_stage(const uint8_t* xs, int quarter, int lane, float* x) {
    if (!MN) {
        const int row = quarter * 32 + lane;
        const float4* rp = reinterpret_cast<const float4*>(xs + row * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const float4 t = rp[c ^ (row & 7)];
            x[4 * c] = t.x;
            x[4 * c + 1] = t.y;
            x[4 * c + 2] = t.z;
            x[4 * c + 3] = t.w;
        }
    } else {
        const uint8_t* bx = xs + quarter * 4096 + (lane & 7) * 4;
#pragma unroll
        for (int k = 0; k < 32; ++k)
            x[k] = *reinterpret_cast<const float*>(bx + k * 128 + (((lane >> 3) ^ (k & 3)) << 5));
    }
}

// tf32 hi / lo of the 32 values into TMEM columns [a, a + 32) / [a + 32, a + 64)
__device__ __forceinline__ void store_hilo(float* x, uint32_t a_addr) {
    float lo[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) tf32_hilo(x[k], x[k], lo[k]);
    tc::tmem_st32(a_addr, x);
    tc::tmem_st32(a_addr + 32, lo);
}

// ---------------------------------------------------------------------------
// The pipeline shared by both steps.  Role functions get (pass index p, j)
// and must agree on the iteration order: for p: for kb: [operand], for j: [X].
// trace (debug): CTA 0 records clock64 per X stage for the first kTrace stages:
// [0] TMA issued, [1] split start (data landed), [2] split done, [3] MMA
// start (operands ready), [4] MMAs issued + committed
constexpr int kTrace = 256;
__device__ __forceinline__ void trace_at(unsigned long long* tr, int what, int xit) {
    if (tr && blockIdx.x == 0 && xit < kTrace) tr[what * kTrace + xit] = clock64();
}

template <bool MN, class PassOf, class LoadX, class LoadOp, class Epi>
__device__ __forceinline__ void run_pipeline(uint8_t* base, Bars& B, uint32_t tmem, int npass,
                                             const PassOf& pass_of, const LoadX& load_x,
                                             const LoadOp& load_op, const Epi& epilogue,
                                             unsigned long long* tr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* xring = base;
    uint8_t* oring = base + XST * SX;
    if (warp == 0) {
        if (lane == 0) {
            int xit = 0, oit = 0;
            for (int p = 0; p < npass; ++p) {
                const Pass P = pass_of(p);
                for (int kb = 0; kb < P.nkb; ++kb, ++oit) {
                    const int os = oit % OST;
                    tc::mbar_wait(&B.oempty[os], ((oit / OST) & 1) ^ 1);
                    tc::mbar_expect_tx(&B.ofull[os], 2 * SOP);
                    load_op(p, kb, oring + os * 2 * SOP, &B.ofull[os]);
                    for (int j = 0; j < P.nacc; ++j, ++xit) {
                        const int xs = xit % XST;
                        tc::mbar_wait(&B.xempty[xs], ((xit / XST) & 1) ^ 1);
                        tc::mbar_expect_tx(&B.xfull[xs], SX);
                        load_x(p, kb, j, xring + xs * SX, &B.xfull[xs]);
                        trace_at(tr, 0, xit);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int xit = 0, oit = 0;
            for (int p = 0; p < npass; ++p) {
                const Pass P = pass_of(p);
                if (p > 0) tc::mbar_wait(&B.dempty, (p - 1) & 1);
                tc::tc_fence_after();
                for (int kb = 0; kb < P.nkb; ++kb, ++oit) {
                    const int os = oit % OST;
                    tc::mbar_wait(&B.ofull[os], (oit / OST) & 1);
                    const uint8_t* ob = oring + os * 2 * SOP;
                    for (int j = 0; j < P.nacc; ++j, ++xit) {
                        const int ab = xit % NA;
                        tc::mbar_wait(&B.afull[ab], (xit / NA) & 1);
                        trace_at(tr, 3, xit);
                        tc::tc_fence_after();
                        issue_stage<MN>(tmem + j * ACC, tmem + TM_A + ab * 64, ob, kb == 0);
                        tc::mma_commit(&B.aempty[ab]);   // A buffer ab free once these finish
                        trace_at(tr, 4, xit);
                    }
                    tc::mma_commit(&B.oempty[os]);
                }
                tc::mma_commit(&B.dfull);
            }
        }
    } else if (warp < 2 + NCONV) {
        const int g = (warp - 2) >> 2, quarter = warp & 3;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        int xit = 0;
        for (int p = 0; p < npass; ++p) {
            const Pass P = pass_of(p);
            for (int kb = 0; kb < P.nkb; ++kb) {
                for (int j = 0; j < P.nacc; ++j, ++xit) {
                    if (xit % NGROUP != g) continue;
                    const int xs = xit % XST, ab = xit % NA;
                    tc::mbar_wait(&B.xfull[xs], (xit / XST) & 1);
                    if (quarter == 0 && lane == 0) trace_at(tr, 1, xit);
                    float x[32];
                    read_stage<MN>(xring + xs * SX, quarter, lane, x);
                    // the values are in registers (consumed below): release the slot
                    tc::mbar_arrive(&B.xempty[xs]);
                    // A buffer ab was last read by the MMAs of stage xit - NA
                    if (xit >= NA) tc::mbar_wait(&B.aempty[ab], ((xit / NA) - 1) & 1);
                    tc::tc_fence_after();
                    if (!(c_dbg & 2)) store_hilo(x, tmem + TM_A + ab * 64 + lane_off);
                    tc::tmem_st_wait();
                    tc::tc_fence_before();
                    tc::mbar_arrive(&B.afull[ab]);
                    if (quarter == 0 && lane == 0) trace_at(tr, 2, xit);
                }
            }
        }
    } else {
        const int quarter = warp & 3;
        for (int p = 0; p < npass; ++p) {
            const Pass P = pass_of(p);
            tc::mbar_wait(&B.dfull, p & 1);
            tc::tc_fence_after();
            for (int j = 0; j < P.nacc; ++j)
                epilogue(p, j, quarter, lane,
                         tmem + j * ACC + ((uint32_t)(quarter * 32) << 16), P.nkb > 0);
            tc::tc_fence_before();
            tc::mbar_arrive(&B.dempty);
        }
    }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
nnmf_vstep_tc(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mWh,
              const __grid_constant__ CUtensorMap mWl, const float* __restrict__ V,
              const float* __restrict__ DEN, float* __restrict__ Vout, float* __restrict__ Vhi,
              float* __restrict__ Vlo, int m, int n, double* __restrict__ part,
              unsigned long long* tr) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = align1024(smem_raw);
    __shared__ Bars B;
    __shared__ uint32_t tmem_base;
    __shared__ double red[kThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (m + BM - 1) / BM, nk = (n + BK - 1) / BK;
    const int mine = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int npass = (mine + TMAX - 1) / TMAX;
    if (threadIdx.x == 0) {
        init_bars(B);
        tc::tma_prefetch(&mX);
        tc::tma_prefetch(&mWh);
        tc::tma_prefetch(&mWl);
    }
    if (warp == 1) tc::tmem_alloc<TM_COLS>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    double acc = 0.0;
    auto tile_of = [&](int p, int j) { return (int)blockIdx.x + (p * TMAX + j) * (int)gridDim.x; };
    auto pass_of = [&](int p) {
        const int left = mine - p * TMAX;
        return Pass{left < TMAX ? left : TMAX, nk};
    };
    auto load_op = [&](int, int kb, uint8_t* dst, uint64_t* bar) {
        tc::tma_load_2d(dst, &mWh, bar, kb * BK, 0);
        tc::tma_load_2d(dst + SOP, &mWl, bar, kb * BK, 0);
    };
    auto load_x = [&](int p, int kb, int j, uint8_t* dst, uint64_t* bar) {
        tc::tma_load_2d(dst, &mX, bar, kb * BK, tile_of(p, j) * BM);
    };
    auto epilogue = [&](int p, int j, int quarter, int ln, uint32_t ta, bool) {
        const long long row = (long long)tile_of(p, j) * BM + quarter * 32 + ln;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            float q[32], q2[32];
            tc::tmem_ld32(ta + h * 32, q);
            tc::tmem_ld32(ta + R + h * 32, q2);
#pragma unroll
            for (int i = 0; i < 32; ++i) q[i] += q2[i];
            if (row >= m) continue;
            const float4* v4 = reinterpret_cast<const float4*>(V + row * R + h * 32);
            const float4* d4 = reinterpret_cast<const float4*>(DEN + row * R + h * 32);
            float4* o = reinterpret_cast<float4*>(Vout + row * R + h * 32);
            float4* oh = reinterpret_cast<float4*>(Vhi + row * R + h * 32);
            float4* ol = reinterpret_cast<float4*>(Vlo + row * R + h * 32);
#pragma unroll
            for (int k4 = 0; k4 < 8; ++k4) {
                const float4 vv = v4[k4], dd = d4[k4];
                const float va[4] = {vv.x, vv.y, vv.z, vv.w};
                const float da[4] = {dd.x, dd.y, dd.z, dd.w};
                float nv[4], hh[4], ll[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double vk = (double)va[i];
                    const double qk = (double)q[4 * k4 + i];
                    acc = fma(vk, qk, acc);
                    nv[i] = (float)(vk * (qk / ((double)da[i] + kDenomGuard)));
                    tc::split_tf32(nv[i], hh[i], ll[i]);
                }
                o[k4] = make_float4(nv[0], nv[1], nv[2], nv[3]);
                oh[k4] = make_float4(hh[0], hh[1], hh[2], hh[3]);
                ol[k4] = make_float4(ll[0], ll[1], ll[2], ll[3]);
            }
        }
    };
    run_pipeline<false>(base, B, tmem, npass, pass_of, load_x, load_op, epilogue, tr);
    // per-CTA partial <V, Q> (epilogue warps)
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    tc::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        double c = 0.0;
        for (int w = 2 + NCONV; w < kThreads / 32; ++w) c += red[w];
        part[blockIdx.x] = c;
    }
    if (warp == 1) tc::tmem_free<TM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// P^T partials: item (row split s, column super-block cs of CB x 128 columns)
// D[col][k] = sum_{rows of s} X[row][col] V'[row][k]; V' chunks are shared
// by the CB column blocks of an item.  X tiles arrive MN-major (4 boxes of
// 32 rows x 32 columns, 32-byte-atom swizzle) and serve as the hi operand.
__global__ void __launch_bounds__(kThreads, 1)
nnmf_wstep_tc(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mVh,
              const __grid_constant__ CUtensorMap mVl, int m, int n, int splits,
              int rows_per_split, float* __restrict__ wpart, unsigned long long* tr) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = align1024(smem_raw);
    __shared__ Bars B;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5;
    const int ncb = (n + BM - 1) / BM;
    const int ncs = (ncb + CB - 1) / CB;
    const int nitems = ncs * splits;
    const int npass = nitems > (int)blockIdx.x ? (nitems - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (threadIdx.x == 0) {
        init_bars(B);
        tc::tma_prefetch(&mX);
        tc::tma_prefetch(&mVh);
        tc::tma_prefetch(&mVl);
    }
    if (warp == 1) tc::tmem_alloc<TM_COLS>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    auto item_of = [&](int p) { return (int)blockIdx.x + p * (int)gridDim.x; };
    auto pass_of = [&](int p) {
        const int item = item_of(p), s = item / ncs, cs = item % ncs;
        const int r0 = s * rows_per_split;
        int r1 = r0 + rows_per_split;
        if (r1 > m) r1 = m;
        const int left = ncb - cs * CB;
        return Pass{left < CB ? left : CB, r1 > r0 ? (r1 - r0 + BK - 1) / BK : 0};
    };
    auto load_op = [&](int p, int kb, uint8_t* dst, uint64_t* bar) {
        const int row = (item_of(p) / ncs) * rows_per_split + kb * BK;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            tc::tma_load_2d(dst + jj * 4096, &mVh, bar, 32 * jj, row);
            tc::tma_load_2d(dst + SOP + jj * 4096, &mVl, bar, 32 * jj, row);
        }
    };
    auto load_x = [&](int p, int kb, int j, uint8_t* dst, uint64_t* bar) {
        const int item = item_of(p);
        const int row = (item / ncs) * rows_per_split + kb * BK;
        const int col0 = ((item % ncs) * CB + j) * BM;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) tc::tma_load_2d(dst + jj * 4096, &mX, bar, col0 + 32 * jj, row);
    };
    auto epilogue = [&](int p, int j, int quarter, int ln, uint32_t ta, bool any) {
        const int item = item_of(p), s = item / ncs;
        const long long col = (long long)((item % ncs) * CB + j) * BM + quarter * 32 + ln;
        float4* o = reinterpret_cast<float4*>(wpart + ((long long)s * n + col) * R);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            float v[32];
            if (any) {
                float v2[32];
                tc::tmem_ld32(ta + h * 32, v);
                tc::tmem_ld32(ta + R + h * 32, v2);
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] += v2[k];
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = 0.f;
            }
            if (col < n) {
#pragma unroll
                for (int k4 = 0; k4 < 8; ++k4)
                    o[h * 8 + k4] = make_float4(v[4 * k4], v[4 * k4 + 1], v[4 * k4 + 2], v[4 * k4 + 3]);
            }
        }
    };
    run_pipeline<true>(base, B, tmem, npass, pass_of, load_x, load_op, epilogue, tr);
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free<TM_COLS>(tmem);
}

// sum of x^2 over X, cached in the workspace and keyed by (X, m, n, ldx):
// X is constant over a run, so after the first call this is a no-op launch.
struct XXCache {
    double xx;
    unsigned long long key[4];
};

__global__ void sumsq_kernel(const float* __restrict__ X, long long ldx, long long m, long long n,
                             XXCache* cache, double* __restrict__ part, unsigned int* counter) {
    const unsigned long long k0 = reinterpret_cast<unsigned long long>(X);
    if (cache->key[0] == k0 && cache->key[1] == (unsigned long long)m &&
        cache->key[2] == (unsigned long long)n && cache->key[3] == (unsigned long long)ldx)
        return;   // uniform across the grid: every block exits, the counter is untouched
    __shared__ double sc[32];
    double s = 0.0;
    for (long long i = blockIdx.x; i < m; i += gridDim.x) {
        const float* row = X + i * ldx;
        for (long long j = threadIdx.x; j < n; j += blockDim.x) {
            const double v = row[j];
            s = fma(v, v, s);
        }
    }
    s = block_sum(s, sc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(part, gridDim.x, sc);
        if (threadIdx.x == 0) {
            cache->xx = tot;
            cache->key[1] = (unsigned long long)m;
            cache->key[2] = (unsigned long long)n;
            cache->key[3] = (unsigned long long)ldx;
            __threadfence();
            cache->key[0] = k0;
        }
    }
}

// DEN = V G_W (the V-step denominator without its guard): fp32 FFMA with
// G_W rounded to fp32 -- the denominator only needs fp32 accuracy (SURVEY.md
// 7.3-1: Gram-side products in fp32 keep raw V within 5e-6 of fp64).  A block
// computes 64 rows x 64 columns with 4 x 4 register tiles per thread.
constexpr int VGW_SMEM = 2 * R * (64 + 4) * 4;
__global__ void __launch_bounds__(256)
vgw_kernel(const float* __restrict__ V, const double* __restrict__ GW, float* __restrict__ DEN,
           long long m) {
    extern __shared__ float vgw_smem[];
    float(*G)[64 + 4] = reinterpret_cast<float(*)[64 + 4]>(vgw_smem);
    float(*Vt)[64 + 4] = reinterpret_cast<float(*)[64 + 4]>(vgw_smem + R * (64 + 4));
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const long long r0 = (long long)blockIdx.x * 64;
    for (int i = threadIdx.x; i < R * R; i += 256) G[i / R][i % R] = (float)GW[i];
    for (int i = threadIdx.x; i < 16 * R; i += 256) {
        const int rr = i / 16, l4 = (i % 16) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r0 + rr < m) v = *reinterpret_cast<const float4*>(V + (r0 + rr) * R + l4);
        Vt[l4][rr] = v.x;
        Vt[l4 + 1][rr] = v.y;
        Vt[l4 + 2][rr] = v.z;
        Vt[l4 + 3][rr] = v.w;
    }
    __syncthreads();
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 8
    for (int l = 0; l < R; ++l) {
        const float4 a = *reinterpret_cast<const float4*>(&Vt[l][4 * ty]);
        const float4 b = *reinterpret_cast<const float4*>(&G[l][4 * tx]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const long long row = r0 + 4 * ty + i;
        if (row < m)
            *reinterpret_cast<float4*>(DEN + row * R + 4 * tx) =
                make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
}

// Rank-64 Gram G = sum_c a_c a_c^T of fp32 vectors a_c (VEC_ROWS: A is
// 64 x len, the vectors are columns of the row-major W; else A is len x 64,
// the rows of V).  Products are formed in fp32 and summed 8 at a time in
// fp32, then folded into fp64 accumulators (4 x 4 per thread); each block
// writes its partial, gram_sum_kernel adds the partials in block order.
template <bool VEC_ROWS>
__global__ void __launch_bounds__(256)
gram32_kernel(const float* __restrict__ A, long long len, long long per_block,
              double* __restrict__ part) {
    __shared__ __align__(16) float S[32][64 + 4];
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
            for (int idx = threadIdx.x; idx < 32 * 64; idx += 256) {
                const int a = idx >> 5, cc = idx & 31;
                S[cc][a] = (c0 + cc < c_end) ? A[(long long)a * len + c0 + cc] : 0.f;
            }
        } else {
            for (int idx = threadIdx.x; idx < 32 * 16; idx += 256) {
                const int cc = idx >> 4, a4 = (idx & 15) * 4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (c0 + cc < c_end) v = *reinterpret_cast<const float4*>(A + (c0 + cc) * 64 + a4);
                *reinterpret_cast<float4*>(&S[cc][a4]) = v;
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
    double* pb = part + (long long)blockIdx.x * (R * R);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) pb[(4 * ty + i) * R + 4 * tx + j] = acc[i][j];
}

// out[e] = sum_b part[b][e] in block order: 8 groups of 128 threads take
// interleaved partials, combined in group order (deterministic)
__global__ void __launch_bounds__(1024)
gram_sum_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out) {
    __shared__ double sm[8][128];
    const int o = blockIdx.x * 128 + (threadIdx.x & 127), g = threadIdx.x >> 7;
    double s = 0.0;
#pragma unroll 4
    for (int b = g; b < nparts; b += 8) s += part[(long long)b * (R * R) + o];
    sm[g][threadIdx.x & 127] = s;
    __syncthreads();
    if (g == 0) {
        double t = sm[0][threadIdx.x];
#pragma unroll
        for (int k = 1; k < 8; ++k) t += sm[k][threadIdx.x];
        out[o] = t;
    }
}

// ---------------------------------------------------------------------------
__global__ void split_w_kernel(const float* __restrict__ W, float* __restrict__ Wh,
                               float* __restrict__ Wl, long long len) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= len) return;
    float h, l;
    tc::split_tf32(W[t], h, l);
    Wh[t] = h;
    Wl[t] = l;
}

// red[k n + j] = sum_s wpart[s][j][k] (fixed split order); a block owns 32
// columns j: coalesced reads of the [32 j][64 k] slab of every split, fp64
// sums, transposed through shared memory for coalesced writes
__global__ void __launch_bounds__(256)
wreduce_tc_kernel(const float* __restrict__ wpart, int splits, long long n,
                  double* __restrict__ red) {
    __shared__ double T[R][32 + 1];
    const long long j0 = (long long)blockIdx.x * 32;
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    // element e = q * 256 + tid of the slab: j = e / 64, k = e % 64
    for (int sp = 0; sp < splits; ++sp) {
        const float* src = wpart + ((long long)sp * n + j0) * R;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = q * 256 + threadIdx.x;
            if (j0 + e / R < n) acc[q] += (double)src[e];
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int e = q * 256 + threadIdx.x;
        T[e % R][e / R] = acc[q];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * 32; e += 256) {
        const int k = e / 32, jj = e % 32;
        if (j0 + jj < n) red[(long long)k * n + j0 + jj] = T[k][jj];
    }
}

// f-partial = sum x^2 - 2 <V, Q> + <G_V, G_W> (all over this rank's rows)
__global__ void tc_objective_kernel(const double* __restrict__ part, int nparts,
                                    const XXCache* __restrict__ cache,
                                    const double* __restrict__ GV, const double* __restrict__ GW,
                                    double* __restrict__ out) {
    __shared__ double sc[32];
    double cr = 0.0, gg = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) cr += part[i];
    for (int i = threadIdx.x; i < R * R; i += blockDim.x) gg = fma(GV[i], GW[i], gg);
    cr = block_sum(cr, sc);
    gg = block_sum(gg, sc);
    if (threadIdx.x == 0) *out = cache->xx - 2.0 * cr + gg;
}

struct TcPlan {
    int vgrid, wgrid, splits, rows_per_split;
};

TcPlan tc_plan(long long m, long long n) {
    TcPlan P;
    const int ntiles = (int)((m + BM - 1) / BM);
    P.vgrid = ntiles < kNumSMs ? ntiles : kNumSMs;
    const int ncb = (int)((n + BM - 1) / BM);
    const int ncs = (ncb + CB - 1) / CB;
    // smallest split count whose item count fills whole waves of SMs
    // (ncs * S a multiple of 148 when possible), rows per split >= 4 K-blocks
    const int max_splits = (int)((m + 4 * BK - 1) / (4 * BK));
    int best = 1;
    double best_eff = 0.0;
    for (int S = 1; S <= max_splits && S <= 4 * kNumSMs; ++S) {
        const int items = ncs * S;
        const int waves = (items + kNumSMs - 1) / kNumSMs;
        const double eff = (double)items / ((double)waves * kNumSMs);
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = S;
        }
        if (eff > 0.999) break;
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

// G = Gram of A (see gram32_kernel) into out (fp64 64 x 64)
void gram32(const float* A, long long len, bool vec_rows, double* gpart, double* out,
            cudaStream_t st) {
    long long per = (len + kGramBlocks - 1) / kGramBlocks;
    per = (per + 31) / 32 * 32;
    const int blocks = (int)((len + per - 1) / per);
    if (vec_rows)
        MMK_LAUNCH("nnmf_gram32", st,
                   (gram32_kernel<true><<<blocks, 256, 0, st>>>(A, len, per, gpart)));
    else
        MMK_LAUNCH("nnmf_gram32", st,
                   (gram32_kernel<false><<<blocks, 256, 0, st>>>(A, len, per, gpart)));
    MMK_LAUNCH("nnmf_gram_sum", st,
               (gram_sum_kernel<<<R * R / 128, 1024, 0, st>>>(gpart, blocks, out)));
}

struct TcWs {
    float *Wh, *Wl, *Vhi, *Vlo, *wpart, *DEN;
    double *GVn, *part, *sqpart, *gpart;
    XXCache* xx;
    unsigned int* counter;
};

inline char* c_base(void* p) { return reinterpret_cast<char*>(p); }

size_t tc_layout(long long m, long long n, void* base, TcWs* L) {
    const TcPlan P = tc_plan(m, n);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    size_t oWh = take(4 * (size_t)R * n), oWl = take(4 * (size_t)R * n);
    size_t oVh = take(4 * (size_t)R * m), oVl = take(4 * (size_t)R * m);
    size_t oD = take(4 * (size_t)R * m);
    size_t oWp = take(4 * (size_t)P.splits * n * R);
    size_t oG = take(8 * (size_t)R * R);
    size_t oP = take(16 * (size_t)kNumSMs);
    size_t oS = take(8 * (size_t)kNumSMs * 4);
    size_t oC = take(sizeof(XXCache) + 64);
    size_t oGP = take(8 * (size_t)R * R * kGramBlocks);
    if (base && L) {
        L->sqpart = (double*)(c_base(base) + oS);
        L->xx = (XXCache*)(c_base(base) + oC);
        L->counter = (unsigned int*)(c_base(base) + oC + sizeof(XXCache));
        char* c = reinterpret_cast<char*>(base);
        L->Wh = (float*)(c + oWh);
        L->Wl = (float*)(c + oWl);
        L->Vhi = (float*)(c + oVh);
        L->Vlo = (float*)(c + oVl);
        L->DEN = (float*)(c + oD);
        L->wpart = (float*)(c + oWp);
        L->GVn = (double*)(c + oG);
        L->part = (double*)(c + oP);
        L->gpart = (double*)(c + oGP);
    }
    return off;
}

bool g_attr_done = false;
unsigned long long* g_trace_v = nullptr;   // debug: mmk_tc_set_trace
unsigned long long* g_trace_w = nullptr;

}  // namespace

namespace mmk_tc {

bool eligible(int dtype, long long m, long long n, long long r, long long ldx, const void* X) {
    if (dtype != MMK_F32 || r != R) return false;
    if ((n & 3) || (ldx & 3) || (reinterpret_cast<uintptr_t>(X) & 15)) return false;
    if (m < BM || n < BM) return false;
    if (m > 0x7fffffffLL || n > 0x7fffffffLL) return false;
    const char* env = getenv("MMK_NNMF_TC");
    if (env && env[0] == '0') return false;
    return true;
}

size_t ws_bytes(long long m, long long n) { return tc_layout(m, n, nullptr, nullptr); }

// Phase A of one iteration on the tensor cores.  `gram` callbacks run the
// CUDA-core fp64 Gram kernels of nnmf.cu.  Writes V_out and red = [P | G_V | f].
int iter_a(const float* X, long long ldx, const float* V, const float* W, float* V_out,
           long long m, long long n, void* tcws, double* GW, double* red,
           const GramFn& gram_w, const GramFn& gram_v_into, cudaStream_t st) {
    TcWs L;
    tc_layout(m, n, tcws, &L);
    const TcPlan P = tc_plan(m, n);
    if (!g_attr_done) {
        const char* dbg = getenv("MMK_TC_DBG");
        if (dbg) {
            const int v = atoi(dbg);
            cudaMemcpyToSymbol(c_dbg, &v, sizeof(int));
        }
        cudaFuncSetAttribute(nnmf_vstep_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        cudaFuncSetAttribute(nnmf_wstep_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        cudaFuncSetAttribute(vgw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, VGW_SMEM);
        g_attr_done = true;
    }
    CUtensorMap mX, mWh, mWl, mXt, mVh, mVl;
    int rc;
    if ((rc = mmk_host::make_map_f32(&mX, X, m, n, ldx, BM))) return rc;
    if ((rc = mmk_host::make_map_f32(&mWh, L.Wh, R, n, n, R))) return rc;
    if ((rc = mmk_host::make_map_f32(&mWl, L.Wl, R, n, n, R))) return rc;
    if ((rc = mmk_host::make_map_f32(&mXt, X, m, n, ldx, BK, 32))) return rc;
    if ((rc = mmk_host::make_map_f32(&mVh, L.Vhi, m, R, R, BK, 32))) return rc;
    if ((rc = mmk_host::make_map_f32(&mVl, L.Vlo, m, R, R, BK, 32))) return rc;
    const long long rn = (long long)R * n;
    MMK_LAUNCH("nnmf_split_w", st,
               (split_w_kernel<<<ceil_div(rn, 256), 256, 0, st>>>(W, L.Wh, L.Wl, rn)));
    (void)gram_w;
    (void)gram_v_into;
    gram32(W, n, true, L.gpart, GW, st);
    gram32(V, m, false, L.gpart, L.GVn, st);
    MMK_LAUNCH("nnmf_sumsq_cached", st,
               (sumsq_kernel<<<4 * kNumSMs, 256, 0, st>>>(X, ldx, m, n, L.xx, L.sqpart,
                                                           L.counter)));
    MMK_LAUNCH("nnmf_vgw", st,
               (vgw_kernel<<<ceil_div(m, 64), 256, VGW_SMEM, st>>>(V, GW, L.DEN, m)));
    MMK_LAUNCH("nnmf_vstep_tc", st,
               (nnmf_vstep_tc<<<P.vgrid, kThreads, SMEM, st>>>(mX, mWh, mWl, V, L.DEN, V_out, L.Vhi,
                                                                L.Vlo, (int)m, (int)n, L.part,
                                                                g_trace_v)));
    MMK_CHECK_LAUNCH("nnmf_vstep_tc");
    MMK_LAUNCH("nnmf_objective_tc", st,
               (tc_objective_kernel<<<1, 256, 0, st>>>(L.part, P.vgrid, L.xx, L.GVn, GW,
                                                        red + rn + (long long)R * R)));
    gram32(V_out, m, false, L.gpart, red + rn, st);
    MMK_LAUNCH("nnmf_wstep_tc", st,
               (nnmf_wstep_tc<<<P.wgrid, kThreads, SMEM, st>>>(mXt, mVh, mVl, (int)m, (int)n,
                                                                P.splits, P.rows_per_split,
                                                                L.wpart, g_trace_w)));
    MMK_CHECK_LAUNCH("nnmf_wstep_tc");
    MMK_LAUNCH("nnmf_wreduce_tc", st,
               (wreduce_tc_kernel<<<ceil_div(n, 32), 256, 0, st>>>(L.wpart, P.splits, n, red)));
    MMK_CHECK_LAUNCH("nnmf_tc_iter_a");
    return MMK_OK;
}

}  // namespace mmk_tc

// Debug hook: per-stage pipeline timestamps of CTA 0 (5 x 256 uint64 each, or
// NULL to disable).  Not part of the solver ABI contract.
extern "C" int mmk_tc_set_trace(unsigned long long* vstep, unsigned long long* wstep) {
    g_trace_v = vstep;
    g_trace_w = wstep;
    return 0;
}
