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
constexpr int STAGES = 6;
constexpr int kThreads = 320;    // 10 warps: TMA, MMA, 4 split, 4 epilogue
constexpr uint32_t SX = BM * BK * 4;        // 16 KB  raw X tile
constexpr uint32_t SOP = R * BK * 4;        //  8 KB  W (or V') chunk hi; same again for lo
constexpr uint32_t SSTAGE = SX + 2 * SOP;   // 32 KB
constexpr uint32_t SMEM = STAGES * SSTAGE + 1024;
constexpr uint32_t TX_BYTES = SSTAGE;
// TMEM columns: [0,128) two fp32 accumulators (64 each), [128,256) two
// tf32-split A buffers (hi 32 + lo 32 columns each)
constexpr int TM_COLS = 256;
constexpr uint32_t TM_A = 128;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// hi/lo split of 32 values into the TMEM A buffer of this thread's lane
__device__ __forceinline__ void split_to_tmem(const float* x, uint32_t a_lane_addr, double& xx) {
    float hi[32], lo[32];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
        tc::split_tf32(x[i], hi[i], lo[i]);
        tc::split_tf32(x[i + 1], hi[i + 1], lo[i + 1]);
        tc::split_tf32(x[i + 2], hi[i + 2], lo[i + 2]);
        tc::split_tf32(x[i + 3], hi[i + 3], lo[i + 3]);
        s0 = fma((double)x[i], (double)x[i], s0);
        s1 = fma((double)x[i + 1], (double)x[i + 1], s1);
        s2 = fma((double)x[i + 2], (double)x[i + 2], s2);
        s3 = fma((double)x[i + 3], (double)x[i + 3], s3);
    }
    xx += (s0 + s1) + (s2 + s3);
    tc::tmem_st32(a_lane_addr, hi);
    tc::tmem_st32(a_lane_addr + 32, lo);
}

struct Bars {
    uint64_t full[STAGES], empty[STAGES], afull[2], aempty[2], qfull[2], qempty[2];
};

__device__ __forceinline__ void init_bars(Bars& B) {
    for (int s = 0; s < STAGES; ++s) {
        tc::mbar_init(&B.full[s], 1);
        tc::mbar_init(&B.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
        tc::mbar_init(&B.afull[b], 128);
        tc::mbar_init(&B.aempty[b], 1);
        tc::mbar_init(&B.qfull[b], 1);
        tc::mbar_init(&B.qempty[b], 128);
    }
    tc::fence_barrier_init();
}

// MMA issue for one stage: D += X (A in TMEM, hi/lo) . B (smem hi/lo), 3xTF32
template <bool B_MN>
__device__ __forceinline__ void issue_stage(uint32_t d, uint32_t a, const uint8_t* bh,
                                            const uint8_t* bl, bool first) {
    constexpr uint32_t idesc = tc::idesc_tf32(BM, R, 0, B_MN ? 1 : 0);
#pragma unroll
    for (int ks = 0; ks < BK / 8; ++ks) {
        uint64_t dh, dl;
        if (B_MN) {   // rows = K (8 per step = two 512-byte atoms), 32 N per 4 KB box
            dh = tc::sdesc_sw128_32b(bh + ks * 1024, 4096, 512);
            dl = tc::sdesc_sw128_32b(bl + ks * 1024, 4096, 512);
        } else {      // rows = N, K contiguous within the 128-byte swizzle row
            dh = tc::sdesc_sw128(bh + ks * 32, 16, 1024);
            dl = tc::sdesc_sw128(bl + ks * 32, 16, 1024);
        }
        const uint32_t ah = a + ks * 8, al = a + 32 + ks * 8;
        tc::mma_tf32_ts(d, al, dh, idesc, (first && ks == 0) ? 0u : 1u);
        tc::mma_tf32_ts(d, ah, dl, idesc, 1);
        tc::mma_tf32_ts(d, ah, dh, idesc, 1);
    }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
nnmf_vstep_tc(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mWh,
              const __grid_constant__ CUtensorMap mWl, const float* __restrict__ V,
              const double* __restrict__ GW, float* __restrict__ Vout, float* __restrict__ Vhi,
              float* __restrict__ Vlo, int m, int n, double* __restrict__ part) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = align1024(smem_raw);
    __shared__ Bars B;
    __shared__ uint32_t tmem_base;
    __shared__ double red[kThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (m + BM - 1) / BM, nk = (n + BK - 1) / BK;
    if (threadIdx.x == 0) init_bars(B);
    if (warp == 1) tc::tmem_alloc<TM_COLS>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    double acc = 0.0;

    if (warp == 0) {
        if (lane == 0) {
            tc::tma_prefetch(&mX);
            tc::tma_prefetch(&mWh);
            tc::tma_prefetch(&mWl);
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % STAGES;
                    tc::mbar_wait(&B.empty[s], ((it / STAGES) & 1) ^ 1);
                    uint8_t* st = base + s * SSTAGE;
                    tc::mbar_expect_tx(&B.full[s], TX_BYTES);
                    tc::tma_load_2d(st, &mX, &B.full[s], kb * BK, tile * BM);
                    tc::tma_load_2d(st + SX, &mWh, &B.full[s], kb * BK, 0);
                    tc::tma_load_2d(st + SX + SOP, &mWl, &B.full[s], kb * BK, 0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int it = 0, ti = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
                const int b = ti & 1;
                tc::mbar_wait(&B.qempty[b], ((ti >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t d = tmem + b * R;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % STAGES, ab = it & 1;
                    tc::mbar_wait(&B.afull[ab], (it >> 1) & 1);
                    tc::tc_fence_after();
                    const uint8_t* st = base + s * SSTAGE;
                    issue_stage<false>(d, tmem + TM_A + ab * 64, st + SX, st + SX + SOP, kb == 0);
                    tc::mma_commit(&B.empty[s]);
                    tc::mma_commit(&B.aempty[ab]);
                }
                tc::mma_commit(&B.qfull[b]);
            }
        }
    } else if (warp < 6) {
        // split warps: lane = row of the tile; read the row (128-byte swizzled)
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % STAGES, ab = it & 1;
                tc::mbar_wait(&B.full[s], (it / STAGES) & 1);
                const float4* rp = reinterpret_cast<const float4*>(base + s * SSTAGE + row * 128);
                float x[32];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float4 t = rp[c ^ (row & 7)];
                    x[4 * c] = t.x;
                    x[4 * c + 1] = t.y;
                    x[4 * c + 2] = t.z;
                    x[4 * c + 3] = t.w;
                }
                tc::mbar_wait(&B.aempty[ab], ((it >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                split_to_tmem(x, tmem + TM_A + ab * 64 + lane_off, acc);
                tc::tmem_st_wait();
                tc::tc_fence_before();
                tc::mbar_arrive(&B.afull[ab]);
            }
        }
    } else {
        const int quarter = warp & 3;
        int ti = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
            const int b = ti & 1;
            tc::mbar_wait(&B.qfull[b], (ti >> 1) & 1);
            tc::tc_fence_after();
            float q[R];
            const uint32_t ta = tmem + b * R + ((uint32_t)(quarter * 32) << 16);
            tc::tmem_ld32(ta, q);
            tc::tmem_ld32(ta + 32, q + 32);
            tc::tc_fence_before();
            tc::mbar_arrive(&B.qempty[b]);
            const long long row = (long long)tile * BM + quarter * 32 + lane;
            if (row < m) {
                float v[R];
                const float4* v4 = reinterpret_cast<const float4*>(V + row * R);
#pragma unroll
                for (int k4 = 0; k4 < R / 4; ++k4) {
                    const float4 t = v4[k4];
                    v[4 * k4] = t.x;
                    v[4 * k4 + 1] = t.y;
                    v[4 * k4 + 2] = t.z;
                    v[4 * k4 + 3] = t.w;
                }
#pragma unroll 2
                for (int k = 0; k < R; ++k) {
                    acc = fma((double)v[k], (double)q[k], acc);
                    double d0 = 0.0, d1 = 0.0;
#pragma unroll
                    for (int l = 0; l < R; l += 2) {
                        d0 = fma((double)v[l], __ldg(GW + l * R + k), d0);
                        d1 = fma((double)v[l + 1], __ldg(GW + (l + 1) * R + k), d1);
                    }
                    q[k] = (float)((double)v[k] * ((double)q[k] / ((d0 + d1) + kDenomGuard)));
                }
                float4* o = reinterpret_cast<float4*>(Vout + row * R);
                float4* oh = reinterpret_cast<float4*>(Vhi + row * R);
                float4* ol = reinterpret_cast<float4*>(Vlo + row * R);
#pragma unroll
                for (int k4 = 0; k4 < R / 4; ++k4) {
                    float4 t = make_float4(q[4 * k4], q[4 * k4 + 1], q[4 * k4 + 2], q[4 * k4 + 3]);
                    float4 h, l;
                    tc::split_tf32(t.x, h.x, l.x);
                    tc::split_tf32(t.y, h.y, l.y);
                    tc::split_tf32(t.z, h.z, l.z);
                    tc::split_tf32(t.w, h.w, l.w);
                    o[k4] = t;
                    oh[k4] = h;
                    ol[k4] = l;
                }
            }
        }
    }
    // per-CTA partials: [0] sum x^2 (split warps), [1] <V, Q> (epilogue warps)
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    tc::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = (red[2] + red[3]) + (red[4] + red[5]);
        part[2 * blockIdx.x + 1] = (red[6] + red[7]) + (red[8] + red[9]);
    }
    if (warp == 1) tc::tmem_free<TM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// P^T partial for (column block cb, row split s): D[col][k] = sum_rows X[row][col] V'[row][k]
// X tile arrives unswizzled (4 boxes of 32 rows x 32 columns); each split
// lane owns one column and transposes it into TMEM (lane = column, K = row).
__global__ void __launch_bounds__(kThreads, 1)
nnmf_wstep_tc(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mVh,
              const __grid_constant__ CUtensorMap mVl, int m, int n, int splits,
              int rows_per_split, float* __restrict__ wpart) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = align1024(smem_raw);
    __shared__ Bars B;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncb = (n + BM - 1) / BM;
    const int nitems = ncb * splits;
    if (threadIdx.x == 0) init_bars(B);
    if (warp == 1) tc::tmem_alloc<TM_COLS>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    auto item_rows = [&](int item, int& r0, int& nkb) {
        const int s = item / ncb;
        r0 = s * rows_per_split;
        int r1 = r0 + rows_per_split;
        if (r1 > m) r1 = m;
        nkb = r1 > r0 ? (r1 - r0 + BK - 1) / BK : 0;
    };

    if (warp == 0) {
        if (lane == 0) {
            tc::tma_prefetch(&mX);
            tc::tma_prefetch(&mVh);
            tc::tma_prefetch(&mVl);
            int it = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                const int cb = item % ncb;
                int r0, nkb;
                item_rows(item, r0, nkb);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % STAGES;
                    tc::mbar_wait(&B.empty[s], ((it / STAGES) & 1) ^ 1);
                    uint8_t* st = base + s * SSTAGE;
                    const int row = r0 + kb * BK;
                    tc::mbar_expect_tx(&B.full[s], TX_BYTES);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        tc::tma_load_2d(st + j * 4096, &mX, &B.full[s], cb * BM + 32 * j, row);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        tc::tma_load_2d(st + SX + j * 4096, &mVh, &B.full[s], 32 * j, row);
                        tc::tma_load_2d(st + SX + SOP + j * 4096, &mVl, &B.full[s], 32 * j, row);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int it = 0, ti = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++ti) {
                int r0, nkb;
                item_rows(item, r0, nkb);
                const int b = ti & 1;
                tc::mbar_wait(&B.qempty[b], ((ti >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t d = tmem + b * R;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % STAGES, ab = it & 1;
                    tc::mbar_wait(&B.afull[ab], (it >> 1) & 1);
                    tc::tc_fence_after();
                    const uint8_t* st = base + s * SSTAGE;
                    issue_stage<true>(d, tmem + TM_A + ab * 64, st + SX, st + SX + SOP, kb == 0);
                    tc::mma_commit(&B.empty[s]);
                    tc::mma_commit(&B.aempty[ab]);
                }
                tc::mma_commit(&B.qfull[b]);
            }
        }
    } else if (warp < 6) {
        const int quarter = warp & 3;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        double unused = 0.0;
        int it = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int r0, nkb;
            item_rows(item, r0, nkb);
            for (int kb = 0; kb < nkb; ++kb, ++it) {
                const int s = it % STAGES, ab = it & 1;
                tc::mbar_wait(&B.full[s], (it / STAGES) & 1);
                // column (quarter*32 + lane) of the tile = lane of box `quarter`
                const float* cp = reinterpret_cast<const float*>(base + s * SSTAGE + quarter * 4096) + lane;
                float x[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) x[k] = cp[k * 32];
                tc::mbar_wait(&B.aempty[ab], ((it >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                split_to_tmem(x, tmem + TM_A + ab * 64 + lane_off, unused);
                tc::tmem_st_wait();
                tc::tc_fence_before();
                tc::mbar_arrive(&B.afull[ab]);
            }
        }
    } else {
        const int quarter = warp & 3;
        int ti = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++ti) {
            const int cb = item % ncb, s = item / ncb;
            int r0, nkb;
            item_rows(item, r0, nkb);
            const int b = ti & 1;
            float p[R];
            tc::mbar_wait(&B.qfull[b], (ti >> 1) & 1);
            tc::tc_fence_after();
            if (nkb > 0) {
                const uint32_t ta = tmem + b * R + ((uint32_t)(quarter * 32) << 16);
                tc::tmem_ld32(ta, p);
                tc::tmem_ld32(ta + 32, p + 32);
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k) p[k] = 0.f;
            }
            tc::tc_fence_before();
            tc::mbar_arrive(&B.qempty[b]);
            const long long col = (long long)cb * BM + quarter * 32 + lane;
            if (col < n) {
                float4* o = reinterpret_cast<float4*>(wpart + ((long long)s * n + col) * R);
#pragma unroll
                for (int k4 = 0; k4 < R / 4; ++k4)
                    o[k4] = make_float4(p[4 * k4], p[4 * k4 + 1], p[4 * k4 + 2], p[4 * k4 + 3]);
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free<TM_COLS>(tmem);
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

// red[k n + j] = sum_s wpart[s][j][k] (fixed split order)
__global__ void wreduce_tc_kernel(const float* __restrict__ wpart, int splits, long long n,
                                  double* __restrict__ red) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * R) return;
    const long long j = t / R;
    const int k = (int)(t - j * R);
    double s = 0.0;
    for (int q = 0; q < splits; ++q) s += (double)wpart[((long long)q * n + j) * R + k];
    red[(long long)k * n + j] = s;
}

// f-partial = sum x^2 - 2 <V, Q> + <G_V, G_W> (all over this rank's rows)
__global__ void tc_objective_kernel(const double* __restrict__ part, int nparts,
                                    const double* __restrict__ GV, const double* __restrict__ GW,
                                    double* __restrict__ out) {
    __shared__ double sc[32];
    double xx = 0.0, cr = 0.0, gg = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
        xx += part[2 * i];
        cr += part[2 * i + 1];
    }
    for (int i = threadIdx.x; i < R * R; i += blockDim.x) gg = fma(GV[i], GW[i], gg);
    xx = block_sum(xx, sc);
    cr = block_sum(cr, sc);
    gg = block_sum(gg, sc);
    if (threadIdx.x == 0) *out = xx - 2.0 * cr + gg;
}

struct TcPlan {
    int vgrid, wgrid, splits, rows_per_split;
};

TcPlan tc_plan(long long m, long long n) {
    TcPlan P;
    const int ntiles = (int)((m + BM - 1) / BM);
    P.vgrid = ntiles < kNumSMs ? ntiles : kNumSMs;
    const int ncb = (int)((n + BM - 1) / BM);
    int splits = (4 * kNumSMs + ncb - 1) / ncb;
    const int max_splits = (int)((m + 4 * BK - 1) / (4 * BK));
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    long long rps = (m + splits - 1) / splits;
    rps = (rps + BK - 1) / BK * BK;
    P.rows_per_split = (int)rps;
    P.splits = (int)((m + rps - 1) / rps);
    const int items = ncb * P.splits;
    P.wgrid = items < kNumSMs ? items : kNumSMs;
    return P;
}

struct TcWs {
    float *Wh, *Wl, *Vhi, *Vlo, *wpart;
    double *GVn, *part;
};

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
    size_t oWp = take(4 * (size_t)P.splits * n * R);
    size_t oG = take(8 * (size_t)R * R);
    size_t oP = take(16 * (size_t)kNumSMs);
    if (base && L) {
        char* c = reinterpret_cast<char*>(base);
        L->Wh = (float*)(c + oWh);
        L->Wl = (float*)(c + oWl);
        L->Vhi = (float*)(c + oVh);
        L->Vlo = (float*)(c + oVl);
        L->wpart = (float*)(c + oWp);
        L->GVn = (double*)(c + oG);
        L->part = (double*)(c + oP);
    }
    return off;
}

bool g_attr_done = false;

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
        cudaFuncSetAttribute(nnmf_vstep_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        cudaFuncSetAttribute(nnmf_wstep_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        g_attr_done = true;
    }
    CUtensorMap mX, mWh, mWl, mXt, mVh, mVl;
    int rc;
    if ((rc = mmk_host::make_map_f32(&mX, X, m, n, ldx, BM))) return rc;
    if ((rc = mmk_host::make_map_f32(&mWh, L.Wh, R, n, n, R))) return rc;
    if ((rc = mmk_host::make_map_f32(&mWl, L.Wl, R, n, n, R))) return rc;
    if ((rc = mmk_host::make_map_f32(&mXt, X, m, n, ldx, BK, 0))) return rc;
    if ((rc = mmk_host::make_map_f32(&mVh, L.Vhi, m, R, R, BK, 32))) return rc;
    if ((rc = mmk_host::make_map_f32(&mVl, L.Vlo, m, R, R, BK, 32))) return rc;
    const long long rn = (long long)R * n;
    MMK_LAUNCH("nnmf_split_w", st,
               (split_w_kernel<<<ceil_div(rn, 256), 256, 0, st>>>(W, L.Wh, L.Wl, rn)));
    gram_w(W, GW, st);
    gram_v_into(V, L.GVn, st);
    MMK_LAUNCH("nnmf_vstep_tc", st,
               (nnmf_vstep_tc<<<P.vgrid, kThreads, SMEM, st>>>(mX, mWh, mWl, V, GW, V_out, L.Vhi,
                                                                L.Vlo, (int)m, (int)n, L.part)));
    MMK_CHECK_LAUNCH("nnmf_vstep_tc");
    MMK_LAUNCH("nnmf_objective_tc", st,
               (tc_objective_kernel<<<1, 256, 0, st>>>(L.part, P.vgrid, L.GVn, GW,
                                                        red + rn + (long long)R * R)));
    gram_v_into(V_out, red + rn, st);
    MMK_LAUNCH("nnmf_wstep_tc", st,
               (nnmf_wstep_tc<<<P.wgrid, kThreads, SMEM, st>>>(mXt, mVh, mVl, (int)m, (int)n,
                                                                P.splits, P.rows_per_split,
                                                                L.wpart)));
    MMK_CHECK_LAUNCH("nnmf_wstep_tc");
    MMK_LAUNCH("nnmf_wreduce_tc", st,
               (wreduce_tc_kernel<<<ceil_div(rn, 256), 256, 0, st>>>(L.wpart, P.splits, n, red)));
    MMK_CHECK_LAUNCH("nnmf_tc_iter_a");
    return MMK_OK;
}

}  // namespace mmk_tc
