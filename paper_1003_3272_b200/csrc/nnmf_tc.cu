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
constexpr int BK = 32;           // K per stage: one 128-byte swizzle row of fp32
constexpr int STAGES = 4;
constexpr int kThreads = 320;    // 10 warps: TMA, MMA, 4 split, 4 epilogue
constexpr uint32_t SX = BM * BK * 4;        // 16 KB  X tile (hi in place)
constexpr uint32_t SXL = SX;                // 16 KB  X lo
constexpr uint32_t SOP = R * BK * 4;        //  8 KB  W or V' chunk (hi), same for lo
constexpr uint32_t SSTAGE = SX + SXL + 2 * SOP;   // 48 KB
constexpr uint32_t SMEM = STAGES * SSTAGE + 1024;
constexpr uint32_t TX_BYTES = SX + 2 * SOP;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// split warps: hi/lo of the stage's X tile, position-preserving (the swizzle
// is a permutation of positions, so an elementwise rewrite keeps the layout)
__device__ __forceinline__ double split_stage(uint8_t* st, int ct) {
    float4* xr = reinterpret_cast<float4*>(st);
    float4* xl = reinterpret_cast<float4*>(st + SX);
    double xx = 0.0;
#pragma unroll
    for (int q = ct; q < (int)(SX / 16); q += 128) {
        const float4 v = xr[q];
        float4 h, l;
        tc::split_tf32(v.x, h.x, l.x);
        tc::split_tf32(v.y, h.y, l.y);
        tc::split_tf32(v.z, h.z, l.z);
        tc::split_tf32(v.w, h.w, l.w);
        xr[q] = h;
        xl[q] = l;
        xx = fma((double)v.x, (double)v.x, xx);
        xx = fma((double)v.y, (double)v.y, xx);
        xx = fma((double)v.z, (double)v.z, xx);
        xx = fma((double)v.w, (double)v.w, xx);
    }
    tc::fence_async_smem();
    return xx;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
nnmf_vstep_tc(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mWh,
              const __grid_constant__ CUtensorMap mWl, const float* __restrict__ V,
              const double* __restrict__ GW, float* __restrict__ Vout, float* __restrict__ Vhi,
              float* __restrict__ Vlo, int m, int n, double* __restrict__ part) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = align1024(smem_raw);
    __shared__ uint64_t full[STAGES], conv[STAGES], empty[STAGES], qfull[2], qempty[2];
    __shared__ uint32_t tmem_base;
    __shared__ double red[kThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (m + BM - 1) / BM, nk = (n + BK - 1) / BK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&conv[s], 128);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&qfull[b], 1);
            tc::mbar_init(&qempty[b], 128);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<128>(&tmem_base);
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
                    const uint32_t ph = (it / STAGES) & 1;
                    tc::mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* st = base + s * SSTAGE;
                    tc::mbar_expect_tx(&full[s], TX_BYTES);
                    tc::tma_load_2d(st, &mX, &full[s], kb * BK, tile * BM);
                    tc::tma_load_2d(st + SX + SXL, &mWh, &full[s], kb * BK, 0);
                    tc::tma_load_2d(st + SX + SXL + SOP, &mWl, &full[s], kb * BK, 0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(BM, R, 0, 0);
            int it = 0, ti = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
                const int b = ti & 1;
                tc::mbar_wait(&qempty[b], ((ti >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t d = tmem + b * R;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % STAGES;
                    tc::mbar_wait(&conv[s], (it / STAGES) & 1);
                    tc::tc_fence_after();
                    uint8_t* st = base + s * SSTAGE;
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        const uint64_t ah = tc::sdesc_sw128(st + ks * 32, 16, 1024);
                        const uint64_t al = tc::sdesc_sw128(st + SX + ks * 32, 16, 1024);
                        const uint64_t bh = tc::sdesc_sw128(st + SX + SXL + ks * 32, 16, 1024);
                        const uint64_t bl = tc::sdesc_sw128(st + SX + SXL + SOP + ks * 32, 16, 1024);
                        tc::mma_tf32(d, al, bh, idesc, (kb | ks) != 0);
                        tc::mma_tf32(d, ah, bl, idesc, 1);
                        tc::mma_tf32(d, ah, bh, idesc, 1);
                    }
                    tc::mma_commit(&empty[s]);
                }
                tc::mma_commit(&qfull[b]);
            }
        }
    } else if (warp < 6) {
        const int ct = threadIdx.x - 64;
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % STAGES;
                tc::mbar_wait(&full[s], (it / STAGES) & 1);
                acc += split_stage(base + s * SSTAGE, ct);
                tc::mbar_arrive(&conv[s]);
            }
        }
    } else {
        const int quarter = warp & 3;
        int ti = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
            const int b = ti & 1;
            tc::mbar_wait(&qfull[b], (ti >> 1) & 1);
            tc::tc_fence_after();
            float q[R];
            const uint32_t ta = tmem + b * R + ((uint32_t)(quarter * 32) << 16);
            tc::tmem_ld32(ta, q);
            tc::tmem_ld32(ta + 32, q + 32);
            tc::tc_fence_before();
            tc::mbar_arrive(&qempty[b]);
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
                    double den = 0.0;
#pragma unroll
                    for (int l = 0; l < R; ++l) den = fma((double)v[l], __ldg(GW + l * R + k), den);
                    q[k] = (float)((double)v[k] * ((double)q[k] / (den + kDenomGuard)));  // v'_k
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
        part[2 * blockIdx.x] = red[2] + red[3] + red[4] + red[5];
        part[2 * blockIdx.x + 1] = red[6] + red[7] + red[8] + red[9];
    }
    if (warp == 1) tc::tmem_free<128>(tmem);
}

// ---------------------------------------------------------------------------
// P^T partial for (column block cb, row split s): D[col][k] = sum_rows X[row][col] V'[row][k]
__global__ void __launch_bounds__(kThreads, 1)
nnmf_wstep_tc(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mVh,
              const __grid_constant__ CUtensorMap mVl, int m, int n, int splits,
              int rows_per_split, float* __restrict__ wpart) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = align1024(smem_raw);
    __shared__ uint64_t full[STAGES], conv[STAGES], empty[STAGES], qfull[2], qempty[2];
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncb = (n + BM - 1) / BM;
    const int nitems = ncb * splits;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&conv[s], 128);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&qfull[b], 1);
            tc::mbar_init(&qempty[b], 128);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<128>(&tmem_base);
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
                    tc::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    uint8_t* st = base + s * SSTAGE;
                    const int row = r0 + kb * BK;
                    tc::mbar_expect_tx(&full[s], TX_BYTES);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        tc::tma_load_2d(st + j * 4096, &mX, &full[s], cb * BM + 32 * j, row);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        tc::tma_load_2d(st + SX + SXL + j * 4096, &mVh, &full[s], 32 * j, row);
                        tc::tma_load_2d(st + SX + SXL + SOP + j * 4096, &mVl, &full[s], 32 * j, row);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(BM, R, 1, 1);
            int it = 0, ti = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++ti) {
                int r0, nkb;
                item_rows(item, r0, nkb);
                const int b = ti & 1;
                tc::mbar_wait(&qempty[b], ((ti >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t d = tmem + b * R;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = it % STAGES;
                    tc::mbar_wait(&conv[s], (it / STAGES) & 1);
                    tc::tc_fence_after();
                    uint8_t* st = base + s * SSTAGE;
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        const uint64_t ah = tc::sdesc_sw128_32b(st + ks * 1024, 4096, 512);
                        const uint64_t al = tc::sdesc_sw128_32b(st + SX + ks * 1024, 4096, 512);
                        const uint64_t bh = tc::sdesc_sw128_32b(st + SX + SXL + ks * 1024, 4096, 512);
                        const uint64_t bl =
                            tc::sdesc_sw128_32b(st + SX + SXL + SOP + ks * 1024, 4096, 512);
                        tc::mma_tf32(d, al, bh, idesc, (kb | ks) != 0);
                        tc::mma_tf32(d, ah, bl, idesc, 1);
                        tc::mma_tf32(d, ah, bh, idesc, 1);
                    }
                    tc::mma_commit(&empty[s]);
                }
                tc::mma_commit(&qfull[b]);
            }
        }
    } else if (warp < 6) {
        const int ct = threadIdx.x - 64;
        int it = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int r0, nkb;
            item_rows(item, r0, nkb);
            for (int kb = 0; kb < nkb; ++kb, ++it) {
                const int s = it % STAGES;
                tc::mbar_wait(&full[s], (it / STAGES) & 1);
                split_stage(base + s * SSTAGE, ct);
                tc::mbar_arrive(&conv[s]);
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
            if (nkb > 0) {
                tc::mbar_wait(&qfull[b], (ti >> 1) & 1);
                tc::tc_fence_after();
                const uint32_t ta = tmem + b * R + ((uint32_t)(quarter * 32) << 16);
                tc::tmem_ld32(ta, p);
                tc::tmem_ld32(ta + 32, p + 32);
                tc::tc_fence_before();
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k) p[k] = 0.f;
                tc::mbar_wait(&qfull[b], (ti >> 1) & 1);
            }
            tc::mbar_arrive(&qempty[b]);
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
    if (warp == 1) tc::tmem_free<128>(tmem);
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
    if ((rc = mmk_host::make_map_f32(&mXt, X, m, n, ldx, BK, true))) return rc;
    if ((rc = mmk_host::make_map_f32(&mVh, L.Vhi, m, R, R, BK, true))) return rc;
    if ((rc = mmk_host::make_map_f32(&mVl, L.Vlo, m, R, R, BK, true))) return rc;
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
