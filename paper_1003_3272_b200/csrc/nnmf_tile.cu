// nnmf_tile.cu -- register-blocked CUDA-core kernels of the Frobenius NNMF
// iteration for ranks 17..128 (rank tiles of 64 or 128): the fp64 path at any
// shape (BASELINE config 4
// in fp64: 131072 x 16384, r = 64) and fp32 shapes the tensor-core path does
// not take (nnmf_tc.cu: fp32 ranks 17..128, TMA-aligned shapes).  Reference: nnmf_objective / nnmf_update_v /
// nnmf_update_w (nnmf.py:75-110).
//
// The warp-per-row kernels of nnmf.cu keep a row's r dot products in
// registers -- right for the paper shape (r = 10), but at r = 64 that is
// 2 x 64 values per thread and the fp64 C4 V step spilled to 443 ms.  Here a
// CTA owns a 64 x 64 output tile and every thread a 4 x 4 block of it
// (rows / ranks ty + 16 i, tx + 16 j: the operand a thread reads from shared
// memory is either a warp broadcast or 16 consecutive values -- one
// wavefront), with the X / W chunks of the next K step prefetched into
// registers while the current one is consumed.  A thread's 4 rows (V step)
// or 4 ranks (W step) are contiguous in a transposed smem copy, so the
// broadcast operand arrives as two 16-byte loads: the kernels are bound by
// shared-memory wavefronts (ncu: L1 ~90 %, FP64 pipe ~47 % with scalar loads).
//
//   nnmf_vstep_tile  rows [64 b, 64 b + 64): Q = X W^T (K = n in chunks of
//                    32 columns), the residual sum (x - v.w)^2 of the same X
//                    chunk (V tile resident in smem, the W chunk a second
//                    time rank-major), then V' = V Q / (V G_W + 1e-300) (or
//                    the gradient 2 (V G_W - Q)) -- the same fused
//                    objective / update contract as nnmf_vstep_kernel
//   nnmf_wpart_tile  P = V'^T X over a row split: 64 ranks x 64 columns per
//                    CTA, K = 32 rows per chunk, partials [split][r][n] in
//                    fp64 (reduced in split order by nnmf_wreduce_kernel)
// Both sum in a fixed order: deterministic run to run.
#include <type_traits>

#include "mmk_common.cuh"
#include "nnmf_tile.h"

namespace {

using namespace mmk;

constexpr int TT = 256;   // threads
constexpr int TR = 64;    // rows (V step) / ranks (W step) per CTA
constexpr int TK = 32;    // K per chunk
constexpr int TC = 64;    // columns per CTA (W step)
enum { F_UPDATE = 1, F_RESID = 2, F_GRAD = 4 };   // as nnmf.cu VSTEP_*

// transposed rows padded by 16 bytes: 16-byte aligned for the vector loads,
// and the transposing stores hit 8 bank groups per warp (4-way) instead of 4
template <typename T, int RK>   // RK: rank tile, 64 or 128
struct VSmem {
    static constexpr int TP = 16 / (int)sizeof(T);
    T xt[TK][TR + TP];   // X chunk [col][row]
    T wa[TK][RK + 1];    // W chunk [col][rank] (Q operand)
    T wb[RK][TK + 1];    // W chunk [rank][col] (residual operand)
    T vt[RK][TR + TP];   // V tile [rank][row]
};

// the 4 consecutive values p[0..3] (16-byte aligned) as two / one vector loads
template <typename T>
__device__ __forceinline__ void ld4(const T* p, T (&a)[4]);
template <>
__device__ __forceinline__ void ld4<double>(const double* p, double (&a)[4]) {
    const double2 u = *reinterpret_cast<const double2*>(p);
    const double2 v = *reinterpret_cast<const double2*>(p + 2);
    a[0] = u.x;
    a[1] = u.y;
    a[2] = v.x;
    a[3] = v.y;
}
template <>
__device__ __forceinline__ void ld4<float>(const float* p, float (&a)[4]) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    a[0] = u.x;
    a[1] = u.y;
    a[2] = u.z;
    a[3] = u.w;
}

template <typename T, int RK>
__global__ void __launch_bounds__(TT)
nnmf_vstep_tile(const T* __restrict__ X, long long ldx, const T* __restrict__ V,
                const T* __restrict__ W, const double* __restrict__ GW, T* __restrict__ Vout,
                long long m, long long n, int r, int flags, double* __restrict__ respart,
                unsigned int* counter, double* res_out) {
    extern __shared__ __align__(16) unsigned char tile_smem[];
    constexpr int RJ = RK / 16;   // ranks per thread: tx + 16 j
    VSmem<T, RK>& S = *reinterpret_cast<VSmem<T, RK>*>(tile_smem);
    __shared__ double sc[32];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long long row0 = (long long)blockIdx.x * TR;
    const bool resid = flags & F_RESID;
    for (int e = tid; e < TR * RK; e += TT) {
        const int i = e / RK, k = e % RK;
        S.vt[k][i] = (row0 + i < m && k < r) ? V[(row0 + i) * r + k] : T(0);
    }
    // chunk loads: X rows tid/32 + 8u, column tid%32; W ranks tid/32 + 8u, same column
    const int lr = tid >> 5, lc = tid & 31;
    T xr[8], wr[RK / 8];
    auto load = [&](long long j0) {
        const long long j = j0 + lc;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long i = row0 + lr + 8 * u;
            xr[u] = (i < m && j < n) ? X[i * ldx + j] : T(0);
        }
#pragma unroll
        for (int u = 0; u < RK / 8; ++u) {
            const int k = lr + 8 * u;
            wr[u] = (k < r && j < n) ? W[(long long)k * n + j] : T(0);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int u = 0; u < 8; ++u) S.xt[lc][lr + 8 * u] = xr[u];
#pragma unroll
        for (int u = 0; u < RK / 8; ++u) {
            S.wb[lr + 8 * u][lc] = wr[u];
            S.wa[lc][lr + 8 * u] = wr[u];
        }
    };
    T q[4][RJ];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < RJ; ++j) q[i][j] = T(0);
    double res = 0.0;
    const long long nch = (n + TK - 1) / TK;
    load(0);
    store();
    __syncthreads();
    for (long long c = 0; c < nch; ++c) {
        const long long j0 = c * TK;
        if (c + 1 < nch) load(j0 + TK);   // in flight while this chunk is consumed
#pragma unroll 8
        for (int kk = 0; kk < TK; ++kk) {
            T a[4], b[RJ];
            ld4<T>(&S.xt[kk][4 * ty], a);   // rows 4 ty .. 4 ty + 3
#pragma unroll
            for (int j = 0; j < RJ; ++j) b[j] = S.wa[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < RJ; ++j) q[i][j] = fma(a[i], b[j], q[i][j]);
        }
        if (resid) {   // rows 4 ty + i, chunk columns tx + 16 j (j < 2)
            T rec[4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i) rec[i][0] = rec[i][1] = T(0);
#pragma unroll 8
            for (int k = 0; k < RK; ++k) {
                T a[4];
                ld4<T>(&S.vt[k][4 * ty], a);
                const T b0 = S.wb[k][tx], b1 = S.wb[k][tx + 16];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    rec[i][0] = fma(a[i], b0, rec[i][0]);
                    rec[i][1] = fma(a[i], b1, rec[i][1]);
                }
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                T xv[4];
                ld4<T>(&S.xt[tx + 16 * j][4 * ty], xv);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (row0 + 4 * ty + i < m && j0 + tx + 16 * j < n) {
                        const double d = (double)xv[i] - (double)rec[i][j];
                        res = fma(d, d, res);
                    }
                }
            }
        }
        __syncthreads();
        if (c + 1 < nch) {
            store();
            __syncthreads();
        }
    }
    if (flags & F_UPDATE) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const long long row = row0 + 4 * ty + i;
            double den[RJ];
#pragma unroll
            for (int j = 0; j < RJ; ++j) den[j] = 0.0;
            for (int l = 0; l < r; ++l) {
                const double vl = (double)S.vt[l][4 * ty + i];
#pragma unroll
                for (int j = 0; j < RJ; ++j) {
                    const int k = tx + 16 * j;
                    if (k < r) den[j] = fma(vl, GW[l * r + k], den[j]);
                }
            }
            if (row >= m) continue;
#pragma unroll
            for (int j = 0; j < RJ; ++j) {
                const int k = tx + 16 * j;
                if (k >= r) continue;
                if (flags & F_GRAD) {   // 2 (V G_W - X W^T)
                    Vout[row * r + k] = (T)(2.0 * (den[j] - (double)q[i][j]));
                } else {
                    const double vk = (double)S.vt[k][4 * ty + i];
                    Vout[row * r + k] = (T)(vk * ((double)q[i][j] / (den[j] + kDenomGuard)));
                }
            }
        }
    }
    if (!resid) return;
    const double bs = block_sum(res, sc);
    if (tid == 0) respart[blockIdx.x] = bs;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(respart, gridDim.x, sc);
        if (tid == 0) *res_out = tot;
    }
}

// ---------------------------------------------------------------------------
// fp64 on the FP64 tensor cores (DMMA, mma.sync m8n8k4 .f64): the same CTA
// tiles, shared-memory layouts and contract as nnmf_vstep_tile /
// nnmf_wpart_tile, with the three contractions -- Q = X W^T, the residual's
// V W and P = V'^T X -- as 8 x 8 x 4 fp64 MMAs (exact fp64 products, fp64
// accumulation; the order of the K sums differs from the FMA kernels only by
// rounding).  Fragments (PTX m8n8k4 .f64, lane = 4 g + t): A[g][t], B[t][g],
// C[g][2t + {0, 1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// DMMA tiles keep every operand in its natural orientation with rows padded
// to a stride of 4 (mod 16) doubles: the fragment reads [k + t][base + g] and
// [base + g][k + t] of a 16-lane phase then hit 16 distinct bank pairs, and
// the chunk stores (consecutive lanes, consecutive columns) are conflict-free.
template <int RK>
struct VSmemD {
    double xs[TR][TK + 4];   // X chunk [row][col]
    double wb[RK][TK + 4];   // W chunk [rank][col]
    double v[TR][RK + 4];    // V tile [row][rank]
};

template <int RK>
__global__ void __launch_bounds__(TT)
nnmf_vstep_dmma(const double* __restrict__ X, long long ldx, const double* __restrict__ V,
                const double* __restrict__ W, const double* __restrict__ GW,
                double* __restrict__ Vout, long long m, long long n, int r, int flags,
                double* __restrict__ respart, unsigned int* counter, double* res_out) {
    using T = double;
    extern __shared__ __align__(16) unsigned char tile_smem[];
    constexpr int NT = RK / 16;   // Q n-tiles (8 ranks) per warp: warp (wm, wn) = 16 rows x RK/2
    VSmemD<RK>& S = *reinterpret_cast<VSmemD<RK>*>(tile_smem);
    __shared__ double sc[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3, wm = warp >> 1, wn = warp & 1;
    const long long row0 = (long long)blockIdx.x * TR;
    const bool resid = flags & F_RESID;
    for (int e = tid; e < TR * RK; e += TT) {
        const int i = e / RK, k = e % RK;
        S.v[i][k] = (row0 + i < m && k < r) ? V[(row0 + i) * r + k] : T(0);
    }
    const int lr = tid >> 5, lc = tid & 31;
    T xr[8], wr[RK / 8];
    auto load = [&](long long j0) {
        const long long j = j0 + lc;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long i = row0 + lr + 8 * u;
            xr[u] = (i < m && j < n) ? X[i * ldx + j] : T(0);
        }
#pragma unroll
        for (int u = 0; u < RK / 8; ++u) {
            const int k = lr + 8 * u;
            wr[u] = (k < r && j < n) ? W[(long long)k * n + j] : T(0);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int u = 0; u < 8; ++u) S.xs[lr + 8 * u][lc] = xr[u];
#pragma unroll
        for (int u = 0; u < RK / 8; ++u) S.wb[lr + 8 * u][lc] = wr[u];
    };
    T q[2][NT][2];   // Q tiles: rows 16 wm + 8 mt + g, ranks wn RK/2 + 8 nt + 2 t + e
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) q[a][b][0] = q[a][b][1] = T(0);
    double res = 0.0;
    const long long nch = (n + TK - 1) / TK;
    load(0);
    store();
    __syncthreads();
    for (long long c = 0; c < nch; ++c) {
        const long long j0 = c * TK;
        if (c + 1 < nch) load(j0 + TK);   // in flight while this chunk is consumed
#pragma unroll 2
        for (int kk = 0; kk < TK; kk += 4) {
            T a[2], b[NT];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) a[mt] = S.xs[16 * wm + 8 * mt + g][kk + t];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) b[nt] = S.wb[wn * (RK / 2) + 8 * nt + g][kk + t];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma884(q[mt][nt][0], q[mt][nt][1], a[mt], b[nt]);
        }
        if (resid) {   // V W of the chunk: rows 16 wm + 8 mt + g, columns 16 wn + 8 nt + 2 t + e
            T rec[2][2][2];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 2; ++b) rec[a][b][0] = rec[a][b][1] = T(0);
#pragma unroll 4
            for (int ks = 0; ks < RK; ks += 4) {
                T a[2], b[2];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) a[mt] = S.v[16 * wm + 8 * mt + g][ks + t];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) b[nt] = S.wb[ks + t][16 * wn + 8 * nt + g];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
                        dmma884(rec[mt][nt][0], rec[mt][nt][1], a[mt], b[nt]);
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int il = 16 * wm + 8 * mt + g, jl = 16 * wn + 8 * nt + 2 * t + e;
                        if (row0 + il < m && j0 + jl < n) {
                            const double d = S.xs[il][jl] - rec[mt][nt][e];
                            res = fma(d, d, res);
                        }
                    }
        }
        __syncthreads();
        if (c + 1 < nch) {
            store();
            __syncthreads();
        }
    }
    if (flags & F_UPDATE) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const int il = 16 * wm + 8 * mt + g;
            const long long row = row0 + il;
            double den[NT][2];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) den[nt][0] = den[nt][1] = 0.0;
            for (int l = 0; l < r; ++l) {
                const double vl = S.v[il][l];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int k = wn * (RK / 2) + 8 * nt + 2 * t + e;
                        if (k < r) den[nt][e] = fma(vl, GW[l * r + k], den[nt][e]);
                    }
            }
            if (row >= m) continue;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int k = wn * (RK / 2) + 8 * nt + 2 * t + e;
                    if (k >= r) continue;
                    if (flags & F_GRAD) {   // 2 (V G_W - X W^T)
                        Vout[row * r + k] = 2.0 * (den[nt][e] - q[mt][nt][e]);
                    } else {
                        const double vk = S.v[il][k];
                        Vout[row * r + k] = vk * (q[mt][nt][e] / (den[nt][e] + kDenomGuard));
                    }
                }
        }
    }
    if (!resid) return;
    const double bs = block_sum(res, sc);
    if (tid == 0) respart[blockIdx.x] = bs;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(respart, gridDim.x, sc);
        if (tid == 0) *res_out = tot;
    }
}

template <typename T, int RK>
struct WSmem {
    T vs[TK][RK + 16 / sizeof(T)];   // V' chunk [row][rank]
    T xs[TK][TC + 1];                // X chunk [row][col]
};

template <typename T, int RK>
__global__ void __launch_bounds__(TT)
nnmf_wpart_tile(const T* __restrict__ X, long long ldx, const T* __restrict__ V, long long m,
                long long n, int r, long long rows_per_split, double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char tile_smem[];
    constexpr int RI = RK / 16;   // ranks per thread: RI ty .. RI ty + RI - 1
    WSmem<T, RK>& S = *reinterpret_cast<WSmem<T, RK>*>(tile_smem);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long long c0 = (long long)blockIdx.x * TC;
    const long long lo = (long long)blockIdx.y * rows_per_split;
    const long long hi = lo + rows_per_split < m ? lo + rows_per_split : m;
    // chunk loads: X rows tid/64 + 4u, column tid%64; V rows tid/64 + 4u, rank tid%64
    const int lr = tid >> 6, lc = tid & 63;
    T xr[8], vr[8][RK / 64];
    auto load = [&](long long i0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long i = i0 + lr + 4 * u;
            xr[u] = (i < hi && c0 + lc < n) ? X[i * ldx + c0 + lc] : T(0);
#pragma unroll
            for (int h = 0; h < RK / 64; ++h)
                vr[u][h] = (i < hi && lc + 64 * h < r) ? V[i * r + lc + 64 * h] : T(0);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            S.xs[lr + 4 * u][lc] = xr[u];
#pragma unroll
            for (int h = 0; h < RK / 64; ++h) S.vs[lr + 4 * u][lc + 64 * h] = vr[u][h];
        }
    };
    T acc[RI][4];
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    const long long nch = hi > lo ? (hi - lo + TK - 1) / TK : 0;
    if (nch > 0) {
        load(lo);
        store();
        __syncthreads();
    }
    for (long long c = 0; c < nch; ++c) {
        if (c + 1 < nch) load(lo + (c + 1) * TK);
#pragma unroll 8
        for (int kk = 0; kk < TK; ++kk) {
            T a[RI], b[4];
#pragma unroll
            for (int h = 0; h < RI / 4; ++h) {   // ranks RI ty .. (warp broadcast)
                T a4[4];
                ld4<T>(&S.vs[kk][RI * ty + 4 * h], a4);
#pragma unroll
                for (int e = 0; e < 4; ++e) a[4 * h + e] = a4[e];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = S.xs[kk][tx + 16 * j];   // columns: 16 consecutive
#pragma unroll
            for (int i = 0; i < RI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
        if (c + 1 < nch) {
            store();
            __syncthreads();
        }
    }
    double* o = out + (long long)blockIdx.y * r * n;
#pragma unroll
    for (int i = 0; i < RI; ++i) {
        const int k = RI * ty + i;
        if (k >= r) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long col = c0 + tx + 16 * j;
            if (col < n) o[(long long)k * n + col] = (double)acc[i][j];
        }
    }
}

// ---------------------------------------------------------------------------
// Poisson loss (nnmf.py:178-265), ranks 17..128 (rank tiles of 64 and 128), the contract of
// pois_vstep_kernel / pois_wpart_kernel (nnmf_poisson.cu): per X chunk the
// reconstruction b = v.w of every element (K = r, as the residual above), the
// objective terms x ln b - b, and the ratio x / b (0 where x = 0) written over
// the X chunk in smem, then the same Q contraction with the ratio in place of
// X; v' = v sqrt(q / (sum_j w_kj + 1e-300)).  A zero b under a positive count
// flags site 1 (objective class) in the V step, site 2 (update only) in the W
// step.
template <typename T, int RK>
__global__ void __launch_bounds__(TT)
pois_vstep_tile(const T* __restrict__ X, long long ldx, const T* __restrict__ V,
                const T* __restrict__ W, const double* __restrict__ wsum, T* __restrict__ Vout,
                long long m, long long n, int r, double* __restrict__ fpart,
                unsigned int* counter, double* f_out, int64_t* err) {
    constexpr int RJ = RK / 16;   // ranks per thread (tx + 16 j)
    extern __shared__ __align__(16) unsigned char tile_smem[];
    VSmem<T, RK>& S = *reinterpret_cast<VSmem<T, RK>*>(tile_smem);
    __shared__ double sc[32];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long long row0 = (long long)blockIdx.x * TR;
    for (int e = tid; e < TR * RK; e += TT) {
        const int i = e / RK, k = e % RK;
        S.vt[k][i] = (row0 + i < m && k < r) ? V[(row0 + i) * r + k] : T(0);
    }
    const int lr = tid >> 5, lc = tid & 31;
    T xr[8], wr[RK / 8];
    auto load = [&](long long j0) {
        const long long j = j0 + lc;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long i = row0 + lr + 8 * u;
            xr[u] = (i < m && j < n) ? X[i * ldx + j] : T(0);
        }
#pragma unroll
        for (int u = 0; u < RK / 8; ++u) {
            const int k = lr + 8 * u;
            wr[u] = (k < r && j < n) ? W[(long long)k * n + j] : T(0);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int u = 0; u < 8; ++u) S.xt[lc][lr + 8 * u] = xr[u];
#pragma unroll
        for (int u = 0; u < RK / 8; ++u) {
            S.wb[lr + 8 * u][lc] = wr[u];
            S.wa[lc][lr + 8 * u] = wr[u];
        }
    };
    T q[4][RJ];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < RJ; ++j) q[i][j] = T(0);
    double f = 0.0;
    const long long nch = (n + TK - 1) / TK;
    load(0);
    store();
    __syncthreads();
    for (long long c = 0; c < nch; ++c) {
        const long long j0 = c * TK;
        if (c + 1 < nch) load(j0 + TK);
        {   // b, objective terms and ratio for rows 4 ty + i, columns tx + 16 j
            T rec[4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i) rec[i][0] = rec[i][1] = T(0);
#pragma unroll 8
            for (int k = 0; k < RK; ++k) {
                T a[4];
                ld4<T>(&S.vt[k][4 * ty], a);
                const T b0 = S.wb[k][tx], b1 = S.wb[k][tx + 16];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    rec[i][0] = fma(a[i], b0, rec[i][0]);
                    rec[i][1] = fma(a[i], b1, rec[i][1]);
                }
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const long long col = j0 + tx + 16 * j;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const long long row = row0 + 4 * ty + i;
                    T* xp = &S.xt[tx + 16 * j][4 * ty + i];
                    const T x = *xp, b = rec[i][j];
                    T ratio = T(0);
                    if (row < m && col < n) {
                        f -= (double)b;
                        if (x > T(0)) {
                            if (b == T(0)) {
                                flag_error(err, MMK_E_NUMERICS, err_at(1, row * n + col));
                            } else {
                                f = fma((double)x, log((double)b), f);
                                ratio = x / b;
                            }
                        }
                    }
                    *xp = ratio;
                }
            }
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < TK; ++kk) {
            T a[4], b[RJ];
            ld4<T>(&S.xt[kk][4 * ty], a);   // ratios of rows 4 ty .. 4 ty + 3
#pragma unroll
            for (int j = 0; j < RJ; ++j) b[j] = S.wa[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < RJ; ++j) q[i][j] = fma(a[i], b[j], q[i][j]);
        }
        __syncthreads();
        if (c + 1 < nch) {
            store();
            __syncthreads();
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const long long row = row0 + 4 * ty + i;
        if (row >= m) continue;
#pragma unroll
        for (int j = 0; j < RJ; ++j) {
            const int k = tx + 16 * j;
            if (k >= r) continue;
            const double vk = (double)S.vt[k][4 * ty + i];
            Vout[row * r + k] = (T)(vk * sqrt((double)q[i][j] / (wsum[k] + kDenomGuard)));
        }
    }
    const double bs = block_sum(f, sc);
    if (tid == 0) fpart[blockIdx.x] = bs;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(fpart, gridDim.x, sc);
        if (tid == 0) *f_out = tot;
    }
}

template <typename T, int RK>
struct PWSmem {
    T vs[TK][RK + 16 / sizeof(T)];   // V' chunk [row][rank]
    T xs[TK][TC + 1];                // X chunk [row][col], then the ratios
    T wt[RK][TC + 1];                // W [rank][col] of this column block (resident)
};

template <typename T, int RK>
__global__ void __launch_bounds__(TT)
pois_wpart_tile(const T* __restrict__ X, long long ldx, const T* __restrict__ V,
                const T* __restrict__ W, long long m, long long n, int r,
                long long rows_per_split, double* __restrict__ out, int64_t* err) {
    constexpr int RI = RK / 16;   // ranks per thread (RI ty + i)
    constexpr int VH = RK / 64;   // V' values per thread and row (ranks lc + 64 h)
    extern __shared__ __align__(16) unsigned char tile_smem[];
    PWSmem<T, RK>& S = *reinterpret_cast<PWSmem<T, RK>*>(tile_smem);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long long c0 = (long long)blockIdx.x * TC;
    const long long lo = (long long)blockIdx.y * rows_per_split;
    const long long hi = lo + rows_per_split < m ? lo + rows_per_split : m;
    for (int e = tid; e < RK * TC; e += TT) {
        const int k = e / TC, cc = e % TC;
        S.wt[k][cc] = (k < r && c0 + cc < n) ? W[(long long)k * n + c0 + cc] : T(0);
    }
    const int lr = tid >> 6, lc = tid & 63;
    T xr[8], vr[8][VH];
    auto load = [&](long long i0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long i = i0 + lr + 4 * u;
            xr[u] = (i < hi && c0 + lc < n) ? X[i * ldx + c0 + lc] : T(0);
#pragma unroll
            for (int h = 0; h < VH; ++h)
                vr[u][h] = (i < hi && lc + 64 * h < r) ? V[i * r + lc + 64 * h] : T(0);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            S.xs[lr + 4 * u][lc] = xr[u];
#pragma unroll
            for (int h = 0; h < VH; ++h) S.vs[lr + 4 * u][lc + 64 * h] = vr[u][h];
        }
    };
    T acc[RI][4];
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    const long long nch = hi > lo ? (hi - lo + TK - 1) / TK : 0;
    if (nch > 0) {
        load(lo);
        store();
    }
    __syncthreads();   // wt and the first chunk
    for (long long ch = 0; ch < nch; ++ch) {
        const long long i0 = lo + ch * TK;
        if (ch + 1 < nch) load(i0 + TK);
        // ratios of this thread's elements (rows lr + 4 u, column lc), in place
#pragma unroll 2
        for (int u = 0; u < 8; ++u) {
            const int rl = lr + 4 * u;
            const T x = S.xs[rl][lc];
            T ratio = T(0);
            if (x > T(0)) {
                T b = T(0);
#pragma unroll 8
                for (int k = 0; k < RK; ++k) b = fma(S.vs[rl][k], S.wt[k][lc], b);
                if (b == T(0))
                    flag_error(err, MMK_E_NUMERICS, err_at_update(2, (i0 + rl) * n + c0 + lc));
                else
                    ratio = x / b;
            }
            S.xs[rl][lc] = ratio;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < TK; ++kk) {
            T a[RI], b[4];
#pragma unroll
            for (int h = 0; h < RI / 4; ++h) {   // ranks RI ty .. (warp broadcast)
                T a4[4];
                ld4<T>(&S.vs[kk][RI * ty + 4 * h], a4);
#pragma unroll
                for (int i = 0; i < 4; ++i) a[4 * h + i] = a4[i];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = S.xs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < RI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
        if (ch + 1 < nch) {
            store();
            __syncthreads();
        }
    }
    double* o = out + (long long)blockIdx.y * r * n;
#pragma unroll
    for (int i = 0; i < RI; ++i) {
        const int k = RI * ty + i;
        if (k >= r) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long col = c0 + tx + 16 * j;
            if (col < n) o[(long long)k * n + col] = (double)acc[i][j];
        }
    }
}

// P = V'^T X over a row split on the FP64 tensor cores (see nnmf_vstep_dmma):
// RK ranks x 64 columns per CTA, warp (wm, wn) = RK/4 ranks x 32 columns.
template <int RK>
struct WSmemD {
    double vs[TK][RK + 4];   // V' chunk [row][rank]
    double xs[TK][TC + 4];   // X chunk [row][col]
};
template <int RK>
__global__ void __launch_bounds__(TT)
nnmf_wpart_dmma(const double* __restrict__ X, long long ldx, const double* __restrict__ V,
                long long m, long long n, int r, long long rows_per_split,
                double* __restrict__ out) {
    using T = double;
    extern __shared__ __align__(16) unsigned char tile_smem[];
    constexpr int MT = RK / 32;   // m-tiles (8 ranks) per warp
    WSmemD<RK>& S = *reinterpret_cast<WSmemD<RK>*>(tile_smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3, wm = warp >> 1, wn = warp & 1;
    const long long c0 = (long long)blockIdx.x * TC;
    const long long lo = (long long)blockIdx.y * rows_per_split;
    const long long hi = lo + rows_per_split < m ? lo + rows_per_split : m;
    const int lr = tid >> 6, lc = tid & 63;
    T xr[8], vr[8][RK / 64];
    auto load = [&](long long i0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long i = i0 + lr + 4 * u;
            xr[u] = (i < hi && c0 + lc < n) ? X[i * ldx + c0 + lc] : T(0);
#pragma unroll
            for (int h = 0; h < RK / 64; ++h)
                vr[u][h] = (i < hi && lc + 64 * h < r) ? V[i * r + lc + 64 * h] : T(0);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            S.xs[lr + 4 * u][lc] = xr[u];
#pragma unroll
            for (int h = 0; h < RK / 64; ++h) S.vs[lr + 4 * u][lc + 64 * h] = vr[u][h];
        }
    };
    T acc[MT][4][2];   // ranks wm RK/4 + 8 mt + g, columns 32 wn + 8 nt + 2 t + e
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = T(0);
    const long long nch = hi > lo ? (hi - lo + TK - 1) / TK : 0;
    if (nch > 0) {
        load(lo);
        store();
        __syncthreads();
    }
    for (long long c = 0; c < nch; ++c) {
        if (c + 1 < nch) load(lo + (c + 1) * TK);
#pragma unroll 2
        for (int kk = 0; kk < TK; kk += 4) {
            T a[MT], b[4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) a[mt] = S.vs[kk + t][wm * (RK / 4) + 8 * mt + g];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) b[nt] = S.xs[kk + t][32 * wn + 8 * nt + g];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
                    dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
        }
        __syncthreads();
        if (c + 1 < nch) {
            store();
            __syncthreads();
        }
    }
    double* o = out + (long long)blockIdx.y * r * n;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const int k = wm * (RK / 4) + 8 * mt + g;
        if (k >= r) continue;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long long col = c0 + 32 * wn + 8 * nt + 2 * t + e;
                if (col < n) o[(long long)k * n + col] = acc[mt][nt][e];
            }
    }
}

}  // namespace

namespace mmk_tile {

bool applies(long long r) { return r > 16 && r <= 128; }

long long vstep_blocks(long long m) { return (m + TR - 1) / TR; }

template <typename T, int RK>
void vstep_rk(const T* X, long long ldx, const T* V, const T* W, const double* GW, T* Vout,
              long long m, long long n, int r, int flags, double* respart, unsigned int* counter,
              double* res_out, cudaStream_t st) {
    const size_t smem = sizeof(VSmem<T, RK>);
    if constexpr (std::is_same<T, double>::value) {   // fp64: the DMMA form
        const size_t dsm = sizeof(VSmemD<RK>);
        if (mmk_host::first_on_device(reinterpret_cast<const void*>(nnmf_vstep_dmma<RK>)))
            cudaFuncSetAttribute(nnmf_vstep_dmma<RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dsm);
        MMK_LAUNCH("nnmf_vstep_tile", st,
                   (nnmf_vstep_dmma<RK><<<(unsigned)vstep_blocks(m), TT, dsm, st>>>(
                       X, ldx, V, W, GW, Vout, m, n, r, flags, respart, counter, res_out)));
        return;
    }
    if (mmk_host::first_on_device(reinterpret_cast<const void*>(nnmf_vstep_tile<T, RK>)))
        cudaFuncSetAttribute(nnmf_vstep_tile<T, RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    MMK_LAUNCH("nnmf_vstep_tile", st,
               (nnmf_vstep_tile<T, RK><<<(unsigned)vstep_blocks(m), TT, smem, st>>>(
                   X, ldx, V, W, GW, Vout, m, n, r, flags, respart, counter, res_out)));
}

template <typename T>
void vstep(const T* X, long long ldx, const T* V, const T* W, const double* GW, T* Vout,
           long long m, long long n, int r, int flags, double* respart, unsigned int* counter,
           double* res_out, cudaStream_t st) {
    if (r <= 64)
        vstep_rk<T, 64>(X, ldx, V, W, GW, Vout, m, n, r, flags, respart, counter, res_out, st);
    else
        vstep_rk<T, 128>(X, ldx, V, W, GW, Vout, m, n, r, flags, respart, counter, res_out, st);
}

template <typename T>
int wpart_splits(long long m, long long n, int max_splits) {
    const long long cb = (n + TC - 1) / TC;
    long long S = (2 * kNumSMs + cb - 1) / cb;
    const long long smax = (m + TK - 1) / TK;
    if (S > smax) S = smax;
    if (S > max_splits) S = max_splits;
    return S < 1 ? 1 : (int)S;
}

int wpart_splits_dmma(long long m, long long n, int r, int max_splits) {
    // resident CTAs per SM: rank tile 64 -> 2 (35 KB smem, 94 registers), 128 -> 1
    const long long slots = (long long)kNumSMs * (r <= 64 ? 2 : 1);
    const long long cb = (n + TC - 1) / TC;
    const long long smax = (m + 4 * TK - 1) / (4 * TK);   // >= 4 row chunks per CTA
    int best = 1;
    double best_t = 1e300;
    for (int S = 1; S <= max_splits && S <= smax; ++S) {
        // a CTA covers m / S rows: time ~ waves * m / S, plus the S r n fp64
        // partials written and read back (relative to one pass over X)
        const long long waves = (cb * S + slots - 1) / slots;
        const double t = (double)waves / S + 2.0 * S * (double)r / (double)m;
        if (t < best_t - 1e-12) {
            best_t = t;
            best = S;
        }
    }
    return best;
}

template <typename T, int RK>
void wpart_rk(const T* X, long long ldx, const T* V, long long m, long long n, int r, int S,
              double* out, cudaStream_t st) {
    const size_t smem = sizeof(WSmem<T, RK>);
    if constexpr (std::is_same<T, double>::value) {   // fp64: the DMMA form
        const size_t dsm = sizeof(WSmemD<RK>);
        if (mmk_host::first_on_device(reinterpret_cast<const void*>(nnmf_wpart_dmma<RK>)))
            cudaFuncSetAttribute(nnmf_wpart_dmma<RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dsm);
        const long long rps = (m + S - 1) / S;
        dim3 grid((unsigned)((n + TC - 1) / TC), (unsigned)S);
        MMK_LAUNCH("nnmf_wpart_tile", st,
                   (nnmf_wpart_dmma<RK><<<grid, TT, dsm, st>>>(X, ldx, V, m, n, r, rps, out)));
        return;
    }
    if (mmk_host::first_on_device(reinterpret_cast<const void*>(nnmf_wpart_tile<T, RK>)))
        cudaFuncSetAttribute(nnmf_wpart_tile<T, RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    const long long rps = (m + S - 1) / S;
    dim3 grid((unsigned)((n + TC - 1) / TC), (unsigned)S);
    MMK_LAUNCH("nnmf_wpart_tile", st,
               (nnmf_wpart_tile<T, RK><<<grid, TT, smem, st>>>(X, ldx, V, m, n, r, rps, out)));
}

template <typename T>
void wpart(const T* X, long long ldx, const T* V, long long m, long long n, int r, int S,
           double* out, cudaStream_t st) {
    if (r <= 64)
        wpart_rk<T, 64>(X, ldx, V, m, n, r, S, out, st);
    else
        wpart_rk<T, 128>(X, ldx, V, m, n, r, S, out, st);
}

template <typename T, int RK>
void pois_vstep_rk(const T* X, long long ldx, const T* V, const T* W, const double* wsum,
                   T* Vout, long long m, long long n, int r, double* fpart, unsigned int* counter,
                   double* f_out, int64_t* err, cudaStream_t st) {
    const size_t smem = sizeof(VSmem<T, RK>);
    if (mmk_host::first_on_device(reinterpret_cast<const void*>(pois_vstep_tile<T, RK>)))
        cudaFuncSetAttribute(pois_vstep_tile<T, RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    MMK_LAUNCH("pois_vstep_tile", st,
               (pois_vstep_tile<T, RK><<<(unsigned)vstep_blocks(m), TT, smem, st>>>(
                   X, ldx, V, W, wsum, Vout, m, n, r, fpart, counter, f_out, err)));
}

template <typename T>
void pois_vstep(const T* X, long long ldx, const T* V, const T* W, const double* wsum, T* Vout,
                long long m, long long n, int r, double* fpart, unsigned int* counter,
                double* f_out, int64_t* err, cudaStream_t st) {
    if (r <= 64)
        pois_vstep_rk<T, 64>(X, ldx, V, W, wsum, Vout, m, n, r, fpart, counter, f_out, err, st);
    else
        pois_vstep_rk<T, 128>(X, ldx, V, W, wsum, Vout, m, n, r, fpart, counter, f_out, err, st);
}

template <typename T, int RK>
void pois_wpart_rk(const T* X, long long ldx, const T* V, const T* W, long long m, long long n,
                   int r, int S, double* out, int64_t* err, cudaStream_t st) {
    const size_t smem = sizeof(PWSmem<T, RK>);
    if (mmk_host::first_on_device(reinterpret_cast<const void*>(pois_wpart_tile<T, RK>)))
        cudaFuncSetAttribute(pois_wpart_tile<T, RK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    const long long rps = (m + S - 1) / S;
    dim3 grid((unsigned)((n + TC - 1) / TC), (unsigned)S);
    MMK_LAUNCH("pois_wpart_tile", st,
               (pois_wpart_tile<T, RK><<<grid, TT, smem, st>>>(X, ldx, V, W, m, n, r, rps, out,
                                                                err)));
}

template <typename T>
void pois_wpart(const T* X, long long ldx, const T* V, const T* W, long long m, long long n,
                int r, int S, double* out, int64_t* err, cudaStream_t st) {
    if (r <= 64)
        pois_wpart_rk<T, 64>(X, ldx, V, W, m, n, r, S, out, err, st);
    else
        pois_wpart_rk<T, 128>(X, ldx, V, W, m, n, r, S, out, err, st);
}

template void pois_vstep<float>(const float*, long long, const float*, const float*,
                                const double*, float*, long long, long long, int, double*,
                                unsigned int*, double*, int64_t*, cudaStream_t);
template void pois_vstep<double>(const double*, long long, const double*, const double*,
                                 const double*, double*, long long, long long, int, double*,
                                 unsigned int*, double*, int64_t*, cudaStream_t);
template void pois_wpart<float>(const float*, long long, const float*, const float*, long long,
                                long long, int, int, double*, int64_t*, cudaStream_t);
template void pois_wpart<double>(const double*, long long, const double*, const double*,
                                 long long, long long, int, int, double*, int64_t*, cudaStream_t);
template void vstep<float>(const float*, long long, const float*, const float*, const double*,
                           float*, long long, long long, int, int, double*, unsigned int*,
                           double*, cudaStream_t);
template void vstep<double>(const double*, long long, const double*, const double*,
                            const double*, double*, long long, long long, int, int, double*,
                            unsigned int*, double*, cudaStream_t);
template int wpart_splits<float>(long long, long long, int);
template int wpart_splits<double>(long long, long long, int);
template void wpart<float>(const float*, long long, const float*, long long, long long, int, int,
                           double*, cudaStream_t);
template void wpart<double>(const double*, long long, const double*, long long, long long, int,
                            int, double*, cudaStream_t);

}  // namespace mmk_tile
