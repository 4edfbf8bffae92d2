// nnmf.cu -- Lee-Seung multiplicative MM for the Frobenius loss (reference
// nnmf.py:75-156), CUDA-core (FFMA/DFMA) path.
//
// One MM iteration from (V, W), X m x n, rank r:
//   gram_kernel<rows>  G_W = W W^T                          (fp64, split-K)
//   nnmf_vstep_kernel  per row i of X (one warp per row, W staged in smem):
//                        q_i  = X_i W^T                       (r dot products)
//                        res += sum_j (x_ij - v_i . w_j)^2    (objective at (V,W), fp64)
//                        v_i' = v_i * q_i / (v_i G_W + 1e-300)
//   gram_kernel<cols>  G_V = V'^T V'                        (fp64, split-K)
//   nnmf_wpart_kernel  P = V'^T X, split over row ranges (deterministic partials)
//   nnmf_wreduce_kernel  partials -> red[P]
//   nnmf_wfinish_kernel  W' = W * P / (G_V W + 1e-300)
// The reference groups the denominators as (VW)W^T and V^T(VW)
// (nnmf.py:93-94, 107-108); G_W = W W^T and G_V = V^T V give the same values
// up to rounding with O((m+n) r^2) instead of O(m n r) work.
//
// Multi-GPU: rows of X/V are sharded; phase A ends with this rank's
// red = [P | G_V | f-partial]; the caller all-reduces red; phase B finishes
// W' redundantly on every rank.  See nnmf_tc.cu for the tcgen05 path used for
// large r (3xTF32 contraction of X on the tensor cores).
#include "mmk_common.cuh"
#include "nnmf_tc.h"
#include "nnmf_tile.h"

namespace mmk_ref {   // nnmf_ref.cu: fp64 single ops in the reference's arithmetic order
size_t ws_bytes(long long m, long long n, long long r);
int objective(const double* X, long long ldx, const double* V, const double* W, long long m,
              long long n, long long r, void* ws, double* f_dev, cudaStream_t st);
int update_v(const double* X, long long ldx, const double* V, const double* W, double* Vout,
             long long m, long long n, long long r, void* ws, cudaStream_t st);
int update_w(const double* X, long long ldx, const double* V, const double* W, double* Wout,
             long long m, long long n, long long r, void* ws, cudaStream_t st);
int gradient(const double* X, long long ldx, const double* V, const double* W, double* GV,
             double* GW, long long m, long long n, long long r, void* ws, cudaStream_t st);
}  // namespace mmk_ref

#include <type_traits>

namespace {

using namespace mmk;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
enum { VSTEP_UPDATE = 1, VSTEP_RESID = 2, VSTEP_GRAD = 4 };

// ---------------------------------------------------------------------------
// G[a][b] = sum_c A(a, c) A(b, c); VEC_ROWS: A is r x len (vectors are rows,
// W), else A is len x r (vectors are columns, V).
template <typename T, int RMAX, bool VEC_ROWS>
__global__ void __launch_bounds__(kThreads)
gram_kernel(const T* __restrict__ A, long long len, int r, int chunks_per_block,
            double* __restrict__ part, unsigned int* counter, double* __restrict__ out) {
    constexpr int PMAX = (RMAX * RMAX + kThreads - 1) / kThreads;
    __shared__ T S[RMAX][33];
    double acc[PMAX];
#pragma unroll
    for (int t = 0; t < PMAX; ++t) acc[t] = 0.0;
    const long long c_begin = (long long)blockIdx.x * chunks_per_block * 32;
    const int rr = r * r;
    for (int ch = 0; ch < chunks_per_block; ++ch) {
        const long long c0 = c_begin + (long long)ch * 32;
        if (c0 >= len) break;
        for (int idx = threadIdx.x; idx < r * 32; idx += kThreads) {
            int a, cc;
            if (VEC_ROWS) {
                a = idx >> 5;
                cc = idx & 31;
            } else {
                cc = idx / r;
                a = idx - cc * r;
            }
            const long long c = c0 + cc;
            T v = T(0);
            if (c < len) v = VEC_ROWS ? A[(long long)a * len + c] : A[c * r + a];
            S[a][cc] = v;
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < PMAX; ++t) {
            const int pidx = threadIdx.x + t * kThreads;
            if (pidx < rr) {
                const int a = pidx / r, b = pidx - a * r;
                double s = 0.0;
#pragma unroll 8
                for (int cc = 0; cc < 32; ++cc) s = fma((double)S[a][cc], (double)S[b][cc], s);
                acc[t] += s;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < PMAX; ++t) {
        const int pidx = threadIdx.x + t * kThreads;
        if (pidx < rr) part[(long long)blockIdx.x * rr + pidx] = acc[t];
    }
    if (arrive_last(counter, gridDim.x)) {
        for (int pidx = threadIdx.x; pidx < rr; pidx += kThreads) {
            double s = 0.0;
            for (unsigned int b = 0; b < gridDim.x; ++b) s += part[(long long)b * rr + pidx];
            out[pidx] = s;
        }
    }
}

// Rank-64 Gram with 4x4 register tiles per thread (16 x 16 threads cover the
// 64 x 64 output); 32 samples per smem stage.  Same deterministic split-K
// reduction as gram_kernel.
template <typename T, bool VEC_ROWS>
__global__ void __launch_bounds__(kThreads)
gram64_kernel(const T* __restrict__ A, long long len, int chunks_per_block,
              double* __restrict__ part, unsigned int* counter, double* __restrict__ out) {
    __shared__ double S[32][64 + 2];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    const long long c_begin = (long long)blockIdx.x * chunks_per_block * 32;
    for (int ch = 0; ch < chunks_per_block; ++ch) {
        const long long c0 = c_begin + (long long)ch * 32;
        if (c0 >= len) break;
        for (int idx = threadIdx.x; idx < 32 * 64; idx += kThreads) {
            int a, cc;
            if (VEC_ROWS) {
                a = idx >> 5;
                cc = idx & 31;
            } else {
                cc = idx >> 6;
                a = idx & 63;
            }
            const long long c = c0 + cc;
            double v = 0.0;
            if (c < len) v = (double)(VEC_ROWS ? A[(long long)a * len + c] : A[c * 64 + a]);
            S[cc][a] = v;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < 32; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                av[i] = S[kk][4 * ty + i];
                bv[i] = S[kk][4 * tx + i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    double* pb = part + (long long)blockIdx.x * 4096;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) pb[(4 * ty + i) * 64 + 4 * tx + j] = acc[i][j];
    (void)counter;
    (void)out;
}

// out[p] = sum_b part[b][p] in block order (one thread per output element)
__global__ void gram_reduce_kernel(const double* __restrict__ part, int nparts, int len,
                                   double* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= len) return;
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[(long long)b * len + p];
    out[p] = s;
}

// ---------------------------------------------------------------------------
template <typename T, int RMAX, int RPW, bool WFULL>
__global__ void __launch_bounds__(kThreads)
nnmf_vstep_kernel(const T* __restrict__ X, long long ldx, const T* __restrict__ V,
                  const T* __restrict__ W, const double* __restrict__ GW, T* __restrict__ Vout,
                  long long m, long long n, int r, int flags, double* __restrict__ respart,
                  unsigned int* counter, double* res_out) {
    // WFULL: all of W (r x n) staged in shared memory once (small problems,
    // e.g. the paper shape), no per-chunk barriers; else 32-column chunks
    extern __shared__ __align__(16) unsigned char vstep_smem[];
    __shared__ T Ws[WFULL ? 1 : RMAX][33];
    __shared__ T qs[kWarps][RPW][RMAX];
    __shared__ double sc[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long i0 = ((long long)blockIdx.x * kWarps + warp) * RPW;
    const bool resid = flags & VSTEP_RESID;

    T q[RPW][RMAX];
    T v[RPW][RMAX];
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const long long i = i0 + rr < m ? i0 + rr : m - 1;
#pragma unroll
        for (int k = 0; k < RMAX; ++k) {
            q[rr][k] = T(0);
            v[rr][k] = (k < r) ? V[i * r + k] : T(0);
        }
    }
    double res = 0.0;
    if (WFULL) {
        T* Wf = reinterpret_cast<T*>(vstep_smem);
        for (long long idx = threadIdx.x; idx < (long long)r * n; idx += kThreads) Wf[idx] = W[idx];
        __syncthreads();
        for (long long j = lane; j < n; j += 32) {
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const long long i = i0 + rr;
                if (i < m) {
                    const T x = X[i * ldx + j];
                    T rec = T(0);
#pragma unroll
                    for (int k = 0; k < RMAX; ++k) {
                        if (k < r) {
                            const T w = Wf[(long long)k * n + j];
                            q[rr][k] = fma(x, w, q[rr][k]);
                            rec = fma(v[rr][k], w, rec);
                        }
                    }
                    if (resid) {
                        const double d = (double)x - (double)rec;
                        res = fma(d, d, res);
                    }
                }
            }
        }
    } else {
    for (long long j0 = 0; j0 < n; j0 += 32) {
        for (int idx = threadIdx.x; idx < r * 32; idx += kThreads) {
            const int k = idx >> 5, c = idx & 31;
            Ws[k][c] = (j0 + c < n) ? W[(long long)k * n + j0 + c] : T(0);
        }
        __syncthreads();
        const long long j = j0 + lane;
        if (j < n) {
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const long long i = i0 + rr;
                if (i < m) {
                    const T x = X[i * ldx + j];
                    T rec = T(0);
#pragma unroll
                    for (int k = 0; k < RMAX; ++k) {
                        if (k < r) {
                            const T w = Ws[k][lane];
                            q[rr][k] = fma(x, w, q[rr][k]);
                            rec = fma(v[rr][k], w, rec);
                        }
                    }
                    if (resid) {
                        const double d = (double)x - (double)rec;
                        res = fma(d, d, res);
                    }
                }
            }
        }
        __syncthreads();
    }
    }
    if (flags & VSTEP_UPDATE) {
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
#pragma unroll
            for (int k = 0; k < RMAX; ++k) {
                if (k < r) {
                    const T t = warp_sum(q[rr][k]);
                    if ((k & 31) == lane) qs[warp][rr][k] = t;
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            const long long i = i0 + rr;
            if (i >= m) continue;
            for (int k = lane; k < r; k += 32) {
                double den = 0.0;
#pragma unroll
                for (int l = 0; l < RMAX; ++l)
                    if (l < r) den = fma((double)v[rr][l], GW[l * r + k], den);
                if (flags & VSTEP_GRAD) {   // 2 (V G_W - X W^T) = 2 (V W - X) W^T
                    Vout[i * r + k] = (T)(2.0 * (den - (double)qs[warp][rr][k]));
                    continue;
                }
                const double vk = (double)V[i * r + k];
                Vout[i * r + k] = (T)(vk * ((double)qs[warp][rr][k] / (den + kDenomGuard)));
            }
        }
    }
    if (!resid) return;
    const double bs = block_sum(res, sc);
    if (threadIdx.x == 0) respart[blockIdx.x] = bs;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(respart, gridDim.x, sc);
        if (threadIdx.x == 0) *res_out = tot;
    }
}

// ---------------------------------------------------------------------------
// P[k][j] partial over rows [s*rows_per_split, ...) of sum_i V[i][k] X[i][j]
template <typename T, int RMAX>
__global__ void __launch_bounds__(kThreads)
nnmf_wpart_kernel(const T* __restrict__ X, long long ldx, const T* __restrict__ V, long long m,
                  long long n, int r, long long rows_per_split, double* __restrict__ out) {
    __shared__ T red[kWarps][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long j = (long long)blockIdx.x * 32 + lane;
    const long long lo = (long long)blockIdx.y * rows_per_split;
    const long long hi = min(m, lo + rows_per_split);
    T acc[RMAX];
#pragma unroll
    for (int k = 0; k < RMAX; ++k) acc[k] = T(0);
    if (j < n) {
        for (long long i = lo + warp; i < hi; i += kWarps) {
            const T x = X[i * ldx + j];
            const T* vi = V + i * r;
#pragma unroll
            for (int k = 0; k < RMAX; ++k)
                if (k < r) acc[k] = fma(vi[k], x, acc[k]);
        }
    }
    double* o = out + (long long)blockIdx.y * r * n;
#pragma unroll
    for (int k = 0; k < RMAX; ++k) {
        if (k < r) {
            red[warp][lane] = acc[k];
            __syncthreads();
            if (warp == 0 && j < n) {
                double s = 0.0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) s += (double)red[w][lane];
                o[(long long)k * n + j] = s;
            }
            __syncthreads();
        }
    }
}

__global__ void nnmf_wreduce_kernel(const double* __restrict__ part, int S, long long len,
                                    double* __restrict__ red) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= len) return;
    double s = 0.0;
    for (int k = 0; k < S; ++k) s += part[(long long)k * len + t];
    red[t] = s;
}

// GRAD: write 2 (G_V W - V^T X) = 2 V^T (V W - X) instead of the update
template <typename T, bool GRAD = false>
__global__ void nnmf_wfinish_kernel(const T* __restrict__ W, T* __restrict__ Wout, long long n,
                                    int r, const double* __restrict__ red, double* f_dev,
                                    const long long* __restrict__ skip = nullptr) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long rn = (long long)r * n;
    if (f_dev && t == 0) *f_dev = red[rn + (long long)r * r];
    if (t >= rn || (skip && *skip)) return;   // skip: the engine's final pass needs only f
    const int k = (int)(t / n);
    const long long j = t - (long long)k * n;
    const double* G = red + rn + (long long)k * r;
    double den = 0.0;
    for (int l = 0; l < r; ++l) den = fma(G[l], (double)W[(long long)l * n + j], den);
    if (GRAD)
        Wout[t] = (T)(2.0 * (den - red[t]));
    else
        Wout[t] = (T)((double)W[t] * (red[t] / (den + kDenomGuard)));
}

// Rank-64 W finish: a block owns 64 columns; G^T and the W slab (fp64) sit in
// shared memory and each thread forms a 4 x 4 register tile of denominators
// (G_V W)[k][j] in fp64, then W' = W * P / (den + guard).
constexpr int kWf64Smem = 2 * 64 * 64 * 8;
template <typename T>
__global__ void __launch_bounds__(256)
nnmf_wfinish64_kernel(const T* __restrict__ W, T* __restrict__ Wout, long long n,
                      const double* __restrict__ red, double* f_dev,
                      const long long* __restrict__ skip) {
    extern __shared__ double wf_smem[];
    double(*Gt)[64] = reinterpret_cast<double(*)[64]>(wf_smem);            // Gt[l][k] = G[k][l]
    double(*Ws)[64] = reinterpret_cast<double(*)[64]>(wf_smem + 64 * 64);  // Ws[l][j]
    const long long rn = 64 * n;
    if (f_dev && blockIdx.x == 0 && threadIdx.x == 0) *f_dev = red[rn + 64 * 64];
    if (skip && *skip) return;   // the engine's final pass (iteration cap) needs only f
    const long long j0 = (long long)blockIdx.x * 64;
    for (int i = threadIdx.x; i < 64 * 64; i += 256) {
        const int k = i / 64, l = i % 64;
        Gt[l][k] = red[rn + i];
        const int jj = i % 64, r = i / 64;
        Ws[r][jj] = (j0 + jj < n) ? (double)W[(long long)r * n + j0 + jj] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll 8
    for (int l = 0; l < 64; ++l) {
        const double2 a01 = *reinterpret_cast<const double2*>(&Gt[l][4 * ty]);
        const double2 a23 = *reinterpret_cast<const double2*>(&Gt[l][4 * ty + 2]);
        const double2 b01 = *reinterpret_cast<const double2*>(&Ws[l][4 * tx]);
        const double2 b23 = *reinterpret_cast<const double2*>(&Ws[l][4 * tx + 2]);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y};
        const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = 4 * ty + i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long col = j0 + 4 * tx + j;
            if (col < n)
                Wout[(long long)k * n + col] =
                    (T)(Ws[k][4 * tx + j] * (red[(long long)k * n + col] / (acc[i][j] + kDenomGuard)));
        }
    }
}

// The same for ranks 65..128 at the 128-rank tile (G^T 128 KB + the W slab 64
// KB of shared memory, zero beyond r; 8 x 4 register tiles, l ascending as
// nnmf_wfinish_kernel, so the denominators are the same fp64 sums).
constexpr int kWf128Smem = (128 * 128 + 128 * 64) * 8;
template <typename T>
__global__ void __launch_bounds__(256)
nnmf_wfinish128_kernel(const T* __restrict__ W, T* __restrict__ Wout, long long n, int r,
                       const double* __restrict__ red, double* f_dev,
                       const long long* __restrict__ skip) {
    extern __shared__ double wf_smem[];
    double(*Gt)[128] = reinterpret_cast<double(*)[128]>(wf_smem);            // Gt[l][k] = G[k][l]
    double(*Ws)[64] = reinterpret_cast<double(*)[64]>(wf_smem + 128 * 128);  // Ws[l][j]
    const long long rn = (long long)r * n;
    if (f_dev && blockIdx.x == 0 && threadIdx.x == 0) *f_dev = red[rn + (long long)r * r];
    if (skip && *skip) return;   // the engine's final pass (iteration cap) needs only f
    const long long j0 = (long long)blockIdx.x * 64;
    for (int i = threadIdx.x; i < 128 * 128; i += 256) {
        const int l = i / 128, k = i % 128;
        Gt[l][k] = (k < r && l < r) ? red[rn + (long long)k * r + l] : 0.0;
    }
    for (int i = threadIdx.x; i < 128 * 64; i += 256) {
        const int l = i / 64, jj = i % 64;
        Ws[l][jj] = (l < r && j0 + jj < n) ? (double)W[(long long)l * n + j0 + jj] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // ranks 8 ty .., columns 4 tx ..
    double acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll 4
    for (int l = 0; l < 128; ++l) {
        double av[8], bv[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const double2 a = *reinterpret_cast<const double2*>(&Gt[l][8 * ty + 2 * h]);
            av[2 * h] = a.x, av[2 * h + 1] = a.y;
        }
        const double2 b01 = *reinterpret_cast<const double2*>(&Ws[l][4 * tx]);
        const double2 b23 = *reinterpret_cast<const double2*>(&Ws[l][4 * tx + 2]);
        bv[0] = b01.x, bv[1] = b01.y, bv[2] = b23.x, bv[3] = b23.y;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int k = 8 * ty + i;
        if (k >= r) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long col = j0 + 4 * tx + j;
            if (col < n)
                Wout[(long long)k * n + col] =
                    (T)(Ws[k][4 * tx + j] * (red[(long long)k * n + col] / (acc[i][j] + kDenomGuard)));
        }
    }
}

// ---------------------------------------------------------------------------
struct Plan {
    int g64w_blocks, g64w_cpb, g64v_blocks, g64v_cpb;   // rank-64 Gram split-K
    int rpw, nvb;            // vstep rows per warp, blocks
    int gw_blocks, gw_cpb;   // gram over W (len n)
    int gv_blocks, gv_cpb;   // gram over V (len m)
    int S;                   // W-step row splits
    long long rows_per_split;
    int colblocks;
    int Sd;                  // fp64 DMMA W part: max row splits (partial buffer bound)
};

struct Ws {
    unsigned int* counters;  // [0] vstep, [1] gram W, [2] gram V
    double* GW;
    double* gpart;
    double* respart;
    double* wpart;
    double* fscratch;
    void* tc;                // tensor-core path scratch (fp32 ranks 17..128)
};

// the tensor-core region (pre-split X, operand copies) is reserved only for
// workspaces of a full iteration (iter_a) whose dtype / shape can take the
// tensor-core path; single ops (update_v/w, objective, gradient) run the SIMT
// kernels and size their workspace without it (mmk_nnmf_op_ws_bytes)
bool tc_region(int dtype, long long m, long long n, int r, bool iter) {
    return iter && mmk_tc::shape_ok(dtype, m, n, r);
}

Plan make_plan(long long m, long long n, int r, int dtype) {
    Plan P;
    P.rpw = r <= 16 ? 2 : 1;
    P.nvb = ceil_div(m > 0 ? m : 1, kWarps * P.rpw);
    const int nch_w = ceil_div(n, 32), nch_v = ceil_div(m > 0 ? m : 1, 32);
    P.gw_blocks = nch_w < kNumSMs ? nch_w : kNumSMs;
    P.gw_cpb = ceil_div(nch_w, P.gw_blocks);
    P.gw_blocks = ceil_div(nch_w, P.gw_cpb);
    P.gv_blocks = nch_v < kNumSMs ? nch_v : kNumSMs;
    P.gv_cpb = ceil_div(nch_v, P.gv_blocks);
    P.gv_blocks = ceil_div(nch_v, P.gv_cpb);
    P.g64w_blocks = nch_w < 4 * kNumSMs ? nch_w : 4 * kNumSMs;
    P.g64w_cpb = ceil_div(nch_w, P.g64w_blocks);
    P.g64w_blocks = ceil_div(nch_w, P.g64w_cpb);
    P.g64v_blocks = nch_v < 4 * kNumSMs ? nch_v : 4 * kNumSMs;
    P.g64v_cpb = ceil_div(nch_v, P.g64v_blocks);
    P.g64v_blocks = ceil_div(nch_v, P.g64v_cpb);
    P.colblocks = ceil_div(n, 32);
    long long S = ceil_div(4 * kNumSMs, P.colblocks);
    long long smax = ceil_div(m > 0 ? m : 1, 64);
    if (S > smax) S = smax;
    if (S < 1) S = 1;
    P.rows_per_split = ceil_div(m > 0 ? m : 1, S);
    P.S = ceil_div(m > 0 ? m : 1, P.rows_per_split);
    // fp64 ranks 17..128 run the DMMA tiles, whose W part picks up to
    // kDmmaMaxSplits row splits (wpart_splits_dmma); other paths use P.S
    P.Sd = (dtype == MMK_F64 && mmk_tile::applies(r)) ? mmk_tile::kDmmaMaxSplits : 1;
    return P;
}

size_t ws_layout(const Plan& P, long long m, long long n, int r, bool tc, void* base, Ws* L) {
    size_t off = 256;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    const size_t rr = (size_t)r * r;
    int gblocks = P.gw_blocks > P.gv_blocks ? P.gw_blocks : P.gv_blocks;
    if (P.g64w_blocks > gblocks) gblocks = P.g64w_blocks;
    if (P.g64v_blocks > gblocks) gblocks = P.g64v_blocks;
    size_t o_gw = take(sizeof(double) * rr);
    size_t o_gp = take(sizeof(double) * rr * gblocks);
    size_t o_rp = take(sizeof(double) * (size_t)P.nvb);
    size_t o_f = take(sizeof(double) * 4);
    const int sw = P.S > P.Sd ? P.S : P.Sd;   // split-K partials (SIMT / FMA tiles, or DMMA)
    size_t o_wp = take(sw > 1 ? sizeof(double) * (size_t)sw * r * (size_t)n : 0);
    size_t o_tc = take(tc ? mmk_tc::ws_bytes(m, n, r) : 0);
    if (base && L) {
        L->tc = reinterpret_cast<char*>(base) + o_tc;
        char* c = reinterpret_cast<char*>(base);
        L->counters = reinterpret_cast<unsigned int*>(c);
        L->GW = reinterpret_cast<double*>(c + o_gw);
        L->gpart = reinterpret_cast<double*>(c + o_gp);
        L->respart = reinterpret_cast<double*>(c + o_rp);
        L->fscratch = reinterpret_cast<double*>(c + o_f);
        L->wpart = reinterpret_cast<double*>(c + o_wp);
    }
    return off;
}

constexpr int kMaxRank = 128;
constexpr size_t kWFullBytes = 96 * 1024;   // stage all of W when it fits

template <typename T, int RMAX>
struct K {
    static void gram64(const T* A, long long len, bool rows, int blocks, int cpb, const Ws& L,
                       double* out, cudaStream_t st) {
        if (rows)
            MMK_LAUNCH("nnmf_gram64", st,
                       (gram64_kernel<T, true><<<blocks, kThreads, 0, st>>>(A, len, cpb, L.gpart,
                                                                            nullptr, nullptr)));
        else
            MMK_LAUNCH("nnmf_gram64", st,
                       (gram64_kernel<T, false><<<blocks, kThreads, 0, st>>>(A, len, cpb, L.gpart,
                                                                             nullptr, nullptr)));
        MMK_LAUNCH("nnmf_gram_reduce",
                   st, (gram_reduce_kernel<<<16, 256, 0, st>>>(L.gpart, blocks, 4096, out)));
    }
    static void gram_w(const T* W, long long n, int r, const Plan& P, const Ws& L, cudaStream_t st) {
        if (RMAX == 64 && r == 64) {
            gram64(W, n, true, P.g64w_blocks, P.g64w_cpb, L, L.GW, st);
            return;
        }
        MMK_LAUNCH("nnmf_gram_w", st,
                   (gram_kernel<T, RMAX, true><<<P.gw_blocks, kThreads, 0, st>>>(
                       W, n, r, P.gw_cpb, L.gpart, L.counters + 1, L.GW)));
    }
    static void gram_v(const T* V, long long m, int r, const Plan& P, const Ws& L, double* out,
                       cudaStream_t st) {
        if (RMAX == 64 && r == 64) {
            gram64(V, m, false, P.g64v_blocks, P.g64v_cpb, L, out, st);
            return;
        }
        MMK_LAUNCH("nnmf_gram_v", st,
                   (gram_kernel<T, RMAX, false><<<P.gv_blocks, kThreads, 0, st>>>(
                       V, m, r, P.gv_cpb, L.gpart, L.counters + 2, out)));
    }
    static void vstep(const T* X, long long ldx, const T* V, const T* W, T* Vout, long long m,
                      long long n, int r, int flags, const Plan& P, const Ws& L, double* res_out,
                      cudaStream_t st) {
        if (RMAX > 16 && mmk_tile::applies(r)) {   // ranks 17..128: nnmf_tile.cu
            mmk_tile::vstep<T>(X, ldx, V, W, L.GW, Vout, m, n, r, flags, L.respart, L.counters,
                               res_out, st);
            return;
        }
        const size_t wbytes = sizeof(T) * (size_t)r * (size_t)n;
        const bool full = wbytes <= kWFullBytes;
        if constexpr (RMAX <= 16) {
            if (P.rpw == 2) {
                if (full) {
                    if (mmk_host::first_on_device(
                            reinterpret_cast<const void*>(nnmf_vstep_kernel<T, RMAX, 2, true>))) {
                        cudaFuncSetAttribute(nnmf_vstep_kernel<T, RMAX, 2, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kWFullBytes);
                    }
                    MMK_LAUNCH("nnmf_vstep", st,
                               (nnmf_vstep_kernel<T, RMAX, 2, true><<<P.nvb, kThreads, wbytes, st>>>(
                                   X, ldx, V, W, L.GW, Vout, m, n, r, flags, L.respart, L.counters,
                                   res_out)));
                    return;
                }
                MMK_LAUNCH("nnmf_vstep", st,
                           (nnmf_vstep_kernel<T, RMAX, 2, false><<<P.nvb, kThreads, 0, st>>>(
                               X, ldx, V, W, L.GW, Vout, m, n, r, flags, L.respart, L.counters,
                               res_out)));
                return;
            }
        }
            MMK_LAUNCH("nnmf_vstep", st,
                       (nnmf_vstep_kernel<T, RMAX, 1, false><<<P.nvb, kThreads, 0, st>>>(
                           X, ldx, V, W, L.GW, Vout, m, n, r, flags, L.respart, L.counters,
                           res_out)));
    }
    static void wpart(const T* X, long long ldx, const T* V, long long m, long long n, int r,
                      const Plan& P, const Ws& L, double* red, cudaStream_t st) {
        if (RMAX > 16 && mmk_tile::applies(r)) {   // ranks 17..128: nnmf_tile.cu
            const int S = std::is_same<T, double>::value
                              ? mmk_tile::wpart_splits_dmma(m, n, r, P.Sd)
                              : mmk_tile::wpart_splits<T>(m, n, P.S);
            mmk_tile::wpart<T>(X, ldx, V, m, n, r, S, S > 1 ? L.wpart : red, st);
            if (S > 1) {
                const long long len = (long long)r * n;
                MMK_LAUNCH("nnmf_wreduce", st,
                           (nnmf_wreduce_kernel<<<ceil_div(len, 256), 256, 0, st>>>(L.wpart, S,
                                                                                   len, red)));
            }
            return;
        }
        dim3 grid(P.colblocks, P.S);
        double* dst = P.S > 1 ? L.wpart : red;
        MMK_LAUNCH("nnmf_wpart", st,
                   (nnmf_wpart_kernel<T, RMAX><<<grid, kThreads, 0, st>>>(
                       X, ldx, V, m, n, r, P.rows_per_split, dst)));
        if (P.S > 1) {
            const long long len = (long long)r * n;
            MMK_LAUNCH("nnmf_wreduce", st,
                       (nnmf_wreduce_kernel<<<ceil_div(len, 256), 256, 0, st>>>(L.wpart, P.S,
                                                                               len, red)));
        }
    }
};

// Runs `fn<T, RMAX>()` for the rank bucket of r.
template <typename T, template <typename, int> class F, typename... A>
int dispatch_rank(int r, A... args) {
    if (r <= 4) return F<T, 4>::run(args...);
    if (r <= 8) return F<T, 8>::run(args...);
    if (r <= 16) return F<T, 16>::run(args...);
    if (r <= 32) return F<T, 32>::run(args...);
    if (r <= 64) return F<T, 64>::run(args...);
    return F<T, 128>::run(args...);
}

struct Args {
    const void *X, *V, *W;
    void *V_out, *W_out;
    long long ldx, m, n;
    int r;
    void* ws;
    double* red;
    double* f_dev;
    int64_t* err;
    cudaStream_t st;
    int mode;  // 0 iter_a, 1 update_v, 2 objective, 3 update_w (a + b), 4 gradient
};

template <typename T, int RMAX>
struct RunA {
    static int run(const Args& a) {
        const int dt = std::is_same<T, float>::value ? MMK_F32 : MMK_F64;
        const Plan P = make_plan(a.m, a.n, a.r, dt);
        Ws L;
        ws_layout(P, a.m, a.n, a.r, tc_region(dt, a.m, a.n, a.r, a.mode == 0), a.ws, &L);
        using KK = K<T, RMAX>;
        const T* X = (const T*)a.X;
        const T* V = (const T*)a.V;
        const T* W = (const T*)a.W;
        const long long rn = (long long)a.r * a.n;
        if constexpr (std::is_same<T, float>::value && (RMAX == 32 || RMAX == 64 || RMAX == 128)) {
            if (a.mode == 0 && tc_region(MMK_F32, a.m, a.n, a.r, true) &&
                mmk_tc::eligible(MMK_F32, a.m, a.n, a.r, a.ldx, a.X)) {
                return mmk_tc::iter_a(X, a.ldx, V, W, (float*)a.V_out, a.m, a.n, a.r, L.tc,
                                      L.GW, a.red, a.st);
            }
        }
        if (a.mode == 0 || a.mode == 1 || a.mode == 2 || a.mode == 4) {
            if (a.m > 0) {
                if (a.mode != 2) KK::gram_w(W, a.n, a.r, P, L, a.st);
                int flags = (a.mode == 0)   ? (VSTEP_UPDATE | VSTEP_RESID)
                            : a.mode == 1 ? VSTEP_UPDATE
                            : a.mode == 4 ? (VSTEP_UPDATE | VSTEP_GRAD)
                                          : VSTEP_RESID;
                double* res_out = a.mode == 0 ? a.red + rn + (long long)a.r * a.r : a.f_dev;
                KK::vstep(X, a.ldx, V, W, (T*)a.V_out, a.m, a.n, a.r, flags, P, L, res_out, a.st);
            } else if (a.mode == 0) {
                cudaMemsetAsync(a.red + rn + (long long)a.r * a.r, 0, sizeof(double), a.st);
            } else if (a.mode == 2) {
                cudaMemsetAsync(a.f_dev, 0, sizeof(double), a.st);
            }
            MMK_CHECK_LAUNCH("nnmf_vstep");
        }
        if (a.mode == 0 || a.mode == 3 || a.mode == 4) {
            // W step uses the new V for iter_a, the given V for update_w / gradient
            const T* Vn = a.mode == 0 ? (const T*)a.V_out : V;
            if (a.m > 0) {
                KK::gram_v(Vn, a.m, a.r, P, L, a.red + rn, a.st);
                KK::wpart(X, a.ldx, Vn, a.m, a.n, a.r, P, L, a.red, a.st);
            } else {
                cudaMemsetAsync(a.red, 0, sizeof(double) * (size_t)(rn + (long long)a.r * a.r),
                                a.st);
            }
            if (a.mode == 3 || a.mode == 4)
                cudaMemsetAsync(a.red + rn + (long long)a.r * a.r, 0, sizeof(double), a.st);
            MMK_CHECK_LAUNCH("nnmf_wstep");
        }
        return MMK_OK;
    }
};

template <typename T>
int finish_b(const void* W, void* W_out, long long n, int r, const double* red, double* f_dev,
             cudaStream_t st, bool grad = false) {
    const long long rn = (long long)r * n;
    if (grad) {
        MMK_LAUNCH("nnmf_wgrad", st,
                   (nnmf_wfinish_kernel<T, true><<<ceil_div(rn, 256), 256, 0, st>>>(
                       (const T*)W, (T*)W_out, n, r, red, f_dev)));
        MMK_CHECK_LAUNCH("nnmf_wfinish_kernel<grad>");
        return MMK_OK;
    }
    if (r == 64) {
        if (mmk_host::first_on_device(reinterpret_cast<const void*>(nnmf_wfinish64_kernel<T>))) {
            cudaFuncSetAttribute(nnmf_wfinish64_kernel<T>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kWf64Smem);
        }
        MMK_LAUNCH("nnmf_wfinish", st,
                   (nnmf_wfinish64_kernel<T><<<ceil_div(n, 64), 256, kWf64Smem, st>>>(
                       (const T*)W, (T*)W_out, n, red, f_dev, mmk_tc::last_flag())));
        MMK_CHECK_LAUNCH("nnmf_wfinish64_kernel");
        return MMK_OK;
    }
    if (r > 64) {
        if (mmk_host::first_on_device(reinterpret_cast<const void*>(nnmf_wfinish128_kernel<T>))) {
            cudaFuncSetAttribute(nnmf_wfinish128_kernel<T>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kWf128Smem);
        }
        MMK_LAUNCH("nnmf_wfinish", st,
                   (nnmf_wfinish128_kernel<T><<<ceil_div(n, 64), 256, kWf128Smem, st>>>(
                       (const T*)W, (T*)W_out, n, r, red, f_dev, mmk_tc::last_flag())));
        MMK_CHECK_LAUNCH("nnmf_wfinish128_kernel");
        return MMK_OK;
    }
    MMK_LAUNCH("nnmf_wfinish", st,
               (nnmf_wfinish_kernel<T><<<ceil_div(rn, 256), 256, 0, st>>>(
                   (const T*)W, (T*)W_out, n, r, red, f_dev, mmk_tc::last_flag())));
    MMK_CHECK_LAUNCH("nnmf_wfinish_kernel");
    return MMK_OK;
}

// the fp64 single ops' reference-order region follows the op workspace
inline size_t ref_offset(size_t op_bytes) { return (op_bytes + 255) & ~size_t(255); }

int check(int dtype, long long m, long long n, long long r, long long ldx, size_t ws_bytes,
          bool iter) {
    if (dtype != MMK_F32 && dtype != MMK_F64) {
        mmk_host::set_error("unknown dtype %d", dtype);
        return MMK_E_SHAPE;
    }
    if (r < 1 || r > kMaxRank || n < 1 || m < 0 || ldx < n) {
        mmk_host::set_error("unsupported NNMF shape m=%lld n=%lld r=%lld ldx=%lld (rank <= %d)",
                            m, n, r, ldx, kMaxRank);
        return MMK_E_SHAPE;
    }
    const Plan P = make_plan(m, n, (int)r, dtype);
    size_t need = ws_layout(P, m, n, (int)r, tc_region(dtype, m, n, (int)r, iter), nullptr,
                            nullptr);
    if (!iter && dtype == MMK_F64) need = ref_offset(need) + mmk_ref::ws_bytes(m, n, r);
    if (ws_bytes < need) {
        mmk_host::set_error("NNMF workspace too small: %zu < %zu", ws_bytes, need);
        return MMK_E_SHAPE;
    }
    return MMK_OK;
}

int run_a(int dtype, Args a) {
    if (dtype == MMK_F32) return dispatch_rank<float, RunA>(a.r, a);
    return dispatch_rank<double, RunA>(a.r, a);
}

}  // namespace

void* mmk_tc::engine_tc_ws(int dtype, const void* X, long long ldx, long long m, long long n,
                          long long r, void* ws) {
    if (!tc_region(dtype, m, n, (int)r, true) || !eligible(MMK_F32, m, n, r, ldx, X))
        return nullptr;
    Ws L;
    ws_layout(make_plan(m, n, (int)r, dtype), m, n, (int)r, true, ws, &L);
    return L.tc;
}

static int ws_bytes_for(int dtype, int64_t m, int64_t n, int64_t r, bool iter, size_t* out) {
    if (r < 1 || r > kMaxRank || n < 1) {
        mmk_host::set_error("unsupported NNMF shape n=%lld r=%lld", (long long)n, (long long)r);
        return MMK_E_SHAPE;
    }
    const Plan P = make_plan(m, n, (int)r, dtype);
    *out = ws_layout(P, m, n, (int)r, tc_region(dtype, m, n, (int)r, iter), nullptr, nullptr);
    if (!iter && dtype == MMK_F64) *out = ref_offset(*out) + mmk_ref::ws_bytes(m, n, r);
    return MMK_OK;
}

extern "C" int mmk_nnmf_ws_bytes(int dtype, int64_t m, int64_t n, int64_t r, size_t* out) {
    return ws_bytes_for(dtype, m, n, r, true, out);
}

extern "C" int mmk_nnmf_op_ws_bytes(int dtype, int64_t m, int64_t n, int64_t r, size_t* out) {
    return ws_bytes_for(dtype, m, n, r, false, out);
}

extern "C" int mmk_nnmf_ws_clear(int dtype, int64_t m, int64_t n, int64_t r, void* ws,
                                 size_t ws_bytes, void* stream) {
    size_t need = 0;
    int rc = ws_bytes_for(dtype, m, n, r, true, &need);
    if (rc) return rc;
    if (ws_bytes < need) {
        mmk_host::set_error("NNMF workspace too small: %zu < %zu", ws_bytes, need);
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    char* c = reinterpret_cast<char*>(ws);
    size_t b = ws_bytes, e = ws_bytes;   // the span left as is (none by default)
    if (tc_region(dtype, m, n, (int)r, true)) {
        Ws L;
        ws_layout(make_plan(m, n, (int)r, dtype), m, n, (int)r, true, ws, &L);
        mmk_tc::presplit_span(m, n, &b, &e);
        b += (size_t)(reinterpret_cast<char*>(L.tc) - c);
        e += (size_t)(reinterpret_cast<char*>(L.tc) - c);
    }
    cudaError_t ce = cudaMemsetAsync(c, 0, b, st);
    if (ce == cudaSuccess && e < ws_bytes) ce = cudaMemsetAsync(c + e, 0, ws_bytes - e, st);
    if (ce != cudaSuccess) return mmk_host::cuda_status(ce, "mmk_nnmf_ws_clear");
    return MMK_OK;
}

// The per-X preparation of the tensor-core path (scale exponent, pre-split
// copy of X) enqueued on `stream` now -- a no-op when the path does not apply
// or X is already prepared in this workspace.  A run calls it before building
// its device-loop engine, so the GPU works while the host captures and
// instantiates the graph (the engine's own prologue then finds X prepared).
extern "C" int mmk_nnmf_prepare(int dtype, const void* X, int64_t ldx, int64_t m, int64_t n,
                                int64_t r, void* ws, size_t ws_bytes, void* stream) {
    MMK_NVTX("mmk_nnmf_prepare");
    int rc = check(dtype, m, n, r, ldx, ws_bytes, true);
    if (rc) return rc;
    void* tcws = mmk_tc::engine_tc_ws(dtype, X, ldx, m, n, r, ws);
    if (!tcws) return MMK_OK;
    return mmk_tc::prepare_x(reinterpret_cast<const float*>(X), ldx, m, n, tcws,
                             reinterpret_cast<cudaStream_t>(stream));
}

// [P (r n) | G (r r) | f | device-error flag]
extern "C" int64_t mmk_nnmf_reduce_len(int64_t n, int64_t r) { return r * n + r * r + 2; }

extern "C" int mmk_nnmf_iter_a(int dtype, const void* X, int64_t ldx, const void* V,
                               const void* W, void* V_out, int64_t m, int64_t n, int64_t r,
                               void* ws, size_t ws_bytes, double* red, int64_t* err_dev,
                               void* stream) {
    MMK_NVTX("mmk_nnmf_iter_a");
    int rc = check(dtype, m, n, r, ldx, ws_bytes, true);
    if (rc) return rc;
    Args a{X, V, W, V_out, nullptr, ldx, m, n, (int)r, ws, red, nullptr, err_dev,
           reinterpret_cast<cudaStream_t>(stream), 0};
    rc = run_a(dtype, a);
    if (rc) return rc;
    mmk_host::err_flag(err_dev, red + mmk_nnmf_reduce_len(n, r) - 1, a.st);
    return MMK_OK;
}

extern "C" int mmk_nnmf_iter_b(int dtype, const void* W, void* W_out, int64_t n, int64_t r,
                               const double* red, double* f_dev, int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_nnmf_iter_b");
    if (r < 1 || n < 1) {
        mmk_host::set_error("bad NNMF shape n=%lld r=%lld", (long long)n, (long long)r);
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    mmk_host::peer_err(red + mmk_nnmf_reduce_len(n, r) - 1, err_dev, st);
    if (dtype == MMK_F32) return finish_b<float>(W, W_out, n, (int)r, red, f_dev, st);
    if (dtype == MMK_F64) return finish_b<double>(W, W_out, n, (int)r, red, f_dev, st);
    mmk_host::set_error("unknown dtype %d", dtype);
    return MMK_E_SHAPE;
}

extern "C" int mmk_nnmf_iter(int dtype, const void* X, int64_t ldx, const void* V, const void* W,
                             void* V_out, void* W_out, int64_t m, int64_t n, int64_t r, void* ws,
                             size_t ws_bytes, double* red, double* f_dev, int64_t* err_dev,
                             void* stream) {
    MMK_NVTX("mmk_nnmf_iter");
    mmk_host::NoFlag one_gpu;   // no collective between the phases
    int rc = mmk_nnmf_iter_a(dtype, X, ldx, V, W, V_out, m, n, r, ws, ws_bytes, red, err_dev,
                             stream);
    if (rc) return rc;
    return mmk_nnmf_iter_b(dtype, W, W_out, n, r, red, f_dev, err_dev, stream);
}

// the reference-order region of a single-op workspace (fp64)
static void* ref_ws(void* ws, long long m, long long n, long long r) {
    const size_t opb = ws_layout(make_plan(m, n, (int)r, MMK_F64), m, n, (int)r, false, nullptr,
                                 nullptr);
    return reinterpret_cast<char*>(ws) + ref_offset(opb);
}

// fp64 single operations run in the reference's arithmetic order
// (nnmf_ref.cu: bitwise equal to mmkit's); fp32 ones on the fused kernels
extern "C" int mmk_nnmf_objective(int dtype, const void* X, int64_t ldx, const void* V,
                                  const void* W, int64_t m, int64_t n, int64_t r, void* ws,
                                  size_t ws_bytes, double* f_dev, int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_nnmf_objective");
    int rc = check(dtype, m, n, r, ldx, ws_bytes, false);
    if (rc) return rc;
    if (dtype == MMK_F64)
        return mmk_ref::objective((const double*)X, ldx, (const double*)V, (const double*)W, m,
                                  n, r, ref_ws(ws, m, n, r), f_dev,
                                  reinterpret_cast<cudaStream_t>(stream));
    Args a{X, V, W, nullptr, nullptr, ldx, m, n, (int)r, ws, nullptr, f_dev, err_dev,
           reinterpret_cast<cudaStream_t>(stream), 2};
    return run_a(dtype, a);
}

extern "C" int mmk_nnmf_update_v(int dtype, const void* X, int64_t ldx, const void* V,
                                 const void* W, void* V_out, int64_t m, int64_t n, int64_t r,
                                 void* ws, size_t ws_bytes, int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_nnmf_update_v");
    int rc = check(dtype, m, n, r, ldx, ws_bytes, false);
    if (rc) return rc;
    if (dtype == MMK_F64)
        return mmk_ref::update_v((const double*)X, ldx, (const double*)V, (const double*)W,
                                 (double*)V_out, m, n, r, ref_ws(ws, m, n, r),
                                 reinterpret_cast<cudaStream_t>(stream));
    Args a{X, V, W, V_out, nullptr, ldx, m, n, (int)r, ws, nullptr, nullptr, err_dev,
           reinterpret_cast<cudaStream_t>(stream), 1};
    return run_a(dtype, a);
}

extern "C" int mmk_nnmf_update_w(int dtype, const void* X, int64_t ldx, const void* V,
                                 const void* W, void* W_out, int64_t m, int64_t n, int64_t r,
                                 void* ws, size_t ws_bytes, double* red, int64_t* err_dev,
                                 void* stream) {
    MMK_NVTX("mmk_nnmf_update_w");
    int rc = check(dtype, m, n, r, ldx, ws_bytes, false);
    if (rc) return rc;
    if (dtype == MMK_F64)
        return mmk_ref::update_w((const double*)X, ldx, (const double*)V, (const double*)W,
                                 (double*)W_out, m, n, r, ref_ws(ws, m, n, r),
                                 reinterpret_cast<cudaStream_t>(stream));
    Args a{X, V, W, nullptr, nullptr, ldx, m, n, (int)r, ws, red, nullptr, err_dev,
           reinterpret_cast<cudaStream_t>(stream), 3};
    rc = run_a(dtype, a);
    if (rc) return rc;
    mmk_host::err_flag(err_dev, red + mmk_nnmf_reduce_len(n, r) - 1, a.st);
    return mmk_nnmf_iter_b(dtype, W, W_out, n, r, red, nullptr, err_dev, stream);
}

// grad_V = 2 (V W - X) W^T, grad_W = 2 V^T (V W - X) (reference nnmf_gradient
// nnmf.py:113-119) in the Gram form 2 (V G_W - X W^T), 2 (G_V W - V^T X):
// products accumulated as in the update kernels, differences in fp64
extern "C" int mmk_nnmf_gradient(int dtype, const void* X, int64_t ldx, const void* V,
                                 const void* W, void* GV, void* GW, int64_t m, int64_t n,
                                 int64_t r, void* ws, size_t ws_bytes, double* red,
                                 int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_nnmf_gradient");
    int rc = check(dtype, m, n, r, ldx, ws_bytes, false);
    if (rc) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == MMK_F64)
        return mmk_ref::gradient((const double*)X, ldx, (const double*)V, (const double*)W,
                                 (double*)GV, (double*)GW, m, n, r, ref_ws(ws, m, n, r), st);
    Args a{X, V, W, GV, nullptr, ldx, m, n, (int)r, ws, red, nullptr, err_dev, st, 4};
    rc = run_a(dtype, a);
    if (rc) return rc;
    return dtype == MMK_F32 ? finish_b<float>(W, GW, n, (int)r, red, nullptr, st, true)
                            : finish_b<double>(W, GW, n, (int)r, red, nullptr, st, true);
}
