// nnmf_poisson.cu -- NNMF under the Poisson log fit (reference nnmf.py:178-265),
// the square-root multiplicative MM updates, CUDA cores (FFMA / DFMA).
//
// One MM iteration from (V, W), X m x n, rank r <= 128 (ranks above 16 on nnmf_tile.cu):
//   pois_wsum_kernel    ws_k = sum_j w_kj                         (fp64)
//   pois_vstep_kernel   per row i of X (one warp per row pair, W chunks in smem):
//                         b_ij = v_i . w_j, ratio = x_ij / b_ij (x_ij > 0, else 0),
//                         f   += x_ij ln b_ij - b_ij             (objective at (V, W), fp64)
//                         q_i += ratio_ij w_j
//                         v_i' = v_i sqrt(q_i / (ws + 1e-300))    (nnmf.py:226-229)
//   pois_colsum_kernel  vs_k = sum_i v'_ik                        (fp64, fixed order)
//   pois_wpart_kernel   P = V'^T R', R' = X / (V' W) masked, split over row ranges
//   nnmf_wreduce        partials -> red[P]    (shared with the Frobenius path)
//   pois_wfinish_kernel W' = W sqrt(P / (vs + 1e-300))           (nnmf.py:235-241)
// A zero reconstruction under a positive count raises the reference's
// NumericsError: site 1 for the state's objective / V half (nnmf.py:198-199,
// 180-181), site 2 for the W half, index = first (i * n + j).
//
// Multi-GPU: rows of X / V are sharded; phase A ends with this rank's
// red = [P (r x n) | vs (r) | f-partial]; the caller all-reduces red; phase B
// finishes W' redundantly on every rank.
#include "mmk_common.cuh"
#include "nnmf_tile.h"

namespace {

using namespace mmk;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxPoisRank = 128;

// ws_k = sum_j w_kj: one block per k, fixed-shape tree
template <typename T>
__global__ void __launch_bounds__(256)
pois_wsum_kernel(const T* __restrict__ W, long long n, double* __restrict__ wsum) {
    __shared__ double sc[32];
    const T* row = W + (long long)blockIdx.x * n;
    double s = 0.0;
    for (long long j = threadIdx.x; j < n; j += blockDim.x) s += (double)row[j];
    s = block_sum(s, sc);
    if (threadIdx.x == 0) wsum[blockIdx.x] = s;
}

template <typename T, int RMAX, int RPW>
__global__ void __launch_bounds__(kThreads)
pois_vstep_kernel(const T* __restrict__ X, long long ldx, const T* __restrict__ V,
                  const T* __restrict__ W, const double* __restrict__ wsum,
                  T* __restrict__ Vout, long long m, long long n, int r,
                  double* __restrict__ fpart, unsigned int* counter, double* f_out,
                  int64_t* err) {
    __shared__ T Ws[RMAX][33];
    __shared__ T qs[kWarps][RPW][RMAX];
    __shared__ double sc[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long i0 = ((long long)blockIdx.x * kWarps + warp) * RPW;
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
    double f = 0.0;
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
                if (i >= m) continue;
                const T x = X[i * ldx + j];
                T b = T(0);
#pragma unroll
                for (int k = 0; k < RMAX; ++k)
                    if (k < r) b = fma(v[rr][k], Ws[k][lane], b);
                f -= (double)b;
                if (x > T(0)) {
                    if (b == T(0)) {
                        flag_error(err, MMK_E_NUMERICS, err_at(1, i * n + j));
                        continue;
                    }
                    f = fma((double)x, log((double)b), f);
                    const T ratio = x / b;
#pragma unroll
                    for (int k = 0; k < RMAX; ++k)
                        if (k < r) q[rr][k] = fma(ratio, Ws[k][lane], q[rr][k]);
                }
            }
        }
        __syncthreads();
    }
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
            const double vk = (double)V[i * r + k];
            Vout[i * r + k] = (T)(vk * sqrt((double)qs[warp][rr][k] / (wsum[k] + kDenomGuard)));
        }
    }
    const double bs = block_sum(f, sc);
    if (threadIdx.x == 0) fpart[blockIdx.x] = bs;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(fpart, gridDim.x, sc);
        if (threadIdx.x == 0) *f_out = tot;
    }
}

// vs_k partials: block b sums rows [b * rpb, ...) of V' (m x r) in fp64
template <typename T>
__global__ void __launch_bounds__(256)
pois_colsum_kernel(const T* __restrict__ V, long long m, int r, long long rpb,
                   double* __restrict__ part) {
    __shared__ double sm[256];
    const int k = threadIdx.x % r, g = threadIdx.x / r, ng = 256 / r;
    const long long lo = (long long)blockIdx.x * rpb;
    long long hi = lo + rpb;
    if (hi > m) hi = m;
    double s = 0.0;
    if (g < ng)
        for (long long i = lo + g; i < hi; i += ng) s += (double)V[i * r + k];
    sm[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < r) {
        double t = 0.0;
        for (int gg = 0; gg < ng; ++gg) t += sm[gg * r + threadIdx.x];
        part[(long long)blockIdx.x * r + threadIdx.x] = t;
    }
}

// out[k] = sum_b part[b][k] in block order
__global__ void pois_colsum_reduce_kernel(const double* __restrict__ part, int nparts, int r,
                                          double* __restrict__ out) {
    const int k = threadIdx.x;
    if (k >= r) return;
    double t = 0.0;
    for (int b = 0; b < nparts; ++b) t += part[(long long)b * r + k];
    out[k] = t;
}

// P[k][j] partial over rows [s * rows_per_split, ...): lane = column, warps
// stride rows; b' = v'_i . w_j, ratio' = x / b' (masked), acc_k += v'_ik ratio'
template <typename T, int RMAX>
__global__ void __launch_bounds__(kThreads)
pois_wpart_kernel(const T* __restrict__ X, long long ldx, const T* __restrict__ V,
                  const T* __restrict__ W, long long m, long long n, int r,
                  long long rows_per_split, double* __restrict__ out, int64_t* err) {
    __shared__ T red[kWarps][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long j = (long long)blockIdx.x * 32 + lane;
    const long long lo = (long long)blockIdx.y * rows_per_split;
    const long long hi = min(m, lo + rows_per_split);
    T acc[RMAX], wj[RMAX];
#pragma unroll
    for (int k = 0; k < RMAX; ++k) {
        acc[k] = T(0);
        wj[k] = (k < r && j < n) ? W[(long long)k * n + j] : T(0);
    }
    if (j < n) {
        for (long long i = lo + warp; i < hi; i += kWarps) {
            const T x = X[i * ldx + j];
            if (!(x > T(0))) continue;
            const T* vi = V + i * r;
            T b = T(0);
#pragma unroll
            for (int k = 0; k < RMAX; ++k)
                if (k < r) b = fma(vi[k], wj[k], b);
            if (b == T(0)) {
                flag_error(err, MMK_E_NUMERICS, err_at_update(2, i * n + j));
                continue;
            }
            const T ratio = x / b;
#pragma unroll
            for (int k = 0; k < RMAX; ++k)
                if (k < r) acc[k] = fma(vi[k], ratio, acc[k]);
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

__global__ void pois_wreduce_kernel(const double* __restrict__ part, int S, long long len,
                                    double* __restrict__ red) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= len) return;
    double s = 0.0;
    for (int k = 0; k < S; ++k) s += part[(long long)k * len + t];
    red[t] = s;
}

template <typename T>
__global__ void pois_wfinish_kernel(const T* __restrict__ W, T* __restrict__ Wout, long long n,
                                    int r, const double* __restrict__ red, double* f_dev) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long rn = (long long)r * n;
    if (f_dev && t == 0) *f_dev = red[rn + r];
    if (t >= rn) return;
    const int k = (int)(t / n);
    Wout[t] = (T)((double)W[t] * sqrt(red[t] / (red[rn + k] + kDenomGuard)));
}

// ---------------------------------------------------------------------------
struct Plan {
    int rpw, nvb;             // V step rows per warp, blocks
    int S;                    // W-step row splits
    long long rows_per_split;
    int colblocks;
    int csb;                  // colsum blocks
    long long csr;            // rows per colsum block
};

Plan make_plan(long long m, long long n, int r) {
    Plan P;
    P.rpw = r <= 16 ? 2 : 1;
    const long long mm = m > 0 ? m : 1;
    P.nvb = ceil_div(mm, kWarps * P.rpw);
    P.colblocks = ceil_div(n, 32);
    long long S = ceil_div(4 * kNumSMs, P.colblocks);
    const long long smax = ceil_div(mm, 64);
    if (S > smax) S = smax;
    if (S < 1) S = 1;
    P.rows_per_split = ceil_div(mm, S);
    P.S = ceil_div(mm, P.rows_per_split);
    P.csr = 4096;
    P.csb = ceil_div(mm, P.csr);
    return P;
}

struct PWs {
    unsigned int* counter;
    double *wsum, *fpart, *wpart, *cpart;
};

size_t ws_layout(const Plan& P, long long n, int r, void* base, PWs* L) {
    size_t off = 256;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    const size_t ow = take(sizeof(double) * (size_t)r);
    const size_t of = take(sizeof(double) * (size_t)P.nvb);
    const size_t oc = take(sizeof(double) * (size_t)P.csb * r);
    const size_t op = take(P.S > 1 ? sizeof(double) * (size_t)P.S * r * (size_t)n : 0);
    if (base && L) {
        char* c = reinterpret_cast<char*>(base);
        L->counter = reinterpret_cast<unsigned int*>(c);
        L->wsum = reinterpret_cast<double*>(c + ow);
        L->fpart = reinterpret_cast<double*>(c + of);
        L->cpart = reinterpret_cast<double*>(c + oc);
        L->wpart = reinterpret_cast<double*>(c + op);
    }
    return off;
}

struct Args {
    const void *X, *V, *W;
    void* V_out;
    long long ldx, m, n;
    int r;
    void* ws;
    double* red;
    int64_t* err;
    cudaStream_t st;
};

template <typename T, int RMAX>
int run_a(const Args& a) {
    const Plan P = make_plan(a.m, a.n, a.r);
    PWs L;
    ws_layout(P, a.n, a.r, a.ws, &L);
    const T* X = (const T*)a.X;
    const T* V = (const T*)a.V;
    const T* W = (const T*)a.W;
    T* Vo = (T*)a.V_out;
    const long long rn = (long long)a.r * a.n;
    double* f_out = a.red + rn + a.r;
    cudaStream_t st = a.st;
    if (a.m == 0) {
        cudaMemsetAsync(a.red, 0, sizeof(double) * (size_t)(rn + a.r + 1), st);
        MMK_CHECK_LAUNCH("pois memset");
        return MMK_OK;
    }
    MMK_LAUNCH("pois_wsum", st,
               (pois_wsum_kernel<T><<<a.r, 256, 0, st>>>(W, a.n, L.wsum)));
    const bool tile = RMAX > 16 && mmk_tile::applies(a.r);   // ranks 17..128: nnmf_tile.cu
    int S = P.S;
    if constexpr (RMAX > 64) {   // ranks above 64 always take the tiles
        if (!tile) return MMK_E_SHAPE;
    }
    if (tile) {
        mmk_tile::pois_vstep<T>(X, a.ldx, V, W, L.wsum, Vo, a.m, a.n, a.r, L.fpart, L.counter,
                                f_out, a.err, st);
    } else if constexpr (RMAX <= 64) {
        if (RMAX <= 16 && P.rpw == 2)
            MMK_LAUNCH("pois_vstep", st,
                       (pois_vstep_kernel<T, RMAX, 2><<<P.nvb, kThreads, 0, st>>>(
                           X, a.ldx, V, W, L.wsum, Vo, a.m, a.n, a.r, L.fpart, L.counter, f_out,
                           a.err)));
        else
            MMK_LAUNCH("pois_vstep", st,
                       (pois_vstep_kernel<T, RMAX, 1><<<P.nvb, kThreads, 0, st>>>(
                           X, a.ldx, V, W, L.wsum, Vo, a.m, a.n, a.r, L.fpart, L.counter, f_out,
                           a.err)));
    }
    MMK_CHECK_LAUNCH("pois_vstep");
    MMK_LAUNCH("pois_colsum", st,
               (pois_colsum_kernel<T><<<P.csb, 256, 0, st>>>(Vo, a.m, a.r, P.csr, L.cpart)));
    MMK_LAUNCH("pois_colsum_reduce", st,
               (pois_colsum_reduce_kernel<<<1, 128, 0, st>>>(L.cpart, P.csb, a.r, a.red + rn)));
    if (tile) {
        S = mmk_tile::wpart_splits<T>(a.m, a.n, P.S);
        mmk_tile::pois_wpart<T>(X, a.ldx, Vo, W, a.m, a.n, a.r, S, S > 1 ? L.wpart : a.red,
                                a.err, st);
    } else if constexpr (RMAX <= 64) {
        dim3 grid(P.colblocks, P.S);
        double* dst = P.S > 1 ? L.wpart : a.red;
        MMK_LAUNCH("pois_wpart", st,
                   (pois_wpart_kernel<T, RMAX><<<grid, kThreads, 0, st>>>(
                       X, a.ldx, Vo, W, a.m, a.n, a.r, P.rows_per_split, dst, a.err)));
    }
    if (S > 1)
        MMK_LAUNCH("pois_wreduce", st,
                   (pois_wreduce_kernel<<<ceil_div(rn, 256), 256, 0, st>>>(L.wpart, S, rn,
                                                                          a.red)));
    MMK_CHECK_LAUNCH("pois_wstep");
    return MMK_OK;
}

template <typename T>
int dispatch(const Args& a) {
    if (a.r <= 4) return run_a<T, 4>(a);
    if (a.r <= 8) return run_a<T, 8>(a);
    if (a.r <= 16) return run_a<T, 16>(a);
    if (a.r <= 32) return run_a<T, 32>(a);
    if (a.r <= 64) return run_a<T, 64>(a);
    return run_a<T, 128>(a);
}

int check(int dtype, long long m, long long n, long long r, long long ldx, size_t ws_bytes) {
    if (dtype != MMK_F32 && dtype != MMK_F64) {
        mmk_host::set_error("unknown dtype %d", dtype);
        return MMK_E_SHAPE;
    }
    if (r < 1 || r > kMaxPoisRank || n < 1 || m < 0 || ldx < n) {
        mmk_host::set_error("unsupported Poisson NNMF shape m=%lld n=%lld r=%lld ldx=%lld "
                            "(rank <= %d)", m, n, r, ldx, kMaxPoisRank);
        return MMK_E_SHAPE;
    }
    const size_t need = ws_layout(make_plan(m, n, (int)r), n, (int)r, nullptr, nullptr);
    if (ws_bytes < need) {
        mmk_host::set_error("Poisson NNMF workspace too small: %zu < %zu", ws_bytes, need);
        return MMK_E_SHAPE;
    }
    return MMK_OK;
}

}  // namespace

extern "C" int mmk_nnmf_poisson_ws_bytes(int dtype, int64_t m, int64_t n, int64_t r,
                                         size_t* out) {
    (void)dtype;
    if (r < 1 || r > kMaxPoisRank || n < 1) {
        mmk_host::set_error("unsupported Poisson NNMF shape n=%lld r=%lld", (long long)n,
                            (long long)r);
        return MMK_E_SHAPE;
    }
    *out = ws_layout(make_plan(m, n, (int)r), n, (int)r, nullptr, nullptr);
    return MMK_OK;
}

// [P (r n) | column sums of V' (r) | f | device-error flag]
extern "C" int64_t mmk_nnmf_poisson_reduce_len(int64_t n, int64_t r) { return r * n + r + 2; }

extern "C" int mmk_nnmf_poisson_iter_a(int dtype, const void* X, int64_t ldx, const void* V,
                                       const void* W, void* V_out, int64_t m, int64_t n,
                                       int64_t r, void* ws, size_t ws_bytes, double* red,
                                       int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_nnmf_poisson_iter_a");
    int rc = check(dtype, m, n, r, ldx, ws_bytes);
    if (rc) return rc;
    Args a{X, V, W, V_out, ldx, m, n, (int)r, ws, red, err_dev,
           reinterpret_cast<cudaStream_t>(stream)};
    rc = dtype == MMK_F32 ? dispatch<float>(a) : dispatch<double>(a);
    if (rc) return rc;
    mmk_host::err_flag(err_dev, red + mmk_nnmf_poisson_reduce_len(n, r) - 1, a.st);
    return MMK_OK;
}

extern "C" int mmk_nnmf_poisson_iter_b(int dtype, const void* W, void* W_out, int64_t n,
                                       int64_t r, const double* red, double* f_dev,
                                       int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_nnmf_poisson_iter_b");
    if (r < 1 || r > kMaxPoisRank || n < 1) {
        mmk_host::set_error("bad Poisson NNMF shape n=%lld r=%lld", (long long)n, (long long)r);
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    mmk_host::peer_err(red + mmk_nnmf_poisson_reduce_len(n, r) - 1, err_dev, st);
    const long long rn = r * n;
    if (dtype == MMK_F32)
        MMK_LAUNCH("pois_wfinish", st,
                   (pois_wfinish_kernel<float><<<ceil_div(rn, 256), 256, 0, st>>>(
                       (const float*)W, (float*)W_out, n, (int)r, red, f_dev)));
    else if (dtype == MMK_F64)
        MMK_LAUNCH("pois_wfinish", st,
                   (pois_wfinish_kernel<double><<<ceil_div(rn, 256), 256, 0, st>>>(
                       (const double*)W, (double*)W_out, n, (int)r, red, f_dev)));
    else {
        mmk_host::set_error("unknown dtype %d", dtype);
        return MMK_E_SHAPE;
    }
    MMK_CHECK_LAUNCH("pois_wfinish_kernel");
    return MMK_OK;
}

extern "C" int mmk_nnmf_poisson_iter(int dtype, const void* X, int64_t ldx, const void* V,
                                     const void* W, void* V_out, void* W_out, int64_t m,
                                     int64_t n, int64_t r, void* ws, size_t ws_bytes, double* red,
                                     double* f_dev, int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_nnmf_poisson_iter");
    mmk_host::NoFlag one_gpu;   // no collective between the phases
    int rc = mmk_nnmf_poisson_iter_a(dtype, X, ldx, V, W, V_out, m, n, r, ws, ws_bytes, red,
                                     err_dev, stream);
    if (rc) return rc;
    return mmk_nnmf_poisson_iter_b(dtype, W, W_out, n, r, red, f_dev, err_dev, stream);
}
