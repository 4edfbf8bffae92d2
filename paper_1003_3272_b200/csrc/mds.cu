// mds.cu -- stress majorization (reference mds.py:79-144), full-row tiling.
//
// One warp owns RPW points i; its lanes sweep j over the row, so per pair the
// kernel forms d_ij = ||theta_i - theta_j|| directly (no Gram matrix, no n x n
// temporary), the coupling z_ij = w_ij y_ij / d_ij, and accumulates
//     zsum_i = sum_j z_ij,   A_i = sum_j (w_ij - z_ij) theta_j,
//     stress_i = sum_{j > i} w_ij (y_ij - d_ij)^2           (fp64)
// then applies the separated update
//     theta_i' = (theta_i (w_i. + zsum_i) + A_i) / (2 w_i.)      (mds.py:141-144)
// Stress partials are reduced deterministically (per-block partial, last
// block sums in block order).
//
// Roofline: HBM-bound on Y (n*rows*sizeof(T) bytes per call; W adds the same
// when weights are explicit).  The packed-triangle variant for large unit-
// weight problems lives in mds_tri.cu.
#include <memory>

#include "mm_control.cuh"
#include "small_engine.h"

namespace {

using namespace mmk;

constexpr int kWarps = 8;

// SPLIT > 1 (small problems): SPLIT warps share a row, each sweeping every
// SPLIT-th 32-column slice; their sums are combined through shared memory in
// warp order (deterministic) before the update.
template <typename T, int DIM, int RPW, int SPLIT>
__global__ void __launch_bounds__(kWarps * 32)
mds_rows_kernel(const T* __restrict__ Y, const T* __restrict__ Wt, long long ldy,
                const double* __restrict__ wsum, const T* __restrict__ theta,
                T* __restrict__ theta_out, long long ldo, int dim_rt, long long n,
                long long row0, long long rows, int flags, double* __restrict__ partials,
                unsigned int* counter, double* f_dev, int64_t* err) {
    const int dim = DIM > 0 ? DIM : dim_rt;
    constexpr int DM = DIM > 0 ? DIM : 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = warp % SPLIT, rw = warp / SPLIT;
    const long long lbase = ((long long)blockIdx.x * (kWarps / SPLIT) + rw) * RPW;  // local row
    const bool do_update = flags & (MMK_MDS_UPDATE | MMK_MDS_GRADIENT);
    const bool do_grad = flags & MMK_MDS_GRADIENT;
    const bool do_obj = flags & MMK_MDS_OBJECTIVE;

    T ti[RPW][DM];
    T acc[RPW][DM];
    T zs[RPW];
    double st[RPW];
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const long long li = lbase + rr;
        const long long gi = row0 + (li < rows ? li : rows - 1);
#pragma unroll
        for (int k = 0; k < DM; ++k) {
            ti[rr][k] = (k < dim) ? theta[(long long)k * n + gi] : T(0);
            acc[rr][k] = T(0);
        }
        zs[rr] = T(0);
        st[rr] = 0.0;
    }

    for (long long j = lane + 32 * seg; j < n; j += 32 * SPLIT) {
        T tj[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k) tj[k] = (k < dim) ? __ldg(theta + (long long)k * n + j) : T(0);
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            const long long li = lbase + rr;
            if (li >= rows) break;
            const long long gi = row0 + li;
            const T y = Y[li * ldy + j];
            const T w = Wt ? Wt[li * ldy + j] : (gi == j ? T(0) : T(1));
            T d2 = T(0);
#pragma unroll
            for (int k = 0; k < DM; ++k) {
                const T g = ti[rr][k] - tj[k];
                d2 = fma(g, g, d2);
            }
            const T wy = w * y;
            T z = T(0);
            // the update needs d > 0 where w y > 0 (mds.py:127-128), the
            // gradient wherever w > 0 (stress_gradient mds.py:154-156)
            if (d2 <= T(0) && (do_grad ? w > T(0) : (do_update && wy > T(0))))
                flag_error(err, MMK_E_NUMERICS, err_at_update(1, gi * n + j));
            if (wy > T(0) && d2 > T(0)) z = wy / sqrt(d2);
            zs[rr] += z;
            const T c = w - z;
#pragma unroll
            for (int k = 0; k < DM; ++k) acc[rr][k] = fma(c, tj[k], acc[rr][k]);
            if (do_obj && j > gi) {
                const double r = (double)y - sqrt((double)d2);
                st[rr] += (double)w * r * r;
            }
        }
    }

    double blk = 0.0;
    double sst[RPW];
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        zs[rr] = warp_sum(zs[rr]);
#pragma unroll
        for (int k = 0; k < DM; ++k) acc[rr][k] = warp_sum(acc[rr][k]);
        sst[rr] = warp_sum(st[rr]);
    }
    if (SPLIT > 1) {
        __shared__ double sh[kWarps][DM + 2];
        if (lane == 0) {
            sh[warp][0] = (double)zs[0];
            sh[warp][1] = sst[0];
#pragma unroll
            for (int k = 0; k < DM; ++k) sh[warp][2 + k] = (double)acc[0][k];
        }
        __syncthreads();
        if (seg == 0 && lane == 0) {
            double z = sh[warp][0], t = sh[warp][1];
            double a[DM];
#pragma unroll
            for (int k = 0; k < DM; ++k) a[k] = sh[warp][2 + k];
            for (int q = 1; q < SPLIT; ++q) {
                z += sh[warp + q][0];
                t += sh[warp + q][1];
#pragma unroll
                for (int k = 0; k < DM; ++k) a[k] += sh[warp + q][2 + k];
            }
            zs[0] = (T)z;
            sst[0] = t;
#pragma unroll
            for (int k = 0; k < DM; ++k) acc[0][k] = (T)a[k];
        }
    }
#pragma unroll
    for (int rr = 0; rr < RPW; ++rr) {
        const long long li = lbase + rr;
        const double s = sst[rr];
        if (li < rows && seg == 0) {
            blk += s;
            if (do_update && lane == 0) {
                const long long gi = row0 + li;
                const double ws = wsum[gi];
                if (do_grad) {   // 2 (theta_i (w_i. - z_i.) - sum_j (w_ij - z_ij) theta_j)
                    const double row = ws - (double)zs[rr];
#pragma unroll
                    for (int k = 0; k < DM; ++k)
                        if (k < dim)
                            theta_out[(long long)k * ldo + li] =
                                (T)(2.0 * ((double)ti[rr][k] * row - (double)acc[rr][k]));
                    continue;
                }
                const double scale = ws + (double)zs[rr];
                const double inv = 2.0 * ws;
#pragma unroll
                for (int k = 0; k < DM; ++k)
                    if (k < dim)
                        theta_out[(long long)k * ldo + li] =
                            (T)(((double)ti[rr][k] * scale + (double)acc[rr][k]) / inv);
            }
        }
    }
    if (!do_obj) return;
    __shared__ double red[kWarps];
    __shared__ double fin[kWarps];
    if (lane == 0) red[warp] = blk;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < kWarps; ++w) b += red[w];
        partials[blockIdx.x] = b;
    }
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(partials, gridDim.x, fin);
        if (threadIdx.x == 0) *f_dev = tot;
    }
}

constexpr int kMaxDim = 32;

template <typename T, int RPW, int SPLIT = 1>
int launch_rows(const T* Y, const T* Wt, long long ldy, const double* wsum, const T* theta,
                T* out, long long ldo, int dim, long long n, long long row0, long long rows,
                int flags, void* ws, double* f_dev, int64_t* err, cudaStream_t st) {
    const int rows_per_block = kWarps / SPLIT * RPW;
    const int grid = ceil_div(rows, rows_per_block);
    unsigned int* counter = reinterpret_cast<unsigned int*>(ws);
    double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + 256);
#define MMK_MDS_CASE(D)                                                                     \
    case D:                                                                                 \
        MMK_LAUNCH("mds_rows", st,                                                          \
                   (mds_rows_kernel<T, D, RPW, SPLIT><<<grid, kWarps * 32, 0, st>>>(               \
                       Y, Wt, ldy, wsum, theta, out, ldo, dim, n, row0, rows, flags,        \
                       partials, counter, f_dev, err)));                                    \
        break;
    switch (dim) {
        MMK_MDS_CASE(1) MMK_MDS_CASE(2) MMK_MDS_CASE(3) MMK_MDS_CASE(4) MMK_MDS_CASE(5)
        MMK_MDS_CASE(6) MMK_MDS_CASE(7) MMK_MDS_CASE(8) MMK_MDS_CASE(9) MMK_MDS_CASE(10)
        default:
            MMK_LAUNCH("mds_rows", st,
                       (mds_rows_kernel<T, 0, RPW, SPLIT><<<grid, kWarps * 32, 0, st>>>(
                           Y, Wt, ldy, wsum, theta, out, ldo, dim, n, row0, rows, flags,
                           partials, counter, f_dev, err)));
    }
#undef MMK_MDS_CASE
    MMK_CHECK_LAUNCH("mds_rows_kernel");
    return MMK_OK;
}

size_t mds_ws(long long rows) {
    const int grid = ceil_div(rows, 1);   // worst case: SPLIT = kWarps, one row per block
    return 256 + sizeof(double) * (size_t)grid;
}

template <typename T>
__global__ void mds_unpack_kernel(const T* __restrict__ g, T* __restrict__ theta, long long dim,
                                  long long n, long long rows_pad) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= dim * n) return;
    const long long k = t / n, i = t - k * n;
    const long long rank = i / rows_pad, c = i - rank * rows_pad;
    theta[t] = g[(rank * dim + k) * rows_pad + c];
}

// ---------------------------------------------------------------------------
// Persistent small-problem engine (BASELINE config 3: n = 401, dim 2..10):
// whole batches of MM iterations in one cooperative kernel.  CTA c owns rows
// [c n / G, (c + 1) n / G) with their rows of Y (and W) resident in shared
// memory; per iteration
//   stage theta_k (dim x n) in shared memory
//   for each of my rows (the whole CTA sweeps its columns, fixed-order
//   block reduction): zs_i, A_i, the stress partial (j > i), the update
//   (the arithmetic of mds_rows_kernel) -> theta_k+1 in slot s^1
//   barrier
//   every CTA sums the stress partials in the same order and applies the
//   stopping rule itself (mm_step); CTA 0 records the trace.
// One grid barrier per iteration.
constexpr int kMdsSmallThr = 512;

template <typename T>
struct MdsSmall {
    const T *Y, *Wt;
    long long ldy;
    const double* wsum;
    T* theta[2];
    int n, rpc;
    double* part;          // [G] stress partials
    unsigned int* flags;   // [32 G]
    unsigned int epoch0;
    long long* ctl;
    double* trace;
    long long* tstamp;
    int64_t* err;
    mmk_stop_rule rule;
};

template <typename T, int DIM>
__global__ void __launch_bounds__(kMdsSmallThr) mds_small_kernel(MdsSmall<T> a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int n = a.n, rpc = a.rpc;
    T* const th = reinterpret_cast<T*>(sm_raw);     // DIM x n
    T* const ys = th + DIM * n;                     // rpc x n: my rows of Y
    T* const wts = ys + rpc * n;                    // rpc x n: my rows of W (if explicit)
    __shared__ double red[kMdsSmallThr / 32][DIM + 2];
    __shared__ int decision;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x, G = gridDim.x;
    const int r0 = (int)((long long)c * n / G), r1 = (int)((long long)(c + 1) * n / G);
    for (int t = tid; t < (r1 - r0) * n; t += kMdsSmallThr) {
        const int i = t / n, j = t - i * n;
        ys[t] = a.Y[(long long)(r0 + i) * a.ldy + j];
        if (a.Wt) wts[t] = a.Wt[(long long)(r0 + i) * a.ldy + j];
    }
    MmState st = mm_load(a.ctl);
    int iter_local = 0;
    unsigned int epoch = a.epoch0;
    int slot = 0;
    for (;;) {
        {
            const T* tg = a.theta[slot];
            for (int t0 = 0; t0 < DIM * n; t0 += kMdsSmallThr * 8) {
                T v8[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int t = t0 + u * kMdsSmallThr + tid;
                    v8[u] = t < DIM * n ? __ldcg(tg + t) : T(0);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int t = t0 + u * kMdsSmallThr + tid;
                    if (t < DIM * n) th[t] = v8[u];
                }
            }
        }
        __syncthreads();
        double stress = 0.0;
        T* out = a.theta[slot ^ 1];
        for (int i = r0; i < r1; ++i) {
            const T* yr = ys + (i - r0) * n;
            const T* wr = wts + (i - r0) * n;
            T ti[DIM], acc[DIM];
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                ti[k] = th[k * n + i];
                acc[k] = T(0);
            }
            T zs = T(0);
            double sti = 0.0;
            for (int j = tid; j < n; j += kMdsSmallThr) {
                const T y = yr[j];
                const T w = a.Wt ? wr[j] : (i == j ? T(0) : T(1));
                T d2 = T(0);
#pragma unroll
                for (int k = 0; k < DIM; ++k) {
                    const T g = ti[k] - th[k * n + j];
                    d2 = fma(g, g, d2);
                }
                const T wy = w * y;
                T z = T(0);
                if (wy > T(0)) {
                    if (d2 <= T(0))
                        flag_error(a.err, MMK_E_NUMERICS, err_at_update(1, (long long)i * n + j));
                    else
                        z = wy / sqrt(d2);
                }
                zs += z;
                const T cw = w - z;
#pragma unroll
                for (int k = 0; k < DIM; ++k) acc[k] = fma(cw, th[k * n + j], acc[k]);
                if (j > i) {
                    const double rr = (double)y - sqrt((double)d2);
                    sti += (double)w * rr * rr;
                }
            }
            // fixed-order block reduction of (zs, acc, stress)
            double v[DIM + 2];
            v[0] = (double)warp_sum(zs);
#pragma unroll
            for (int k = 0; k < DIM; ++k) v[1 + k] = (double)warp_sum(acc[k]);
            v[DIM + 1] = warp_sum(sti);
            if (lane == 0)
#pragma unroll
                for (int q = 0; q < DIM + 2; ++q) red[warp][q] = v[q];
            __syncthreads();
            if (tid == 0) {
                double z = 0.0, s2 = 0.0, A[DIM];
#pragma unroll
                for (int k = 0; k < DIM; ++k) A[k] = 0.0;
                for (int w = 0; w < kMdsSmallThr / 32; ++w) {
                    z += red[w][0];
                    s2 += red[w][DIM + 1];
#pragma unroll
                    for (int k = 0; k < DIM; ++k) A[k] += red[w][1 + k];
                }
                stress += s2;
                const double ws = a.wsum[i];
                const double scale = ws + (double)(T)z;
                const double inv = 2.0 * ws;
#pragma unroll
                for (int k = 0; k < DIM; ++k)
                    out[(long long)k * n + i] = (T)(((double)ti[k] * scale + (double)(T)A[k]) / inv);
            }
            __syncthreads();
        }
        // stress partials of this launch's iteration k in part[k & 1][.]: a CTA
        // past this barrier may write the next iteration's while a slower one
        // still reads these for the stopping rule (iter_local is uniform over
        // the CTA; st advances in one thread)
        double* const part = a.part + (iter_local & 1) * G;
        if (tid == 0) part[c] = stress;
        grid_sync_flags(a.flags, ++epoch);
        if (warp == 0) {
            double s2 = 0.0;
            for (int b = lane; b < G; b += 32) s2 += __ldcg(part + b);
            s2 = warp_sum(s2);
            if (lane == 0) {
                const MmState before = st;
                int reason = 0;
                const int dcs =
                    mm_step(st, slot, s2, err_class(a.err), a.rule, &reason);
                if (c == 0) mm_record(a.ctl, a.trace, a.tstamp, before, st, slot, s2, dcs, reason);
                decision = dcs;
            }
        }
        __syncthreads();
        const int dcs = decision;
        if (dcs != kMmContinue) return;
        slot ^= 1;
        ++iter_local;
    }
}

template <typename T>
size_t mds_small_smem(long long n, int dim, bool weighted) {
    const long long rpc = (n + kNumSMs - 1) / kNumSMs + 1;
    return sizeof(T) * (size_t)(dim * n + (weighted ? 2 : 1) * rpc * n);
}

template <typename T>
const void* mds_small_kernel_for(int dim) {
    switch (dim) {
#define MMK_MDS_SMALL(D) \
    case D:              \
        return reinterpret_cast<const void*>(&mds_small_kernel<T, D>);
        MMK_MDS_SMALL(1) MMK_MDS_SMALL(2) MMK_MDS_SMALL(3) MMK_MDS_SMALL(4) MMK_MDS_SMALL(5)
        MMK_MDS_SMALL(6) MMK_MDS_SMALL(7) MMK_MDS_SMALL(8) MMK_MDS_SMALL(9) MMK_MDS_SMALL(10)
#undef MMK_MDS_SMALL
        default:
            return nullptr;
    }
}

}  // namespace

extern "C" int mmk_mds_unpack(int dtype, const void* gathered, void* theta, int64_t dim, int64_t n,
                              int64_t rows_pad, void* stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int grid = ceil_div(dim * n, 256);
    if (dtype == MMK_F32)
        mds_unpack_kernel<float><<<grid, 256, 0, st>>>((const float*)gathered, (float*)theta, dim,
                                                       n, rows_pad);
    else
        mds_unpack_kernel<double><<<grid, 256, 0, st>>>((const double*)gathered, (double*)theta,
                                                        dim, n, rows_pad);
    MMK_CHECK_LAUNCH("mds_unpack_kernel");
    return MMK_OK;
}

extern "C" int mmk_mds_ws_bytes(int dtype, int64_t n, int64_t dim, int64_t rows, size_t* out) {
    (void)dtype;
    (void)n;
    (void)dim;
    if (rows < 1) rows = 1;
    *out = mds_ws(rows);
    return MMK_OK;
}

extern "C" int mmk_mds_iter(int dtype, const void* Y, const void* Wt, int64_t ldy,
                            const double* wsum, const void* theta, void* theta_out, int64_t ldo,
                            int64_t dim, int64_t n, int64_t row0, int64_t rows, int flags,
                            void* ws, size_t ws_bytes, double* f_dev, int64_t* err_dev,
                            void* stream) {
    MMK_NVTX("mmk_mds_iter");
    if (dim < 1 || dim > kMaxDim) {
        mmk_host::set_error("embedding dimension %lld outside [1, %d]", (long long)dim, kMaxDim);
        return MMK_E_SHAPE;
    }
    if (n < 1 || rows < 1 || row0 < 0 || row0 + rows > n || ldy < n) {
        mmk_host::set_error("bad MDS row range: n=%lld row0=%lld rows=%lld ldy=%lld",
                            (long long)n, (long long)row0, (long long)rows, (long long)ldy);
        return MMK_E_SHAPE;
    }
    if (ws_bytes < mds_ws(rows)) {
        mmk_host::set_error("MDS workspace too small: %zu < %zu", ws_bytes, mds_ws(rows));
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // small problems: one point per warp (more CTAs); large: 4 points per warp
    // small problems: split every row over 8 (4) warps for parallelism;
    // large: 4 points per warp
    const bool big = rows >= 4096;
    const bool tiny = rows <= 1024;
    if (dtype == MMK_F32) {
        auto f = big ? launch_rows<float, 4> : tiny ? launch_rows<float, 1, 8>
                                                    : launch_rows<float, 1, 4>;
        return f((const float*)Y, (const float*)Wt, ldy, wsum, (const float*)theta,
                 (float*)theta_out, ldo, (int)dim, n, row0, rows, flags, ws, f_dev, err_dev, st);
    }
    if (dtype == MMK_F64) {
        auto f = big ? launch_rows<double, 4> : tiny ? launch_rows<double, 1, 8>
                                                     : launch_rows<double, 1, 4>;
        return f((const double*)Y, (const double*)Wt, ldy, wsum, (const double*)theta,
                 (double*)theta_out, ldo, (int)dim, n, row0, rows, flags, ws, f_dev, err_dev, st);
    }
    mmk_host::set_error("unknown dtype %d", dtype);
    return MMK_E_SHAPE;
}

namespace mmk_small {

bool mds_eligible(int dtype, long long n, long long dim, bool weighted) {
    const char* env = getenv("MMK_SMALL_ENGINE");
    if (env && env[0] == '0') return false;
    if ((dtype != MMK_F32 && dtype != MMK_F64) || dim < 1 || dim > 10 || n < 2 || n > 8192)
        return false;
    const size_t smem = dtype == MMK_F32 ? mds_small_smem<float>(n, (int)dim, weighted)
                                         : mds_small_smem<double>(n, (int)dim, weighted);
    return smem <= 160 * 1024;
}

template <typename T>
static int mds_prepare_t(const void* Y, const void* Wt, long long ldy, const double* wsum,
                         void* thetaA, void* thetaB, long long dim, long long n,
                         const mmk_stop_rule* rule, double* trace, int64_t* tstamp, int64_t* ctl,
                         int64_t* err, Launch* out) {
    MdsSmall<T> a;
    a.Y = (const T*)Y;
    a.Wt = (const T*)Wt;
    a.ldy = ldy;
    a.wsum = wsum;
    a.theta[0] = (T*)thetaA;
    a.theta[1] = (T*)thetaB;
    a.n = (int)n;
    const int G = kNumSMs;
    a.rpc = (int)((n + G - 1) / G) + 1;
    const void* kern = mds_small_kernel_for<T>((int)dim);
    const size_t smem = mds_small_smem<T>(n, (int)dim, Wt != nullptr);
    cudaError_t ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem);
    if (ce != cudaSuccess) return mmk_host::cuda_status(ce, "mds_small smem attribute");
    int per_sm = 0;
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMdsSmallThr, smem);
    if (ce != cudaSuccess || per_sm < 1) {
        mmk_host::set_error("mds_small: kernel does not fit an SM (smem %zu)", smem);
        return MMK_E_SHAPE;
    }
    const size_t fbytes = (sizeof(unsigned int) * 32 * G + 255) / 256 * 256;
    void* scratch = scratch_take(fbytes + 2 * sizeof(double) * G, fbytes);   // part [2][G]
    if (!scratch) return mmk_host::cuda_status(cudaErrorMemoryAllocation, "mds_small scratch");
    a.flags = reinterpret_cast<unsigned int*>(scratch);
    a.part = reinterpret_cast<double*>(reinterpret_cast<char*>(scratch) + fbytes);
    a.epoch0 = 0;
    a.ctl = reinterpret_cast<long long*>(ctl);
    a.trace = trace;
    a.tstamp = reinterpret_cast<long long*>(tstamp);
    a.err = err;
    a.rule = *rule;
    out->scratch = scratch;
    auto seq = std::make_shared<unsigned int>(0);
    out->fn = [a, G, smem, kern, seq](cudaStream_t s) -> int {
        MdsSmall<T> arg = a;
        arg.epoch0 = (++*seq) << 20;
        void* args[] = {&arg};
        const bool pr = mmk_host::prof_on();
        if (pr) mmk_host::prof_start("mds_small", s);
        cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(kMdsSmallThr), args,
                                                    smem, s);
        if (pr) mmk_host::prof_stop(s);
        if (e != cudaSuccess) return mmk_host::cuda_status(e, "mds_small_kernel");
        return MMK_OK;
    };
    return MMK_OK;
}

int mds_prepare(int dtype, const void* Y, const void* Wt, long long ldy, const double* wsum,
                void* thetaA, void* thetaB, long long dim, long long n,
                const mmk_stop_rule* rule, double* trace, int64_t* tstamp, int64_t* ctl,
                int64_t* err, Launch* out) {
    if (rule->batch < 2 || (rule->batch & 1)) {
        mmk_host::set_error("engine batch must be an even number >= 2");
        return MMK_E_SHAPE;
    }
    if (dtype == MMK_F32)
        return mds_prepare_t<float>(Y, Wt, ldy, wsum, thetaA, thetaB, dim, n, rule, trace,
                                    tstamp, ctl, err, out);
    return mds_prepare_t<double>(Y, Wt, ldy, wsum, thetaA, thetaB, dim, n, rule, trace, tstamp,
                                 ctl, err, out);
}

}  // namespace mmk_small
