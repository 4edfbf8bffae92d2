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
#include "mmk_common.cuh"

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
                flag_error(err, MMK_E_NUMERICS, err_at(1, gi * n + j));
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
