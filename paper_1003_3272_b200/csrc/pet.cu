// pet.cu -- penalized Poisson MM for emission tomography (reference
// pet.py:288-417): forward projection, back-projection and the pixel update
// of one MM iteration (dense E here; CSR / CSC E below).
//
// Phase A1 (pet_fwd_kernel): one warp per ray forms the forward projection
// m_i = E_i . lam (vectorised row loads, fp64 accumulation), the count ratio
// r_i = y_i / m_i and the loglik term y_i ln m_i - m_i (pet.py:288-315).
// Phase A2 (pet_back_kernel): the back-projection b_j = sum_i e_ij r_i with a
// thread per pixel over coalesced rows of E, split over ray ranges; the last
// split block of each column block adds the split partials in order
// (deterministic) into red = [b | loglik].  E is read twice per iteration
// (a single pass would need each CTA's full rows of E staged until their
// ratios exist, then a cross-CTA reduction of per-CTA b partials); at the
// paper shape (33 MB fp32) both reads are L2 hits, and the paper-shape runs
// take the persistent engine below, which is latency-, not bandwidth-bound.
// A multi-GPU caller all-reduces red across ray shards.
//
// Phase B (pet_pixel_kernel): per pixel c_j = lam_j b_j, neighbour sums over
// the CSR lattice (pet.py:204-210), EM floor or positive-root update
// (pet.py:390-417), and the roughness penalty at lam (pet.py:326-338); the
// last CTA assembles f = loglik - mu/2 * penalty.
#include <memory>

#include "mm_control.cuh"
#include "small_engine.h"

namespace {

using namespace mmk;

constexpr int kRays = 8;      // rays (warps) per projection CTA
constexpr int kPixThreads = 256;

// warp-wide dot product of a row of E with lam, fp64 accumulation; four
// independent accumulators per lane (combined in a fixed order) keep four
// vector loads in flight
template <typename T>
__device__ __forceinline__ double row_dot(const T* __restrict__ e, const T* __restrict__ lam,
                                          long long p, int lane) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (sizeof(T) == 4 && (p & 3) == 0 && ((reinterpret_cast<uintptr_t>(e) & 15) == 0)) {
        const float4* e4 = reinterpret_cast<const float4*>(e);
        const float4* l4 = reinterpret_cast<const float4*>(lam);
        const long long nq = p / 4;
        long long q = lane;
        for (; q + 96 < nq; q += 128) {
            const float4 x0 = __ldg(e4 + q), x1 = __ldg(e4 + q + 32), x2 = __ldg(e4 + q + 64),
                         x3 = __ldg(e4 + q + 96);
            const float4 y0 = __ldg(l4 + q), y1 = __ldg(l4 + q + 32), y2 = __ldg(l4 + q + 64),
                         y3 = __ldg(l4 + q + 96);
            a0 = fma((double)x0.x, (double)y0.x, a0);
            a0 = fma((double)x0.y, (double)y0.y, a0);
            a0 = fma((double)x0.z, (double)y0.z, a0);
            a0 = fma((double)x0.w, (double)y0.w, a0);
            a1 = fma((double)x1.x, (double)y1.x, a1);
            a1 = fma((double)x1.y, (double)y1.y, a1);
            a1 = fma((double)x1.z, (double)y1.z, a1);
            a1 = fma((double)x1.w, (double)y1.w, a1);
            a2 = fma((double)x2.x, (double)y2.x, a2);
            a2 = fma((double)x2.y, (double)y2.y, a2);
            a2 = fma((double)x2.z, (double)y2.z, a2);
            a2 = fma((double)x2.w, (double)y2.w, a2);
            a3 = fma((double)x3.x, (double)y3.x, a3);
            a3 = fma((double)x3.y, (double)y3.y, a3);
            a3 = fma((double)x3.z, (double)y3.z, a3);
            a3 = fma((double)x3.w, (double)y3.w, a3);
        }
        for (; q < nq; q += 32) {
            const float4 a = __ldg(e4 + q), b = __ldg(l4 + q);
            a0 = fma((double)a.x, (double)b.x, a0);
            a0 = fma((double)a.y, (double)b.y, a0);
            a0 = fma((double)a.z, (double)b.z, a0);
            a0 = fma((double)a.w, (double)b.w, a0);
        }
    } else if (sizeof(T) == 8 && (p & 1) == 0 && ((reinterpret_cast<uintptr_t>(e) & 15) == 0)) {
        const double2* e2 = reinterpret_cast<const double2*>(e);
        const double2* l2 = reinterpret_cast<const double2*>(lam);
        const long long nq = p / 2;
        long long q = lane;
        for (; q + 32 < nq; q += 64) {
            const double2 x0 = __ldg(e2 + q), x1 = __ldg(e2 + q + 32);
            const double2 y0 = __ldg(l2 + q), y1 = __ldg(l2 + q + 32);
            a0 = fma(x0.x, y0.x, a0);
            a1 = fma(x0.y, y0.y, a1);
            a2 = fma(x1.x, y1.x, a2);
            a3 = fma(x1.y, y1.y, a3);
        }
        for (; q < nq; q += 32) {
            const double2 a = __ldg(e2 + q), b = __ldg(l2 + q);
            a0 = fma(a.x, b.x, a0);
            a1 = fma(a.y, b.y, a1);
        }
    } else {
        for (long long q = lane; q < p; q += 32) a0 = fma((double)e[q], (double)lam[q], a0);
    }
    return warp_sum((a0 + a1) + (a2 + a3));
}

// Phase A1: kWPR warps per ray (latency hiding at small ray counts) --
// m_i = E_i . lam (fp64 accumulation, the warps' partials combined in a
// fixed order), the count ratio r_i and the loglik term; the last block sums
// the per-block loglik partials in block order into red[p].
constexpr int kWPR = 4;
constexpr int kRaysPB = kRays / kWPR;   // rays per block
template <typename T>
__global__ void __launch_bounds__(kRays * 32)
pet_fwd_kernel(const T* __restrict__ E, long long lde, const T* __restrict__ y,
               const T* __restrict__ lam, long long d, long long p, double* __restrict__ ratio,
               double* __restrict__ llpart, unsigned int* counter, double* __restrict__ red,
               int64_t* err) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rl = warp / kWPR, part = warp % kWPR;
    __shared__ double dots[kRays];
    __shared__ double ll[kRaysPB];
    __shared__ double sc[32];
    const long long i = (long long)blockIdx.x * kRaysPB + rl;
    // this warp's slice of the row: kWPR contiguous pieces, 16-byte aligned
    long long seg = (p + kWPR - 1) / kWPR;
    seg = (seg + 3) & ~3LL;
    long long c0 = part * seg, c1 = c0 + seg;
    if (c1 > p) c1 = p;
    double dot = 0.0;
    if (i < d && c0 < c1) dot = row_dot(E + i * lde + c0, lam + c0, c1 - c0, lane);
    if (lane == 0) dots[warp] = dot;
    __syncthreads();
    if (threadIdx.x < kRaysPB) {
        const long long ii = (long long)blockIdx.x * kRaysPB + threadIdx.x;
        double l = 0.0;
        if (ii < d) {
            double m = 0.0;
            for (int q = 0; q < kWPR; ++q) m += dots[threadIdx.x * kWPR + q];
            const double yi = (double)y[ii];
            double r = 0.0;
            l = -m;
            if (yi > 0.0) {
                if (m == 0.0) flag_error(err, MMK_E_NUMERICS, err_at(1, ii));
                r = yi / m;
                l += yi * log(m);
            }
            ratio[ii] = r;
        }
        ll[threadIdx.x] = l;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s2 = 0.0;
        for (int w = 0; w < kRaysPB; ++w) s2 += ll[w];
        llpart[blockIdx.x] = s2;
    }
    if (arrive_last(counter, gridDim.x)) {
        const double t = block_sum_array(llpart, gridDim.x, sc);
        if (threadIdx.x == 0) red[p] = t;
    }
}

// Phase A2: back-projection b_j = sum_i e_ij r_i, split over ray ranges
// (blockIdx.y); thread = pixel, coalesced rows of E.  The last ray-split
// block of a column block sums the split partials in split order into red.
constexpr int kBackCols = 128;
template <typename T>
__global__ void __launch_bounds__(kBackCols)
pet_back_kernel(const T* __restrict__ E, long long lde, long long d, long long p,
                long long rays_per_split, const double* __restrict__ ratio,
                double* __restrict__ bpart, unsigned int* counters, double* __restrict__ red) {
    const long long j = (long long)blockIdx.x * kBackCols + threadIdx.x;
    const long long i0 = (long long)blockIdx.y * rays_per_split;
    long long i1 = i0 + rays_per_split;
    if (i1 > d) i1 = d;
    if (j < p) {
        double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
        long long i = i0;
        for (; i + 3 < i1; i += 4) {
            const double e0 = (double)E[i * lde + j], e1 = (double)E[(i + 1) * lde + j],
                         e2 = (double)E[(i + 2) * lde + j], e3 = (double)E[(i + 3) * lde + j];
            b0 = fma(e0, ratio[i], b0);
            b1 = fma(e1, ratio[i + 1], b1);
            b2 = fma(e2, ratio[i + 2], b2);
            b3 = fma(e3, ratio[i + 3], b3);
        }
        for (; i < i1; ++i) b0 = fma((double)E[i * lde + j], ratio[i], b0);
        bpart[(long long)blockIdx.y * p + j] = (b0 + b1) + (b2 + b3);
    }
    if (arrive_last(counters + blockIdx.x, gridDim.y) && j < p) {
        double t = 0.0;
        for (unsigned int s2 = 0; s2 < gridDim.y; ++s2) t += bpart[(long long)s2 * p + j];
        red[j] = t;
    }
}

// sparse gather-dot over entries t0, t0 + S, ... < t1: sum val[t] * x[idx[t]]
// in that order (one fp64 chain), with the index/value/gather loads of four
// consecutive entries issued before their fmas so four gathers are in flight
template <int S, typename T, typename X>
__device__ __forceinline__ double gather_dot(const int32_t* __restrict__ idx,
                                             const T* __restrict__ val,
                                             const X* __restrict__ x, int t0, int t1) {
    double m = 0.0;
    int t = t0;
    for (; t + 3 * S < t1; t += 4 * S) {
        const int i0 = idx[t], i1 = idx[t + S], i2 = idx[t + 2 * S], i3 = idx[t + 3 * S];
        const T v0 = val[t], v1 = val[t + S], v2 = val[t + 2 * S], v3 = val[t + 3 * S];
        const X x0 = x[i0], x1 = x[i1], x2 = x[i2], x3 = x[i3];
        m = fma((double)v0, (double)x0, m);
        m = fma((double)v1, (double)x1, m);
        m = fma((double)v2, (double)x2, m);
        m = fma((double)v3, (double)x3, m);
    }
    for (; t < t1; t += S) m = fma((double)val[t], (double)x[idx[t]], m);
    return m;
}

constexpr int kSubW = 8;   // lanes per pixel of the sparse back-projection
constexpr int kFusedPix = kPixThreads / kSubW;   // pixels per fused CTA

// pixel j of the MM update given its back-projection bj (pet.py:388-417):
// c_j = lam_j b_j, neighbour sum, EM floor or positive root -> lam_out[j];
// returns this pixel's share of the roughness penalty at lam (each lattice
// pair once, from its lower index; pet.py:326-331)
template <typename T>
__device__ __forceinline__ double pixel_update(const T* __restrict__ lam, T* __restrict__ lam_out,
                                               const int32_t* __restrict__ nptr,
                                               const int32_t* __restrict__ nidx, double mu,
                                               int flags, long long j, double bj, int64_t* err) {
    double pen = 0.0;
    const double lj = (double)lam[j];
    if ((flags & MMK_PET_CHECK_POSITIVE) && !(lj > 0.0)) flag_error(err, MMK_E_DOMAIN, err_at_update(3, j));
    const int k0 = nptr[j], k1 = nptr[j + 1];
    double nbr = 0.0;
    // neighbours in batches of four: indices, then values, then the in-order
    // sums (same order as one at a time)
    for (int t0 = k0; t0 < k1; t0 += 4) {
        int kk[4];
        double lk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) kk[u] = (t0 + u < k1) ? nidx[t0 + u] : -1;
#pragma unroll
        for (int u = 0; u < 4; ++u) lk[u] = (kk[u] >= 0) ? (double)lam[kk[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (kk[u] < 0) break;
            nbr += lk[u];
            if (kk[u] > j) pen += (lj - lk[u]) * (lj - lk[u]);
        }
    }
    if (flags & MMK_PET_UPDATE) {
        const double c = lj * bj;
        double out;
        if (mu == 0.0) {
            out = c;
        } else {
            const double deg = (double)(k1 - k0);
            const double a = -2.0 * mu * deg;
            const double b = mu * (deg * lj + nbr) - 1.0;
            const double disc = b * b - 4.0 * a * c;
            if (disc < 0.0) flag_error(err, MMK_E_NUMERICS, err_at_update(2, j));
            const double sq = sqrt(disc);
            out = (b < 0.0) ? 2.0 * c / (sq - b) : (-b - sq) / ((a < 0.0) ? 2.0 * a : -1.0);
        }
        lam_out[j] = (T)fmax(out, num<T>::floor());
    }
    return pen;
}

// f = loglik - mu/2 * penalty, assembled by the last CTA from the per-CTA
// penalty partials (fixed order).  The loglik is red[p], or -- when the
// forward kernel skipped its own final reduction (llpart != nullptr) -- the
// same fixed-order sum of its nll per-CTA partials, formed here.
__device__ __forceinline__ void pixel_objective(double pen_block, double mu,
                                                const double* __restrict__ red, long long p,
                                                double* __restrict__ penpart,
                                                unsigned int* counter, double* f_dev,
                                                double* sc, const double* llpart = nullptr,
                                                int nll = 0) {
    if (threadIdx.x == 0) penpart[blockIdx.x] = pen_block;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(penpart, gridDim.x, sc);
        double ll = 0.0;
        if (llpart) {
            __syncthreads();   // sc reuse
            ll = block_sum_array(llpart, nll, sc);
        }
        if (threadIdx.x == 0) {
            double f = llpart ? ll : red[p];
            if (mu > 0.0) f -= 0.5 * mu * tot;
            *f_dev = f;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kPixThreads)
pet_pixel_kernel(const T* __restrict__ lam, T* __restrict__ lam_out, long long p,
                 const int32_t* __restrict__ nptr, const int32_t* __restrict__ nidx, double mu,
                 int flags, const double* __restrict__ red, double* __restrict__ penpart,
                 unsigned int* counter, double* f_dev, int64_t* err) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double pen = 0.0;
    if (j < p)
        pen = pixel_update(lam, lam_out, nptr, nidx, mu, flags, j,
                           (flags & MMK_PET_UPDATE) ? red[j] : 0.0, err);
    if (!(flags & MMK_PET_OBJECTIVE)) return;
    __shared__ double sc[32];
    pixel_objective(block_sum(pen, sc), mu, red, p, penpart, counter, f_dev, sc);
}

// single-GPU sparse phase B: a CTA back-projects kFusedPix pixels (kSubW
// lanes per CSC column, the order of pet_sback_kernel, so b_j is bitwise that
// kernel's) into shared memory, then warp 0 applies their pixel updates --
// b never goes through memory
template <typename T>
__global__ void __launch_bounds__(kPixThreads)
pet_sback_pixel_kernel(const int32_t* __restrict__ cptr, const int32_t* __restrict__ cidx,
                       const T* __restrict__ cval, const double* __restrict__ ratio,
                       const T* __restrict__ lam, T* __restrict__ lam_out, long long p,
                       const int32_t* __restrict__ nptr, const int32_t* __restrict__ nidx,
                       double mu, int flags, const double* __restrict__ red,
                       double* __restrict__ penpart, unsigned int* counter, double* f_dev,
                       int64_t* err, const double* __restrict__ llpart, int nll) {
    __shared__ double bsh[kFusedPix];
    __shared__ double sc[32];
    const int q = threadIdx.x % kSubW;
    const int slot = threadIdx.x / kSubW;
    const long long j0 = (long long)blockIdx.x * kFusedPix;
    const long long jj = j0 + slot;
    double b = 0.0;
    if (jj < p && (flags & MMK_PET_UPDATE))
        b = gather_dot<kSubW>(cidx, cval, ratio, cptr[jj] + q, cptr[jj + 1]);
#pragma unroll
    for (int o = kSubW / 2; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if (q == 0) bsh[slot] = b;
    __syncthreads();
    double pen = 0.0;
    if (threadIdx.x < kFusedPix) {
        const long long j = j0 + threadIdx.x;
        if (j < p) pen = pixel_update(lam, lam_out, nptr, nidx, mu, flags, j, bsh[threadIdx.x], err);
    }
    if (!(flags & MMK_PET_OBJECTIVE)) return;
    static_assert(kFusedPix == 32, "one warp of pixel updates");
    if (threadIdx.x < 32) pen = warp_sum(pen);
    pixel_objective(pen, mu, red, p, penpart, counter, f_dev, sc, llpart, nll);
}

// grad_j = b_j - colsum_j - mu (deg_j lam_j - nbr_j)   (pet.py:349-360)
template <typename T>
__global__ void __launch_bounds__(kPixThreads)
pet_grad_kernel(const T* __restrict__ lam, T* __restrict__ grad, long long p,
                const int32_t* __restrict__ nptr, const int32_t* __restrict__ nidx, double mu,
                const double* __restrict__ colsum, const double* __restrict__ red) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p) return;
    double g = red[j] - colsum[j];
    if (mu > 0.0) {
        const int k0 = nptr[j], k1 = nptr[j + 1];
        double nbr = 0.0;
        for (int t = k0; t < k1; ++t) nbr += (double)lam[nidx[t]];
        g -= mu * ((double)(k1 - k0) * (double)lam[j] - nbr);
    }
    grad[j] = (T)g;
}

struct PetWs {
    unsigned int* counter;    // [0] pixel kernel, [1] forward kernel
    unsigned int* bcounters;  // one per back-projection column block
    double* ratio;
    double* bpart;
    double* llpart;
    double* penpart;
    int nfwd, ncb, splits;
    long long rays_per_split;
};

void back_plan(long long d, long long p, int* ncb, int* splits, long long* rps) {
    *ncb = ceil_div(p, kBackCols);
    long long s = ceil_div(16 * kNumSMs, *ncb);
    const long long smax = d > 32 ? d / 32 : 1;
    if (s > smax) s = smax;
    if (s < 1) s = 1;
    *rps = ceil_div(d > 0 ? d : 1, s);
    *splits = ceil_div(d > 0 ? d : 1, *rps);
}

size_t pet_ws_layout(long long d, long long p, void* base, PetWs* L) {
    const int nfwd = ceil_div(d > 0 ? d : 1, kRaysPB);
    const int npix = ceil_div(p, kFusedPix);   // penalty partials (>= pixel CTAs)
    int ncb, splits;
    long long rps;
    back_plan(d, p, &ncb, &splits, &rps);
    size_t off = 256;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    // counters + penalty partials first so phase B finds them at offsets that
    // do not depend on the ray count
    size_t o_pen = take(sizeof(double) * (size_t)npix);
    size_t o_bc = take(sizeof(unsigned int) * (size_t)ncb);
    size_t o_ll = take(sizeof(double) * (size_t)nfwd);
    size_t o_r = take(sizeof(double) * (size_t)(d > 0 ? d : 1));
    size_t o_b = take(sizeof(double) * (size_t)splits * (size_t)p);
    if (L && base) {
        char* c = reinterpret_cast<char*>(base);
        L->counter = reinterpret_cast<unsigned int*>(c);
        L->bcounters = reinterpret_cast<unsigned int*>(c + o_bc);
        L->ratio = reinterpret_cast<double*>(c + o_r);
        L->bpart = reinterpret_cast<double*>(c + o_b);
        L->llpart = reinterpret_cast<double*>(c + o_ll);
        L->penpart = reinterpret_cast<double*>(c + o_pen);
        L->nfwd = nfwd;
        L->ncb = ncb;
        L->splits = splits;
        L->rays_per_split = rps;
    }
    return off;
}

template <typename T>
int pet_a(const T* E, long long lde, const T* y, const T* lam, long long d, long long p,
          const PetWs& L, double* red, int64_t* err, cudaStream_t st) {
    if (d > 0) {
        MMK_LAUNCH("pet_fwd", st,
                   (pet_fwd_kernel<T><<<L.nfwd, kRays * 32, 0, st>>>(
                       E, lde, y, lam, d, p, L.ratio, L.llpart, L.counter + 1, red, err)));
        MMK_CHECK_LAUNCH("pet_fwd_kernel");
        MMK_LAUNCH("pet_back", st,
                   (pet_back_kernel<T><<<dim3(L.ncb, L.splits), kBackCols, 0, st>>>(
                       E, lde, d, p, L.rays_per_split, L.ratio, L.bpart, L.bcounters, red)));
        MMK_CHECK_LAUNCH("pet_back_kernel");
    } else {
        cudaMemsetAsync(red, 0, sizeof(double) * (size_t)(p + 1), st);
        MMK_CHECK_LAUNCH("pet_a memset");
    }
    return MMK_OK;
}

template <typename T>
int pet_b(const T* lam, T* lam_out, long long p, const int32_t* nptr, const int32_t* nidx,
          double mu, int flags, const double* red, const PetWs& L, double* f_dev, int64_t* err,
          cudaStream_t st) {
    MMK_LAUNCH("pet_pixel", st,
               (pet_pixel_kernel<T><<<ceil_div(p, kPixThreads), kPixThreads, 0, st>>>(
                   lam, lam_out, p, nptr, nidx, mu, flags, red, L.penpart, L.counter, f_dev,
                   err)));
    MMK_CHECK_LAUNCH("pet_pixel_kernel");
    return MMK_OK;
}

int check_ws(long long d, long long p, void* ws, size_t ws_bytes, PetWs* L) {
    const size_t need = pet_ws_layout(d, p, nullptr, nullptr);
    if (ws_bytes < need) {
        mmk_host::set_error("PET workspace too small: %zu < %zu", ws_bytes, need);
        return MMK_E_SHAPE;
    }
    pet_ws_layout(d, p, ws, L);
    return MMK_OK;
}

// ---------------------------------------------------------------------------
// Sparse system matrix (the Siddon matrix of build_system_matrix is ~1 %
// nonzero, pet.py:69-132): E by rays as CSR (forward projection) and by
// pixels as CSC (back-projection), int32 indices.  The back-projection then
// writes red[j] directly -- no partials, deterministic by construction.

// warp per ray: m_i over the CSR row, ratio, loglik; last block -> red[p]
// TAIL: the last CTA sums the loglik partials into red[p]; without it the
// partials stay in llpart for the fused phase-B kernel
template <typename T, bool TAIL = true>
__global__ void __launch_bounds__(kRays * 32)
pet_sfwd_kernel(const int32_t* __restrict__ rptr, const int32_t* __restrict__ ridx,
                const T* __restrict__ rval, const T* __restrict__ y, const T* __restrict__ lam,
                long long d, long long p, double* __restrict__ ratio, double* __restrict__ llpart,
                unsigned int* counter, double* __restrict__ red, int64_t* err) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double ll[kRays];
    __shared__ double sc[32];
    const long long i = (long long)blockIdx.x * kRays + warp;
    double l = 0.0;
    if (i < d) {
        double m = gather_dot<32>(ridx, rval, lam, rptr[i] + lane, rptr[i + 1]);
        m = warp_sum(m);
        if (lane == 0) {
            const double yi = (double)y[i];
            double r = 0.0;
            l = -m;
            if (yi > 0.0) {
                if (m == 0.0) flag_error(err, MMK_E_NUMERICS, err_at(1, i));
                r = yi / m;
                l += yi * log(m);
            }
            ratio[i] = r;
        }
    }
    if (lane == 0) ll[warp] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s2 = 0.0;
        for (int w = 0; w < kRays; ++w) s2 += ll[w];
        llpart[blockIdx.x] = s2;
    }
    if (!TAIL) return;
    if (arrive_last(counter, gridDim.x)) {
        const double t = block_sum_array(llpart, gridDim.x, sc);
        if (threadIdx.x == 0) red[p] = t;
    }
}

// kSubW lanes per pixel: b_j over the CSC column (lane q takes entries
// q, q + kSubW, ...), combined by a fixed xor-shuffle tree -> red[j]
template <typename T>
__global__ void __launch_bounds__(256)
pet_sback_kernel(const int32_t* __restrict__ cptr, const int32_t* __restrict__ cidx,
                 const T* __restrict__ cval, long long p, const double* __restrict__ ratio,
                 double* __restrict__ red) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long j = g / kSubW;
    const int q = (int)(g % kSubW);
    double b = 0.0;
    if (j < p) b = gather_dot<kSubW>(cidx, cval, ratio, cptr[j] + q, cptr[j + 1]);
#pragma unroll
    for (int o = kSubW / 2; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if (j < p && q == 0) red[j] = b;
}

struct SparseWs {
    unsigned int* counter;   // [0] pixel kernel, [1] forward kernel
    double* llpart;
    double* ratio;
    int nfwd;
};

// phase B (shared with the dense path) finds the counter and the penalty
// partials at the same offsets as pet_ws_layout
size_t sparse_ws_layout(long long d, long long p, void* base, SparseWs* L) {
    const int nfwd = ceil_div(d > 0 ? d : 1, kRays);
    const int npix = ceil_div(p, kFusedPix);
    size_t off = 256;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    take(sizeof(double) * (size_t)npix);   // penalty partials (phase B)
    size_t o_ll = take(sizeof(double) * (size_t)nfwd);
    size_t o_r = take(sizeof(double) * (size_t)(d > 0 ? d : 1));
    if (L && base) {
        char* c = reinterpret_cast<char*>(base);
        L->counter = reinterpret_cast<unsigned int*>(c);
        L->llpart = reinterpret_cast<double*>(c + o_ll);
        L->ratio = reinterpret_cast<double*>(c + o_r);
        L->nfwd = nfwd;
    }
    return off;
}

template <typename T>
int pet_sparse_a(const int32_t* rptr, const int32_t* ridx, const T* rval, const int32_t* cptr,
                 const int32_t* cidx, const T* cval, const T* y, const T* lam, long long d,
                 long long p, const SparseWs& L, double* red, int64_t* err, cudaStream_t st) {
    if (d > 0) {
        MMK_LAUNCH("pet_sfwd", st,
                   (pet_sfwd_kernel<T><<<L.nfwd, kRays * 32, 0, st>>>(
                       rptr, ridx, rval, y, lam, d, p, L.ratio, L.llpart, L.counter + 1, red,
                       err)));
        MMK_CHECK_LAUNCH("pet_sfwd_kernel");
        MMK_LAUNCH("pet_sback", st,
                   (pet_sback_kernel<T><<<ceil_div(p * kSubW, 256), 256, 0, st>>>(
                       cptr, cidx, cval, p, L.ratio, red)));
        MMK_CHECK_LAUNCH("pet_sback_kernel");
    } else {
        cudaMemsetAsync(red, 0, sizeof(double) * (size_t)(p + 1), st);
        MMK_CHECK_LAUNCH("pet_sparse_a memset");
    }
    return MMK_OK;
}

// ---------------------------------------------------------------------------
// Persistent small-problem engine for the sparse projector (BASELINE config 2:
// 2016 rays x 4096 pixels, 84,512 nonzeros): whole batches of MM iterations
// in one cooperative kernel.  Per iteration, state lam_k in slot s:
//   stage lam_k in shared memory (every CTA)
//   phase 1  my rays (warp per ray): m_i, ratio_i, loglik partial  -> global
//   barrier
//   stage the ratios in shared memory
//   phase 2  my pixels (8 lanes per CSC column): b_j, the pixel update
//            (pixel_update, the same code as the graph path) -> lam_k+1 in
//            slot s^1; penalty partial at lam_k
//   barrier
//   every CTA sums the loglik / penalty partials in the same fixed order,
//   forms f_k and evaluates the stopping rule (mm_step) itself -- no third
//   barrier; CTA 0 records the trace and ctl.
// The projections gather from shared memory, in the order of pet_sfwd /
// pet_sback, so lam is bitwise the graph path's; f differs from it only in
// the grouping of the partial sums.
constexpr int kPetSmallThr = 512;

template <typename T>
struct PetSmall {
    const int32_t *rptr, *ridx, *cptr, *cidx, *nptr, *nidx;
    const T *rval, *cval, *y;
    T* lam[2];
    int d, p;
    double mu;
    double* ratio;          // [d]
    double* part;           // [2][G]: loglik, penalty partials
    unsigned int* flags;    // [32 G] barrier slots
    unsigned int epoch0;
    long long* ctl;
    double* trace;
    long long* tstamp;
    int64_t* err;
    mmk_stop_rule rule;
    long long* dbg;         // optional: CTA 0 phase stamps (MMK_SMALL_TRACE)
};

template <typename T>
__global__ void __launch_bounds__(kPetSmallThr) pet_small_kernel(PetSmall<T> a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    double* const rs = reinterpret_cast<double*>(sm_raw);   // d ratios
    T* const ls = reinterpret_cast<T*>(rs + a.d);           // p intensities
    __shared__ double wsum[kPetSmallThr / 32];
    __shared__ int decision;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x, G = gridDim.x;
    const int i0 = (int)((long long)c * a.d / G), i1 = (int)((long long)(c + 1) * a.d / G);
    const int j0 = (int)((long long)c * a.p / G), j1 = (int)((long long)(c + 1) * a.p / G);
    MmState st = mm_load(a.ctl);
    unsigned int epoch = a.epoch0;
    int slot = 0;
    int iter_local = 0;
    auto stamp = [&](int ph) {
        if (a.dbg && c == 0 && tid == 0 && iter_local < 64) a.dbg[iter_local * 12 + ph] = clock64();
    };
    for (;;) {
        stamp(0);
        // ---- lam_k into shared memory ------------------------------------------
        {
            const T* lg = a.lam[slot];
            for (int t0 = 0; t0 < a.p; t0 += kPetSmallThr * 8) {
                T v8[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int t = t0 + u * kPetSmallThr + tid;
                    v8[u] = t < a.p ? __ldcg(lg + t) : T(0);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int t = t0 + u * kPetSmallThr + tid;
                    if (t < a.p) ls[t] = v8[u];
                }
            }
        }
        __syncthreads();
        stamp(1);
        // ---- phase 1: rays ------------------------------------------------------
        double ll = 0.0;
        for (int i = i0 + warp; i < i1; i += kPetSmallThr / 32) {
            double m = gather_dot<32>(a.ridx, a.rval, ls, a.rptr[i] + lane, a.rptr[i + 1]);
            m = warp_sum(m);
            if (lane == 0) {
                const double yi = (double)a.y[i];
                double r = 0.0;
                ll -= m;
                if (yi > 0.0) {
                    if (m == 0.0) flag_error(a.err, MMK_E_NUMERICS, err_at(1, i));
                    r = yi / m;
                    ll += yi * log(m);
                }
                a.ratio[i] = r;
            }
        }
        if (lane == 0) wsum[warp] = ll;
        __syncthreads();
        // partials of this launch's iteration k live in part[k & 1][.]: a CTA
        // that has passed the last barrier of an iteration may already write
        // the next one's while a slower CTA still reads these for the stopping
        // rule (iter_local is uniform over the CTA; st advances in one thread)
        double* const part = a.part + (iter_local & 1) * 2 * G;
        if (tid == 0) {
            double s2 = 0.0;
            for (int w = 0; w < kPetSmallThr / 32; ++w) s2 += wsum[w];
            part[c] = s2;
        }
        stamp(2);
        grid_sync_flags(a.flags, ++epoch);
        stamp(3);
        // ---- ratios into shared memory ------------------------------------------
        for (int t0 = 0; t0 < a.d; t0 += kPetSmallThr * 8) {
            double v8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * kPetSmallThr + tid;
                v8[u] = t < a.d ? __ldcg(a.ratio + t) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * kPetSmallThr + tid;
                if (t < a.d) rs[t] = v8[u];
            }
        }
        __syncthreads();
        stamp(4);
        // ---- phase 2: pixels ----------------------------------------------------
        double pen = 0.0;
        {
            const int g = tid / kSubW, q = tid % kSubW;
            T* lo = a.lam[slot ^ 1];
            for (int base = j0; base < j1; base += kPetSmallThr / kSubW) {
                const int j = base + g;
                double b = 0.0;
                if (j < j1) b = gather_dot<kSubW>(a.cidx, a.cval, rs, a.cptr[j] + q, a.cptr[j + 1]);
#pragma unroll
                for (int o = kSubW / 2; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
                if (q == 0 && j < j1)
                    pen += pixel_update(ls, lo, a.nptr, a.nidx, a.mu,
                                        MMK_PET_UPDATE | MMK_PET_OBJECTIVE, j, b, a.err);
            }
        }
        pen = warp_sum(pen);
        if (lane == 0) wsum[warp] = pen;
        __syncthreads();
        if (tid == 0) {
            double s2 = 0.0;
            for (int w = 0; w < kPetSmallThr / 32; ++w) s2 += wsum[w];
            part[G + c] = s2;
        }
        stamp(5);
        grid_sync_flags(a.flags, ++epoch);
        stamp(6);
        // ---- f_k and the stopping rule, redundantly in every CTA -----------------
        if (warp == 0) {
            double l2 = 0.0, p2 = 0.0;
            for (int b = lane; b < G; b += 32) {
                l2 += __ldcg(part + b);
                p2 += __ldcg(part + G + b);
            }
            l2 = warp_sum(l2);
            p2 = warp_sum(p2);
            if (lane == 0) {
                double f = l2;
                if (a.mu > 0.0) f -= 0.5 * a.mu * p2;
                const MmState before = st;
                int reason = 0;
                const int dcs = mm_step(st, slot, f, err_class(a.err), a.rule, &reason);
                if (c == 0) mm_record(a.ctl, a.trace, a.tstamp, before, st, slot, f, dcs, reason);
                decision = dcs;
            }
        }
        __syncthreads();
        stamp(7);
        ++iter_local;
        const int dcs = decision;
        if (dcs != kMmContinue) return;
        slot ^= 1;
    }
}

template <typename T>
size_t pet_small_smem(long long d, long long p) {
    return sizeof(double) * (size_t)d + sizeof(T) * (size_t)p;
}

}  // namespace

extern "C" int mmk_pet_ws_bytes(int dtype, int64_t d, int64_t p, size_t* out) {
    (void)dtype;
    *out = pet_ws_layout(d, p, nullptr, nullptr);
    return MMK_OK;
}

// [b (p) | loglik | device-error flag]
extern "C" int64_t mmk_pet_reduce_len(int64_t p) { return p + 2; }

extern "C" int mmk_pet_iter_a(int dtype, const void* E, int64_t lde, const void* y,
                              const void* lam, int64_t d, int64_t p, void* ws, size_t ws_bytes,
                              double* red, int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_pet_iter_a");
    if (p < 1 || d < 0 || (d > 0 && lde < p)) {
        mmk_host::set_error("bad PET shape d=%lld p=%lld lde=%lld", (long long)d, (long long)p,
                            (long long)lde);
        return MMK_E_SHAPE;
    }
    PetWs L;
    int rc = check_ws(d, p, ws, ws_bytes, &L);
    if (rc) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == MMK_F32)
        rc = pet_a<float>((const float*)E, lde, (const float*)y, (const float*)lam, d, p, L, red,
                          err_dev, st);
    else if (dtype == MMK_F64)
        rc = pet_a<double>((const double*)E, lde, (const double*)y, (const double*)lam, d, p, L,
                           red, err_dev, st);
    else {
        mmk_host::set_error("unknown dtype %d", dtype);
        return MMK_E_SHAPE;
    }
    if (rc) return rc;
    mmk_host::err_flag(err_dev, red + mmk_pet_reduce_len(p) - 1, st);
    return MMK_OK;
}

extern "C" int mmk_pet_iter_b(int dtype, const void* lam, void* lam_out, int64_t p,
                              const int32_t* nbr_ptr, const int32_t* nbr_idx, double mu, int flags,
                              const double* red, void* ws, size_t ws_bytes, double* f_dev,
                              int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_pet_iter_b");
    if (p < 1) {
        mmk_host::set_error("bad PET pixel count %lld", (long long)p);
        return MMK_E_SHAPE;
    }
    PetWs L;
    int rc = check_ws(0, p, ws, ws_bytes, &L);
    if (rc) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    mmk_host::peer_err(red + mmk_pet_reduce_len(p) - 1, err_dev, st);
    if (dtype == MMK_F32)
        return pet_b<float>((const float*)lam, (float*)lam_out, p, nbr_ptr, nbr_idx, mu, flags, red,
                            L, f_dev, err_dev, st);
    if (dtype == MMK_F64)
        return pet_b<double>((const double*)lam, (double*)lam_out, p, nbr_ptr, nbr_idx, mu, flags,
                             red, L, f_dev, err_dev, st);
    mmk_host::set_error("unknown dtype %d", dtype);
    return MMK_E_SHAPE;
}

extern "C" int mmk_pet_iter(int dtype, const void* E, int64_t lde, const void* y, const void* lam,
                            void* lam_out, int64_t d, int64_t p, const int32_t* nbr_ptr,
                            const int32_t* nbr_idx, double mu, int flags, void* ws,
                            size_t ws_bytes, double* red, double* f_dev, int64_t* err_dev,
                            void* stream) {
    MMK_NVTX("mmk_pet_iter");
    mmk_host::NoFlag one_gpu;   // no collective between the phases
    int rc = mmk_pet_iter_a(dtype, E, lde, y, lam, d, p, ws, ws_bytes, red, err_dev, stream);
    if (rc) return rc;
    return mmk_pet_iter_b(dtype, lam, lam_out, p, nbr_ptr, nbr_idx, mu, flags, red, ws, ws_bytes,
                          f_dev, err_dev, stream);
}

extern "C" int mmk_pet_sparse_ws_bytes(int dtype, int64_t d, int64_t p, size_t* out) {
    (void)dtype;
    const size_t a = sparse_ws_layout(d, p, nullptr, nullptr);
    const size_t b = pet_ws_layout(0, p, nullptr, nullptr);   // phase B needs
    *out = a > b ? a : b;
    return MMK_OK;
}

extern "C" int mmk_pet_sparse_iter_a(int dtype, const int32_t* rptr, const int32_t* ridx,
                                     const void* rval, const int32_t* cptr, const int32_t* cidx,
                                     const void* cval, const void* y, const void* lam, int64_t d,
                                     int64_t p, void* ws, size_t ws_bytes, double* red,
                                     int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_pet_sparse_iter_a");
    if (p < 1 || d < 0) {
        mmk_host::set_error("bad sparse PET shape d=%lld p=%lld", (long long)d, (long long)p);
        return MMK_E_SHAPE;
    }
    const size_t need = sparse_ws_layout(d, p, nullptr, nullptr);
    if (ws_bytes < need) {
        mmk_host::set_error("sparse PET workspace too small: %zu < %zu", ws_bytes, need);
        return MMK_E_SHAPE;
    }
    SparseWs L;
    sparse_ws_layout(d, p, ws, &L);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int rc;
    if (dtype == MMK_F32)
        rc = pet_sparse_a<float>(rptr, ridx, (const float*)rval, cptr, cidx, (const float*)cval,
                                 (const float*)y, (const float*)lam, d, p, L, red, err_dev, st);
    else if (dtype == MMK_F64)
        rc = pet_sparse_a<double>(rptr, ridx, (const double*)rval, cptr, cidx,
                                  (const double*)cval, (const double*)y, (const double*)lam, d, p,
                                  L, red, err_dev, st);
    else {
        mmk_host::set_error("unknown dtype %d", dtype);
        return MMK_E_SHAPE;
    }
    if (rc) return rc;
    mmk_host::err_flag(err_dev, red + mmk_pet_reduce_len(p) - 1, st);
    return MMK_OK;
}

// single-GPU sparse iteration: the forward projection, then ONE kernel that
// back-projects each pixel's CSC column and applies the pixel update (the
// per-pixel b_j never goes through memory; results bitwise equal to
// iter_a + iter_b, which a sharded caller uses to all-reduce b in between)
extern "C" int mmk_pet_sparse_iter(int dtype, const int32_t* rptr, const int32_t* ridx,
                                   const void* rval, const int32_t* cptr, const int32_t* cidx,
                                   const void* cval, const void* y, const void* lam,
                                   void* lam_out, int64_t d, int64_t p, const int32_t* nbr_ptr,
                                   const int32_t* nbr_idx, double mu, int flags, void* ws,
                                   size_t ws_bytes, double* red, double* f_dev, int64_t* err_dev,
                                   void* stream) {
    MMK_NVTX("mmk_pet_sparse_iter");
    if (d == 0 || (dtype != MMK_F32 && dtype != MMK_F64)) {
        mmk_host::NoFlag one_gpu;
        int rc = mmk_pet_sparse_iter_a(dtype, rptr, ridx, rval, cptr, cidx, cval, y, lam, d, p,
                                       ws, ws_bytes, red, err_dev, stream);
        if (rc) return rc;
        return mmk_pet_iter_b(dtype, lam, lam_out, p, nbr_ptr, nbr_idx, mu, flags, red, ws,
                              ws_bytes, f_dev, err_dev, stream);
    }
    if (p < 1 || d < 0) {
        mmk_host::set_error("bad sparse PET shape d=%lld p=%lld", (long long)d, (long long)p);
        return MMK_E_SHAPE;
    }
    size_t need = 0;
    mmk_pet_sparse_ws_bytes(dtype, d, p, &need);
    if (ws_bytes < need) {
        mmk_host::set_error("sparse PET workspace too small: %zu < %zu", ws_bytes, need);
        return MMK_E_SHAPE;
    }
    SparseWs L;
    sparse_ws_layout(d, p, ws, &L);
    PetWs Lb;
    pet_ws_layout(0, p, ws, &Lb);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    auto run = [&](auto tag) -> int {
        using T = decltype(tag);
        MMK_LAUNCH("pet_sfwd", st,
                   (pet_sfwd_kernel<T, false><<<L.nfwd, kRays * 32, 0, st>>>(
                       rptr, ridx, (const T*)rval, (const T*)y, (const T*)lam, d, p, L.ratio,
                       L.llpart, L.counter + 1, red, err_dev)));
        MMK_CHECK_LAUNCH("pet_sfwd_kernel");
        MMK_LAUNCH("pet_sback_pixel", st,
                   (pet_sback_pixel_kernel<T><<<ceil_div(p, kFusedPix), kPixThreads, 0, st>>>(
                       cptr, cidx, (const T*)cval, L.ratio, (const T*)lam, (T*)lam_out, p,
                       nbr_ptr, nbr_idx, mu, flags, red, Lb.penpart, Lb.counter, f_dev,
                       err_dev, L.llpart, L.nfwd)));
        MMK_CHECK_LAUNCH("pet_sback_pixel");
        return MMK_OK;
    };
    return dtype == MMK_F32 ? run(float{}) : run(double{});
}

extern "C" int mmk_pet_gradient(int dtype, const void* lam, void* grad, int64_t p,
                                const int32_t* nbr_ptr, const int32_t* nbr_idx, double mu,
                                const double* colsum, const double* red, void* stream) {
    MMK_NVTX("mmk_pet_gradient");
    if (p < 1 || (dtype != MMK_F32 && dtype != MMK_F64)) {
        mmk_host::set_error("bad PET gradient call: dtype %d p=%lld", dtype, (long long)p);
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == MMK_F32)
        MMK_LAUNCH("pet_grad", st,
                   (pet_grad_kernel<float><<<ceil_div(p, kPixThreads), kPixThreads, 0, st>>>(
                       (const float*)lam, (float*)grad, p, nbr_ptr, nbr_idx, mu, colsum, red)));
    else
        MMK_LAUNCH("pet_grad", st,
                   (pet_grad_kernel<double><<<ceil_div(p, kPixThreads), kPixThreads, 0, st>>>(
                       (const double*)lam, (double*)grad, p, nbr_ptr, nbr_idx, mu, colsum, red)));
    MMK_CHECK_LAUNCH("pet_grad_kernel");
    return MMK_OK;
}

namespace mmk_small {

bool pet_eligible(int dtype, long long d, long long p) {
    const char* env = getenv("MMK_SMALL_ENGINE");
    if (env && env[0] == '0') return false;
    if ((dtype != MMK_F32 && dtype != MMK_F64) || d < 1 || p < 1) return false;
    const size_t smem = dtype == MMK_F32 ? pet_small_smem<float>(d, p) : pet_small_smem<double>(d, p);
    return smem <= 160 * 1024 && d * 1.0 * p <= (double)(1LL << 26);
}

template <typename T>
static int pet_prepare_t(const int32_t* rptr, const int32_t* ridx, const void* rval,
                         const int32_t* cptr, const int32_t* cidx, const void* cval,
                         const void* y, void* lamA, void* lamB, long long d, long long p,
                         const int32_t* nbr_ptr, const int32_t* nbr_idx, double mu,
                         const mmk_stop_rule* rule, double* trace, int64_t* tstamp, int64_t* ctl,
                         int64_t* err, Launch* out) {
    PetSmall<T> a;
    a.rptr = rptr;
    a.ridx = ridx;
    a.cptr = cptr;
    a.cidx = cidx;
    a.nptr = nbr_ptr;
    a.nidx = nbr_idx;
    a.rval = (const T*)rval;
    a.cval = (const T*)cval;
    a.y = (const T*)y;
    a.lam[0] = (T*)lamA;
    a.lam[1] = (T*)lamB;
    a.d = (int)d;
    a.p = (int)p;
    a.mu = mu;
    const int G = kNumSMs;
    const size_t smem = pet_small_smem<T>(d, p);
    cudaError_t ce = cudaFuncSetAttribute(pet_small_kernel<T>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ce != cudaSuccess) return mmk_host::cuda_status(ce, "pet_small smem attribute");
    int per_sm = 0;
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pet_small_kernel<T>,
                                                       kPetSmallThr, smem);
    if (ce != cudaSuccess || per_sm < 1) {
        mmk_host::set_error("pet_small: kernel does not fit an SM (smem %zu)", smem);
        return MMK_E_SHAPE;
    }
    const size_t fbytes = (sizeof(unsigned int) * 32 * G + 255) / 256 * 256;
    const size_t bytes = fbytes + sizeof(double) * ((size_t)d + 4 * (size_t)G);   // part [2][2][G]
    void* scratch = scratch_take(bytes, fbytes);
    if (!scratch) return mmk_host::cuda_status(cudaErrorMemoryAllocation, "pet_small scratch");
    a.flags = reinterpret_cast<unsigned int*>(scratch);
    a.ratio = reinterpret_cast<double*>(reinterpret_cast<char*>(scratch) + fbytes);
    a.part = a.ratio + d;
    a.epoch0 = 0;
    a.ctl = reinterpret_cast<long long*>(ctl);
    a.trace = trace;
    a.tstamp = reinterpret_cast<long long*>(tstamp);
    a.err = err;
    a.rule = *rule;
    a.dbg = nullptr;
    if (const char* tr = getenv("MMK_SMALL_TRACE"))
        a.dbg = reinterpret_cast<long long*>(strtoull(tr, nullptr, 0));
    out->scratch = scratch;
    auto seq = std::make_shared<unsigned int>(0);
    out->fn = [a, G, smem, seq](cudaStream_t s) -> int {
        PetSmall<T> arg = a;
        arg.epoch0 = (++*seq) << 20;
        void* args[] = {&arg};
        const bool pr = mmk_host::prof_on();
        if (pr) mmk_host::prof_start("pet_small", s);
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)pet_small_kernel<T>, dim3(G),
                                                    dim3(kPetSmallThr), args, smem, s);
        if (pr) mmk_host::prof_stop(s);
        if (e != cudaSuccess) return mmk_host::cuda_status(e, "pet_small_kernel");
        return MMK_OK;
    };
    return MMK_OK;
}

int pet_prepare(int dtype, const int32_t* rptr, const int32_t* ridx, const void* rval,
                const int32_t* cptr, const int32_t* cidx, const void* cval, const void* y,
                void* lamA, void* lamB, long long d, long long p, const int32_t* nbr_ptr,
                const int32_t* nbr_idx, double mu, const mmk_stop_rule* rule, double* trace,
                int64_t* tstamp, int64_t* ctl, int64_t* err, Launch* out) {
    if (rule->batch < 2 || (rule->batch & 1)) {
        mmk_host::set_error("engine batch must be an even number >= 2");
        return MMK_E_SHAPE;
    }
    if (dtype == MMK_F32)
        return pet_prepare_t<float>(rptr, ridx, rval, cptr, cidx, cval, y, lamA, lamB, d, p,
                                    nbr_ptr, nbr_idx, mu, rule, trace, tstamp, ctl, err, out);
    return pet_prepare_t<double>(rptr, ridx, rval, cptr, cidx, cval, y, lamA, lamB, d, p, nbr_ptr,
                                 nbr_idx, mu, rule, trace, tstamp, ctl, err, out);
}

}  // namespace mmk_small
