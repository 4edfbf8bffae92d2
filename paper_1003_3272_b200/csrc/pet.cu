// pet.cu -- penalized Poisson MM for emission tomography (reference
// pet.py:288-417), as a single pass over the system matrix E.
//
// Phase A (pet_project_kernel): a CTA owns kRays consecutive rays.  Each warp
// forms one forward projection m_i = E_i . lam (vectorised row loads, fp64
// accumulation), then the count ratio r_i = y_i / m_i and the loglik term
// y_i ln m_i - m_i (pet.py:288-315).  The CTA then back-projects its own rays
// while their rows are still in L1/L2: b^R_j = sum_{i in R} e_ij r_i, written
// as a per-CTA partial.  E is therefore streamed from HBM once per iteration
// (d*p*sizeof(T) bytes) -- the kernel's roofline.
// pet_reduce_kernel sums the CTA partials in CTA order (deterministic) into
// red = [b | loglik]; a multi-GPU caller all-reduces red across ray shards.
//
// Phase B (pet_pixel_kernel): per pixel c_j = lam_j b_j, neighbour sums over
// the CSR lattice (pet.py:204-210), EM floor or positive-root update
// (pet.py:390-417), and the roughness penalty at lam (pet.py:326-338); the
// last CTA assembles f = loglik - mu/2 * penalty.
#include "mmk_common.cuh"

namespace {

using namespace mmk;

constexpr int kRays = 8;      // rays (warps) per projection CTA
constexpr int kPixThreads = 256;

template <typename T>
__device__ __forceinline__ double row_dot(const T* __restrict__ e, const T* __restrict__ lam,
                                          long long p, int lane) {
    double acc = 0.0;
    if (sizeof(T) == 4 && (p & 3) == 0 && ((reinterpret_cast<uintptr_t>(e) & 15) == 0)) {
        const float4* e4 = reinterpret_cast<const float4*>(e);
        const float4* l4 = reinterpret_cast<const float4*>(lam);
        for (long long q = lane; q < p / 4; q += 32) {
            const float4 a = __ldg(e4 + q), b = __ldg(l4 + q);
            acc = fma((double)a.x, (double)b.x, acc);
            acc = fma((double)a.y, (double)b.y, acc);
            acc = fma((double)a.z, (double)b.z, acc);
            acc = fma((double)a.w, (double)b.w, acc);
        }
    } else if (sizeof(T) == 8 && (p & 1) == 0 && ((reinterpret_cast<uintptr_t>(e) & 15) == 0)) {
        const double2* e2 = reinterpret_cast<const double2*>(e);
        const double2* l2 = reinterpret_cast<const double2*>(lam);
        for (long long q = lane; q < p / 2; q += 32) {
            const double2 a = __ldg(e2 + q), b = __ldg(l2 + q);
            acc = fma(a.x, b.x, acc);
            acc = fma(a.y, b.y, acc);
        }
    } else {
        for (long long q = lane; q < p; q += 32) acc = fma((double)e[q], (double)lam[q], acc);
    }
    return warp_sum(acc);
}

template <typename T>
__global__ void __launch_bounds__(kRays * 32)
pet_project_kernel(const T* __restrict__ E, long long lde, const T* __restrict__ y,
                   const T* __restrict__ lam, long long d, long long p,
                   double* __restrict__ bpart, double* __restrict__ llpart, int64_t* err) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long ray0 = (long long)blockIdx.x * kRays;
    __shared__ double ratio[kRays];
    __shared__ double ll[kRays];
    const long long i = ray0 + warp;
    if (i < d) {
        const double m = row_dot(E + i * lde, lam, p, lane);
        if (lane == 0) {
            const double yi = (double)y[i];
            double r = 0.0, l = -m;
            if (yi > 0.0) {
                if (m == 0.0) flag_error(err, MMK_E_NUMERICS, err_at(1, i));
                r = yi / m;
                l += yi * log(m);
            }
            ratio[warp] = r;
            ll[warp] = l;
        }
    } else if (lane == 0) {
        ratio[warp] = 0.0;
        ll[warp] = 0.0;
    }
    __syncthreads();
    const long long left = d - ray0;
    const int nr = left < kRays ? (int)left : kRays;
    double* out = bpart + (long long)blockIdx.x * p;
    for (long long j = threadIdx.x; j < p; j += blockDim.x) {
        double b = 0.0;
        for (int w = 0; w < nr; ++w) b = fma((double)E[(ray0 + w) * lde + j], ratio[w], b);
        out[j] = b;
    }
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < nr; ++w) s += ll[w];
        llpart[blockIdx.x] = s;
    }
}

__global__ void pet_reduce_kernel(const double* __restrict__ bpart, const double* __restrict__ llpart,
                                  int nparts, long long p, double* __restrict__ red) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < p) {
        double b = 0.0;
        for (int s = 0; s < nparts; ++s) b += bpart[(long long)s * p + j];
        red[j] = b;
    }
    if (blockIdx.x == 0) {
        __shared__ double sc[32];
        const double t = block_sum_array(llpart, nparts, sc);
        if (threadIdx.x == 0) red[p] = t;
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
    if (j < p) {
        const double lj = (double)lam[j];
        if ((flags & MMK_PET_CHECK_POSITIVE) && !(lj > 0.0)) flag_error(err, MMK_E_DOMAIN, err_at(3, j));
        const int k0 = nptr[j], k1 = nptr[j + 1];
        double nbr = 0.0;
        for (int t = k0; t < k1; ++t) {
            const int k = nidx[t];
            const double lk = (double)lam[k];
            nbr += lk;
            if (k > j) pen += (lj - lk) * (lj - lk);
        }
        if (flags & MMK_PET_UPDATE) {
            const double c = lj * red[j];
            double out;
            if (mu == 0.0) {
                out = c;
            } else {
                const double deg = (double)(k1 - k0);
                const double a = -2.0 * mu * deg;
                const double b = mu * (deg * lj + nbr) - 1.0;
                const double disc = b * b - 4.0 * a * c;
                if (disc < 0.0) flag_error(err, MMK_E_NUMERICS, err_at(2, j));
                const double sq = sqrt(disc);
                out = (b < 0.0) ? 2.0 * c / (sq - b) : (-b - sq) / ((a < 0.0) ? 2.0 * a : -1.0);
            }
            lam_out[j] = (T)fmax(out, num<T>::floor());
        }
    }
    if (!(flags & MMK_PET_OBJECTIVE)) return;
    __shared__ double sc[32];
    const double bs = block_sum(pen, sc);
    if (threadIdx.x == 0) penpart[blockIdx.x] = bs;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(penpart, gridDim.x, sc);
        if (threadIdx.x == 0) {
            double f = red[p];
            if (mu > 0.0) f -= 0.5 * mu * tot;
            *f_dev = f;
        }
    }
}

struct PetWs {
    unsigned int* counter;
    double* bpart;
    double* llpart;
    double* penpart;
    int nparts;
};

size_t pet_ws_layout(long long d, long long p, void* base, PetWs* L) {
    const int nparts = ceil_div(d > 0 ? d : 1, kRays);
    const int npix = ceil_div(p, kPixThreads);
    size_t off = 256;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    // counter + penalty partials first so phase B finds them at offsets that
    // do not depend on the ray count
    size_t o_pen = take(sizeof(double) * (size_t)npix);
    size_t o_ll = take(sizeof(double) * (size_t)nparts);
    size_t o_b = take(sizeof(double) * (size_t)nparts * (size_t)p);
    if (L && base) {
        char* c = reinterpret_cast<char*>(base);
        L->counter = reinterpret_cast<unsigned int*>(c);
        L->bpart = reinterpret_cast<double*>(c + o_b);
        L->llpart = reinterpret_cast<double*>(c + o_ll);
        L->penpart = reinterpret_cast<double*>(c + o_pen);
        L->nparts = nparts;
    }
    return off;
}

template <typename T>
int pet_a(const T* E, long long lde, const T* y, const T* lam, long long d, long long p,
          const PetWs& L, double* red, int64_t* err, cudaStream_t st) {
    if (d > 0) {
        MMK_LAUNCH("pet_project", st,
                   (pet_project_kernel<T><<<L.nparts, kRays * 32, 0, st>>>(
                       E, lde, y, lam, d, p, L.bpart, L.llpart, err)));
        MMK_CHECK_LAUNCH("pet_project_kernel");
        MMK_LAUNCH("pet_reduce", st,
                   (pet_reduce_kernel<<<ceil_div(p, 256), 256, 0, st>>>(L.bpart, L.llpart,
                                                                       L.nparts, p, red)));
    } else {
        cudaMemsetAsync(red, 0, sizeof(double) * (size_t)(p + 1), st);
    }
    MMK_CHECK_LAUNCH("pet_reduce_kernel");
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

}  // namespace

extern "C" int mmk_pet_ws_bytes(int dtype, int64_t d, int64_t p, size_t* out) {
    (void)dtype;
    *out = pet_ws_layout(d, p, nullptr, nullptr);
    return MMK_OK;
}

extern "C" int64_t mmk_pet_reduce_len(int64_t p) { return p + 1; }

extern "C" int mmk_pet_iter_a(int dtype, const void* E, int64_t lde, const void* y,
                              const void* lam, int64_t d, int64_t p, void* ws, size_t ws_bytes,
                              double* red, int64_t* err_dev, void* stream) {
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
        return pet_a<float>((const float*)E, lde, (const float*)y, (const float*)lam, d, p, L, red,
                            err_dev, st);
    if (dtype == MMK_F64)
        return pet_a<double>((const double*)E, lde, (const double*)y, (const double*)lam, d, p, L,
                             red, err_dev, st);
    mmk_host::set_error("unknown dtype %d", dtype);
    return MMK_E_SHAPE;
}

extern "C" int mmk_pet_iter_b(int dtype, const void* lam, void* lam_out, int64_t p,
                              const int32_t* nbr_ptr, const int32_t* nbr_idx, double mu, int flags,
                              const double* red, void* ws, size_t ws_bytes, double* f_dev,
                              int64_t* err_dev, void* stream) {
    if (p < 1) {
        mmk_host::set_error("bad PET pixel count %lld", (long long)p);
        return MMK_E_SHAPE;
    }
    PetWs L;
    int rc = check_ws(0, p, ws, ws_bytes, &L);
    if (rc) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
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
    int rc = mmk_pet_iter_a(dtype, E, lde, y, lam, d, p, ws, ws_bytes, red, err_dev, stream);
    if (rc) return rc;
    return mmk_pet_iter_b(dtype, lam, lam_out, p, nbr_ptr, nbr_idx, mu, flags, red, ws, ws_bytes,
                          f_dev, err_dev, stream);
}
