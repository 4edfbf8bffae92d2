// pet_siddon.cu -- the PET system matrix on the device:
// the reference's Siddon chord-length build (pet.py:69-132) is a Python loop
// over rays (0.68 s at 64 x 64, minutes at 256 x 256) producing a dense
// matrix that is ~99 % zeros.  One thread per ray computes the same crossing
// parameters, merges the sorted vertical / horizontal crossings, and emits
// (pixel, chord length) per interval into a fixed-capacity row (ELL layout);
// the host glue compacts the rows to CSR, sorts them stably by pixel to CSC
// and normalises the columns in ray order.
//
// Arithmetic follows the reference operation by operation in fp64 with
// explicitly rounded intrinsics (no FMA contraction), so chord lengths agree
// with the reference to the rounding of `hypot`.
#include "mmk_common.cuh"

namespace {

__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// crossing parameter of grid line k along one axis, walking in increasing t
struct Axis {
    double start, delta;
    int k, kend, step;   // next line index, one past the last, direction
    bool active;
};

__device__ __forceinline__ double axis_t(const Axis& a, const double* __restrict__ lines) {
    return ddiv(dsub(lines[a.k], a.start), a.delta);
}

__global__ void __launch_bounds__(128)
pet_siddon_kernel(const double* __restrict__ det, int n_det, int side,
                  const double* __restrict__ lines, int cap, int* __restrict__ idx,
                  double* __restrict__ val, int* __restrict__ cnt) {
    const long long n_rays = (long long)n_det * (n_det - 1) / 2;
    const long long ray = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (ray >= n_rays) return;
    // detector pair (a, b), a < b, in the reference's loop order
    int a = 0;
    long long base = 0;
    while (base + (n_det - 1 - a) <= ray) {
        base += n_det - 1 - a;
        ++a;
    }
    const int b = a + 1 + (int)(ray - base);
    const double p0x = det[2 * a], p0y = det[2 * a + 1];
    const double dx = dsub(det[2 * b], p0x), dy = dsub(det[2 * b + 1], p0y);
    const double length = hypot(dx, dy);
    int* ri = idx + ray * cap;
    double* rv = val + ray * cap;
    int nout = 0;
    double t_lo = 0.0, t_hi = 1.0;
    const double st[2] = {p0x, p0y}, de[2] = {dx, dy};
    for (int ax = 0; ax < 2; ++ax) {
        if (de[ax] == 0.0) {
            if (!(-1.0 <= st[ax] && st[ax] <= 1.0)) {
                cnt[ray] = 0;
                return;
            }
        } else {
            double lo = ddiv(dsub(-1.0, st[ax]), de[ax]);
            double hi = ddiv(dsub(1.0, st[ax]), de[ax]);
            if (lo > hi) {
                const double t = lo;
                lo = hi;
                hi = t;
            }
            t_lo = fmax(t_lo, lo);
            t_hi = fmin(t_hi, hi);
        }
    }
    if (t_lo >= t_hi) {
        cnt[ray] = 0;
        return;
    }
    // the sorted crossings of each axis inside (t_lo, t_hi): lines ascend,
    // so t ascends with k for delta > 0 and descends for delta < 0
    Axis A[2];
    for (int ax = 0; ax < 2; ++ax) {
        Axis& x = A[ax];
        x.start = st[ax];
        x.delta = de[ax];
        x.active = de[ax] != 0.0;
        if (de[ax] > 0.0) {
            x.k = 0;
            x.kend = side + 1;
            x.step = 1;
        } else {
            x.k = side;
            x.kend = -1;
            x.step = -1;
        }
        if (x.active)   // skip crossings at or before t_lo
            while (x.k != x.kend && !(axis_t(x, lines) > t_lo)) x.k += x.step;
    }
    const double h = 2.0 / (double)side;
    double prev = t_lo;
    int last_pix = -1;
    while (true) {
        // next cut: the smaller pending crossing below t_hi, else t_hi
        double cut = t_hi;
        int from = -1;
        for (int ax = 0; ax < 2; ++ax) {
            if (!A[ax].active || A[ax].k == A[ax].kend) continue;
            const double t = axis_t(A[ax], lines);
            if (!(t < t_hi)) continue;
            if (t < cut) {
                cut = t;
                from = ax;
            }
        }
        // equal crossings from both axes (a grid corner) are one cut (np.unique)
        for (int ax = 0; ax < 2; ++ax)
            if (A[ax].active && A[ax].k != A[ax].kend && from >= 0 && axis_t(A[ax], lines) == cut)
                A[ax].k += A[ax].step;
        if (cut > prev) {
            const double mid = dmul(0.5, dadd(prev, cut));
            const double x = dadd(p0x, dmul(mid, dx));
            const double y = dadd(p0y, dmul(mid, dy));
            int ix = (int)ddiv(dadd(x, 1.0), h);
            int iy = (int)ddiv(dsub(1.0, y), h);
            ix = ix < side - 1 ? ix : side - 1;
            iy = iy < side - 1 ? iy : side - 1;
            const int pix = iy * side + ix;
            const double seg = dmul(dsub(cut, prev), length);
            if (pix == last_pix && nout > 0) {
                rv[nout - 1] = dadd(rv[nout - 1], seg);
            } else if (nout < cap) {
                ri[nout] = pix;
                rv[nout] = seg;
                ++nout;
                last_pix = pix;
            }
        }
        prev = cut;
        if (from < 0) break;
    }
    cnt[ray] = nout;
}

}  // namespace

extern "C" int mmk_pet_siddon(const double* det, int n_det, int side, const double* lines,
                              int cap, int* idx, double* val, int* cnt, void* stream) {
    MMK_NVTX("mmk_pet_siddon");
    if (n_det < 2 || side < 1 || cap < 2 * side + 3) {
        mmk_host::set_error("bad Siddon geometry: detectors=%d side=%d cap=%d (cap >= 2 side + 3)",
                            n_det, side, cap);
        return MMK_E_SHAPE;
    }
    const long long n_rays = (long long)n_det * (n_det - 1) / 2;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    MMK_LAUNCH("pet_siddon", st,
               (pet_siddon_kernel<<<(unsigned)((n_rays + 127) / 128), 128, 0, st>>>(
                   det, n_det, side, lines, cap, idx, val, cnt)));
    MMK_CHECK_LAUNCH("pet_siddon_kernel");
    return MMK_OK;
}
