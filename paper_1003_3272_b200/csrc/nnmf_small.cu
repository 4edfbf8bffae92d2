// nnmf_small.cu -- persistent cooperative kernel running whole batches of
// Frobenius NNMF MM iterations (nnmf.py:84-110 under run_mm, driver.py:101-149)
// for small problems such as BASELINE config 1 (2429 x 361, r = 10).
//
// One CTA per SM, rows of X / V split contiguously over the CTAs; each CTA
// keeps its own copy of W in shared memory.  Per iteration k, state
// (V_k, W_k) in slot s -> (V_k+1, W_k+1) in slot s^1:
//   phase 1  G_W = W W^T (fp64, every CTA, same order); for my rows (warp per
//            row) q = x_i W^T, the residual of (V_k, W_k) (the lagged
//            objective, fp64) and V'_i = v_i * q / (v_i G_W + 1e-300); then
//            per-CTA partials of V'^T X (thread per column) and V'^T V' in
//            fp64 -> part[cta][.]
//   barrier
//   phase 2  the entries of part are split over the CTAs; each sums its
//            entries over the CTAs in a fixed order (8 lanes per entry, fixed
//            xor tree) -> tot[.]; the owner of the residual entry applies the
//            stopping rule (mm_control) to f_k
//   barrier
//   phase 3  unless stopped: W_k+1 = W_k * P / (G_V W_k + 1e-300) in fp64 in
//            every CTA's shared copy; column j is stored to global by CTA
//            j mod G.
// Two grid barriers per iteration instead of six dependent kernel launches;
// every reduction has a fixed order, so runs are bitwise reproducible.
// X rows, V rows, W (storage type and fp64) and the reduced totals live in
// shared memory; all pointers into it are offsets of the dynamic smem array
// so loads and stores stay LDS/STS.  MMK_SMALL_TRACE=<device int64 pointer>
// records clock64 phase stamps of CTA 0 (12 per iteration, first 64).
// Measured at C1 (fp32, B200): ~41k cycles per iteration (vs ~90k for the
// six-kernel graph body) -- phase 1 rows 8.4k, W partials 5k, G_W 4.7k, the
// W update 5.7k, reduction 3.8k, two barriers ~5k each (mostly waiting for
// the slowest CTA).
#include <memory>

#include "mm_control.cuh"
#include "small_engine.h"

namespace {

using namespace mmk;

constexpr int kThr = 512;
constexpr int kWarps = kThr / 32;
constexpr int kSmallR = 16;
constexpr int kSub = 16;                // lanes per reduced entry in phase 2
constexpr int kPartPerLane = (kNumSMs + kSub - 1) / kSub;   // partials per lane (G <= 148)
constexpr int kMaxRowsPerCta = 64;
constexpr long long kMaxElems = 1LL << 22;

template <typename T>
struct SmallNnmf {
    const T* X;
    long long ldx;
    T* V[2];
    T* W[2];
    int m, n, r, rpc, E;
    double* part;           // [G][E]
    double* tot;            // [E]
    unsigned int* bar;      // [2] the decision of the controlling thread
    long long* ctl;
    double* trace;
    long long* tstamp;
    int64_t* err;
    mmk_stop_rule rule;
    long long* dbg;         // optional: CTA 0 phase timestamps (MMK_SMALL_TRACE)
    unsigned int* flags;    // [32 * G] barrier slots
    unsigned int epoch0;    // first barrier epoch of this launch
};

// POIS: the Poisson log fit (nnmf.py:178-242) instead of the Frobenius loss:
// V' = V sqrt((R W^T) / (1 W^T)), W' = W sqrt((V'^T R') / (V'^T 1)) with
// R = X / (V W) masked to x > 0, objective sum x ln b - b (fp64); the
// reduction entries are [P (r x n) | colsum V' (r) | f].
template <typename T, int R, bool POIS>
__global__ void __launch_bounds__(kThr) nnmf_small_kernel(SmallNnmf<T> a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    constexpr int r = R;
    const int n = a.n, E = a.E, rpc = a.rpc;
    // fp64 arrays first (8-byte aligned offsets), then the storage-type ones;
    // every pointer is sm_raw + a byte offset so the compiler keeps them in
    // the shared window (LDS/STS, no aliasing with global memory)
    double* const Gw = reinterpret_cast<double*>(sm_raw);                 // r x r
    double* const Gv = Gw + kSmallR * kSmallR;                            // r x r
    double* const Wd0 = Gv + kSmallR * kSmallR;                           // 2 x (r x n): W fp64
    double* const Pt = Wd0 + 2 * r * n;                                   // r x n + r x r totals
    T* const Ws = reinterpret_cast<T*>(Pt + r * n + r * r);               // r x n   W (storage)
    T* const Xs = Ws + r * n;                                             // rpc x n my rows of X
    T* const Vs0 = Xs + rpc * n;                                          // rpc x r my rows of V
    T* const Vs1 = Vs0 + rpc * r;
    int wcur = 0;                                        // Wd0[wcur * r * n ...] is W (fp64)
    __shared__ double sc[32];
    __shared__ int decision;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x, G = gridDim.x;
    const int row0 = c * rpc, nrows = max(0, min(a.m, row0 + rpc) - row0);
    const int e0 = (int)((long long)c * E / G), e1 = (int)((long long)(c + 1) * E / G);
    const int jlo = (int)((long long)c * n / G), jhi = (int)((long long)(c + 1) * n / G);
    // launch prologue: W, my rows of X and V into shared memory (many loads in flight)
#pragma unroll 4
    for (int idx = tid; idx < r * n; idx += kThr) {
        const T w = a.W[0][idx];
        Ws[idx] = w;
        Wd0[idx] = (double)w;
    }
#pragma unroll 4
    for (int idx = tid; idx < nrows * n; idx += kThr) {
        const int i = idx / n, j = idx - i * n;
        Xs[idx] = a.X[(long long)(row0 + i) * a.ldx + j];
    }
    for (int idx = tid; idx < nrows * r; idx += kThr) Vs0[idx] = a.V[0][(long long)row0 * r + idx];
    int slot = 0;
    int iter_local = 0;
    unsigned int epoch = a.epoch0;
    auto stamp = [&](int ph) {
        if (a.dbg && c == 0 && tid == 0 && iter_local < 64) a.dbg[iter_local * 12 + ph] = clock64();
    };
    for (;;) {
        __syncthreads();
        stamp(0);
        // ---- phase 1 ---------------------------------------------------------
        if constexpr (POIS) {
            // ws_k = sum_j w_kj (fp64): kWsSeg column segments per k, combined in order
            constexpr int SEG = 256 / R >= 16 ? 16 : 256 / R;   // scratch (Gv) <= 256
            for (int t = tid; t < R * SEG; t += kThr) {
                const int k = t / SEG, sg = t % SEG;
                const int j0 = (int)((long long)sg * n / SEG), j1 = (int)((long long)(sg + 1) * n / SEG);
                const double* Wd = Wd0 + wcur * r * n;
                double s0 = 0.0, s1 = 0.0;
                int j = j0;
                for (; j + 1 < j1; j += 2) {
                    s0 += Wd[k * n + j];
                    s1 += Wd[k * n + j + 1];
                }
                if (j < j1) s0 += Wd[k * n + j];
                Gv[t] = s0 + s1;
            }
            __syncthreads();
            for (int k = tid; k < R; k += kThr) {
                double s = 0.0;
                for (int sg = 0; sg < SEG; ++sg) s += Gv[k * SEG + sg];
                Gw[k] = s;
            }
            __syncthreads();
        } else {
        // G_W = W W^T: the r(r+1)/2 entries x kGwSeg column segments over the
        // threads, segments combined in order (fp64)
        {
            constexpr int NE = r * (r + 1) / 2;
            // segments per entry: enough tasks for the block, scratch (Gv) <= 256
            constexpr int SEG = (NE * 4 <= kThr && NE * 4 <= 256) ? 4
                                : ((NE * 2 <= kThr && NE * 2 <= 256) ? 2 : 1);
            for (int t = tid; t < NE * SEG; t += kThr) {
                const int e = t / SEG, sg = t % SEG;
                int p = 0, rem = e;
                while (rem >= r - p) { rem -= r - p; ++p; }
                const int q = p + rem;
                const int j0 = (int)((long long)sg * n / SEG), j1 = (int)((long long)(sg + 1) * n / SEG);
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int j = j0;
                const double* Wd = Wd0 + wcur * r * n;
                for (; j + 3 < j1; j += 4) {
                    s0 = fma(Wd[p * n + j], Wd[q * n + j], s0);
                    s1 = fma(Wd[p * n + j + 1], Wd[q * n + j + 1], s1);
                    s2 = fma(Wd[p * n + j + 2], Wd[q * n + j + 2], s2);
                    s3 = fma(Wd[p * n + j + 3], Wd[q * n + j + 3], s3);
                }
                for (; j < j1; ++j) s0 = fma(Wd[p * n + j], Wd[q * n + j], s0);
                Gv[t] = (s0 + s1) + (s2 + s3);   // Gv is free until phase 3: segment scratch
            }
            __syncthreads();
            for (int t = tid; t < r * r; t += kThr) {
                const int p = t / r, q = t - p * r;
                const int pp = p < q ? p : q, qq = p < q ? q : p;
                const int e = pp * r - pp * (pp - 1) / 2 + (qq - pp);
                double s = 0.0;
                for (int sg = 0; sg < SEG; ++sg) s += Gv[e * SEG + sg];
                Gw[t] = s;
            }
            __syncthreads();
        }
        }
        stamp(1);
        const T* Vc = slot ? Vs1 : Vs0;
        T* Vn = slot ? Vs0 : Vs1;
        T* Vo = a.V[slot ^ 1];
        double res = 0.0;
        for (int i = warp; i < nrows; i += kWarps) {
            T v[kSmallR], q[kSmallR];
#pragma unroll
            for (int k = 0; k < kSmallR; ++k) {
                v[k] = k < r ? Vc[i * r + k] : T(0);
                q[k] = T(0);
            }
            const T* xr = Xs + i * n;
            for (int j = lane; j < n; j += 32) {
                const T x = xr[j];
                if constexpr (POIS) {
                    T b = T(0);
#pragma unroll
                    for (int k = 0; k < R; ++k) b = fma(v[k], Ws[k * n + j], b);
                    res -= (double)b;
                    if (x > T(0)) {
                        if (b == T(0)) {
                            flag_error(a.err, MMK_E_NUMERICS, err_at(1, (long long)(row0 + i) * n + j));
                            continue;
                        }
                        res = fma((double)x, log((double)b), res);
                        const T ratio = x / b;
#pragma unroll
                        for (int k = 0; k < R; ++k) q[k] = fma(ratio, Ws[k * n + j], q[k]);
                    }
                } else {
                    T rec = T(0);
#pragma unroll
                    for (int k = 0; k < kSmallR; ++k) {
                        if (k < r) {
                            const T w = Ws[k * n + j];
                            q[k] = fma(x, w, q[k]);
                            rec = fma(v[k], w, rec);
                        }
                    }
                    const double d = (double)x - (double)rec;
                    res = fma(d, d, res);
                }
            }
            T qk = T(0), vk = T(0);
            double den = 0.0;
#pragma unroll
            for (int k = 0; k < kSmallR; ++k) {
                if (k < r) {
                    const T t = warp_sum(q[k]);
                    if (k == lane) {
                        qk = t;
                        vk = v[k];
                    }
                    if (!POIS && lane < r) den = fma((double)v[k], Gw[k * r + lane], den);
                }
            }
            if (lane < r) {
                const T nv = POIS ? (T)((double)vk * sqrt((double)qk / (Gw[lane] + kDenomGuard)))
                                  : (T)((double)vk * ((double)qk / (den + kDenomGuard)));
                Vo[(long long)(row0 + i) * r + lane] = nv;
                Vn[i * r + lane] = nv;
            }
        }
        __syncthreads();
        stamp(2);
        double* pc = a.part + (long long)c * E;
        for (int j = tid; j < n; j += kThr) {
            // a CTA's <= 64 rows accumulate in the storage type (the graph
            // path's wpart does the same over far longer row ranges); fp64 across CTAs
            T acc[kSmallR];
#pragma unroll
            for (int k = 0; k < kSmallR; ++k) acc[k] = T(0);
            if constexpr (POIS) {
                T wj[R];
#pragma unroll
                for (int k = 0; k < R; ++k) wj[k] = Ws[k * n + j];
                for (int i = 0; i < nrows; ++i) {
                    const T x = Xs[i * n + j];
                    if (!(x > T(0))) continue;
                    T b = T(0);
#pragma unroll
                    for (int k = 0; k < R; ++k) b = fma(Vn[i * r + k], wj[k], b);
                    if (b == T(0)) {
                        flag_error(a.err, MMK_E_NUMERICS, err_at_update(2, (long long)(row0 + i) * n + j));
                        continue;
                    }
                    const T ratio = x / b;
#pragma unroll
                    for (int k = 0; k < R; ++k) acc[k] = fma(Vn[i * r + k], ratio, acc[k]);
                }
            } else {
                for (int i = 0; i < nrows; ++i) {
                    const T x = Xs[i * n + j];
#pragma unroll
                    for (int k = 0; k < kSmallR; ++k)
                        if (k < r) acc[k] = fma(Vn[i * r + k], x, acc[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < kSmallR; ++k)
                if (k < r) pc[(long long)k * n + j] = (double)acc[k];
        }
        if constexpr (POIS) {
            for (int k = tid; k < R; k += kThr) {
                double s = 0.0;
                for (int i = 0; i < nrows; ++i) s += (double)Vn[i * r + k];
                pc[(long long)r * n + k] = s;
            }
        } else {
            for (int t = tid; t < r * r; t += kThr) {
                const int p = t / r, q = t - p * r;
                double s = 0.0;
                for (int i = 0; i < nrows; ++i)
                    s = fma((double)Vn[i * r + p], (double)Vn[i * r + q], s);
                pc[(long long)r * n + t] = s;
            }
        }
        const double bres = block_sum(res, sc);
        if (tid == 0) pc[E - 1] = bres;
        stamp(3);
        grid_sync_flags(a.flags, ++epoch);
        stamp(4);
        // ---- phase 2: kSub lanes per entry, all their loads in flight ---------
        {
            const int g = tid / kSub, sub = tid % kSub;
            for (int base = e0; base < e1; base += kThr / kSub) {
                const int e = base + g;
                double s = 0.0;
                if (e < e1) {
                    double t[kPartPerLane];
#pragma unroll
                    for (int u = 0; u < kPartPerLane; ++u) {
                        const int cc = sub + u * kSub;
                        t[u] = cc < G ? __ldcg(a.part + (long long)cc * E + e) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < kPartPerLane; ++u) s += t[u];
                }
#pragma unroll
                for (int o = kSub / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (sub == 0 && e < e1) {
                    a.tot[e] = s;
                    if (e == E - 1) {
                        a.ctl[MMK_CTL_FCUR] = ctl_bits(s);
                        a.bar[2] = (unsigned int)mm_control(slot, a.ctl, a.trace, a.tstamp,
                                                            reinterpret_cast<const long long*>(a.err),
                                                            a.rule, s);
                    }
                }
            }
        }
        stamp(5);
        grid_sync_flags(a.flags, ++epoch);
        stamp(6);
        if (tid == 0) decision = (int)*(volatile unsigned int*)(a.bar + 2);
        __syncthreads();
        const int dcs = decision;
        if (dcs == kMmStop) return;
        // ---- phase 3 ---------------------------------------------------------
        // all totals into shared memory at once (one L2 round trip)
        stamp(8);
        constexpr int kSide = POIS ? R : R * R;   // colsum V' (Poisson) or G_V
        for (int t0 = 0; t0 < r * n + kSide; t0 += kThr * 8) {
            double v8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * kThr + tid;
                v8[u] = t < r * n + kSide ? __ldcg(a.tot + t) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * kThr + tid;
                if (t < r * n + kSide) Pt[t] = v8[u];
            }
        }
        __syncthreads();
        stamp(9);
        for (int t = tid; t < kSide; t += kThr) Gv[t] = Pt[r * n + t];
        __syncthreads();
        stamp(10);
        T* Wo = a.W[slot ^ 1];
        // W' column by column from the fp64 copy of W into the other fp64
        // buffer (no in-place hazard); the T copy is only read by phase 1
        {
            const int rd = wcur * r * n, wr = (wcur ^ 1) * r * n;
            for (int j = tid; j < n; j += kThr) {
                double wc[R];
#pragma unroll
                for (int l = 0; l < R; ++l) wc[l] = Wd0[rd + l * n + j];
                const bool mine = j >= jlo && j < jhi;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    T nw;
                    if constexpr (POIS) {
                        nw = (T)(wc[k] * sqrt(Pt[k * n + j] / (Gv[k] + kDenomGuard)));
                    } else {
                        double den = 0.0;
#pragma unroll
                        for (int l = 0; l < R; ++l) den = fma(Gv[k * R + l], wc[l], den);
                        nw = (T)(wc[k] * (Pt[k * n + j] / (den + kDenomGuard)));
                    }
                    Wd0[wr + k * n + j] = (double)nw;
                    Ws[k * n + j] = nw;
                    if (mine) Wo[(long long)k * n + j] = nw;
                }
            }
            wcur ^= 1;
        }
        __syncthreads();
        stamp(7);
        ++iter_local;
        if (dcs == kMmPause) return;
        slot ^= 1;
    }
}

template <typename T, bool POIS>
void* kernel_for(int r) {
    switch (r) {
#define MMK_SMALL_R(R) \
    case R:            \
        return reinterpret_cast<void*>(&nnmf_small_kernel<T, R, POIS>);
        MMK_SMALL_R(1) MMK_SMALL_R(2) MMK_SMALL_R(3) MMK_SMALL_R(4) MMK_SMALL_R(5) MMK_SMALL_R(6)
        MMK_SMALL_R(7) MMK_SMALL_R(8) MMK_SMALL_R(9) MMK_SMALL_R(10) MMK_SMALL_R(11)
        MMK_SMALL_R(12) MMK_SMALL_R(13) MMK_SMALL_R(14) MMK_SMALL_R(15) MMK_SMALL_R(16)
#undef MMK_SMALL_R
        default:
            return nullptr;
    }
}

int grid_of(long long m) { return (int)(m < kNumSMs ? m : kNumSMs); }

template <typename T>
size_t smem_of(long long m, long long n, int r) {
    const int G = grid_of(m);
    const long long rpc = (m + G - 1) / G;
    return 2 * kSmallR * kSmallR * sizeof(double) +
           (size_t)(r * n + rpc * n + 2 * rpc * r) * sizeof(T) + (3 * (size_t)r * n + (size_t)r * r) * sizeof(double);
}

}  // namespace

namespace mmk_small {

bool nnmf_eligible(int dtype, long long m, long long n, long long r, long long ldx) {
    const char* env = getenv("MMK_SMALL_ENGINE");
    if (env && env[0] == '0') return false;
    if ((dtype != MMK_F32 && dtype != MMK_F64) || r < 1 || r > kSmallR || m < 1 || n < 1 ||
        ldx < n || m * n > kMaxElems)
        return false;
    const int G = grid_of(m);
    if ((m + G - 1) / G > kMaxRowsPerCta) return false;
    const size_t smem = dtype == MMK_F32 ? smem_of<float>(m, n, (int)r) : smem_of<double>(m, n, (int)r);
    return smem <= 200 * 1024;
}

template <typename T, bool POIS>
static int prepare_t(const void* X, long long ldx, void* VA, void* WA, void* VB, void* WB,
                     long long m, long long n, int r, const mmk_stop_rule* rule, double* trace,
                     int64_t* tstamp, int64_t* ctl, int64_t* err, Launch* out) {
    SmallNnmf<T> a;
    a.X = (const T*)X;
    a.ldx = ldx;
    a.V[0] = (T*)VA;
    a.V[1] = (T*)VB;
    a.W[0] = (T*)WA;
    a.W[1] = (T*)WB;
    a.m = (int)m;
    a.n = (int)n;
    a.r = r;
    const int G = grid_of(m);
    a.rpc = (int)((m + G - 1) / G);
    a.E = (int)(r * n + (POIS ? r : r * r) + 1);
    const size_t smem = smem_of<T>(m, n, r);
    const void* kern = kernel_for<T, POIS>(r);
    if (!kern) {
        mmk_host::set_error("nnmf_small: rank %d out of range", r);
        return MMK_E_SHAPE;
    }
    cudaError_t ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem);
    if (ce != cudaSuccess) return mmk_host::cuda_status(ce, "nnmf_small smem attribute");
    int per_sm = 0;
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThr, smem);
    if (ce != cudaSuccess || per_sm < 1) {
        mmk_host::set_error("nnmf_small: kernel does not fit an SM (smem %zu)", smem);
        return MMK_E_SHAPE;
    }
    constexpr int kHead = 32;   // bar words before the flag slots
    const size_t bar_bytes = (sizeof(unsigned int) * (kHead + 32 * G) + 255) / 256 * 256;
    const size_t bytes = bar_bytes + sizeof(double) * ((size_t)G * a.E + a.E);
    void* scratch = scratch_take(bytes, bar_bytes);
    if (!scratch) return mmk_host::cuda_status(cudaErrorMemoryAllocation, "nnmf_small scratch");
    a.bar = reinterpret_cast<unsigned int*>(scratch);
    a.flags = a.bar + kHead;
    a.epoch0 = 0;
    a.part = reinterpret_cast<double*>(reinterpret_cast<char*>(scratch) + bar_bytes);
    a.tot = a.part + (size_t)G * a.E;
    a.ctl = reinterpret_cast<long long*>(ctl);
    a.trace = trace;
    a.tstamp = reinterpret_cast<long long*>(tstamp);
    a.err = err;
    a.rule = *rule;
    a.dbg = nullptr;
    if (const char* tr = getenv("MMK_SMALL_TRACE")) {
        unsigned long long v = strtoull(tr, nullptr, 0);
        a.dbg = reinterpret_cast<long long*>(v);
    }
    out->scratch = scratch;
    // each iteration uses 2 barrier epochs; launches leave room for 2^20 of them
    auto seq = std::make_shared<unsigned int>(0);
    out->fn = [a, G, smem, kern, seq](cudaStream_t s) -> int {
        SmallNnmf<T> arg = a;
        arg.epoch0 = (++*seq) << 20;
        void* args[] = {&arg};
        const bool p = mmk_host::prof_on();
        if (p) mmk_host::prof_start("nnmf_small", s);
        cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(kThr), args, smem, s);
        if (p) mmk_host::prof_stop(s);
        if (e != cudaSuccess) return mmk_host::cuda_status(e, "nnmf_small_kernel");
        return MMK_OK;
    };
    return MMK_OK;
}

int nnmf_prepare(int dtype, const void* X, long long ldx, void* VA, void* WA, void* VB, void* WB,
                 long long m, long long n, int r, const mmk_stop_rule* rule, double* trace,
                 int64_t* tstamp, int64_t* ctl, int64_t* err, Launch* out, bool poisson) {
    if (rule->batch < 2 || (rule->batch & 1)) {
        mmk_host::set_error("engine batch must be an even number >= 2");
        return MMK_E_SHAPE;
    }
    if (dtype == MMK_F32)
        return poisson ? prepare_t<float, true>(X, ldx, VA, WA, VB, WB, m, n, r, rule, trace,
                                                tstamp, ctl, err, out)
                       : prepare_t<float, false>(X, ldx, VA, WA, VB, WB, m, n, r, rule, trace,
                                                 tstamp, ctl, err, out);
    return poisson ? prepare_t<double, true>(X, ldx, VA, WA, VB, WB, m, n, r, rule, trace, tstamp,
                                             ctl, err, out)
                   : prepare_t<double, false>(X, ldx, VA, WA, VB, WB, m, n, r, rule, trace, tstamp,
                                              ctl, err, out);
}

}  // namespace mmk_small
