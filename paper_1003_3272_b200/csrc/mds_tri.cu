// mds_tri.cu -- stress majorization for large unit-weight problems
// (BASELINE config 5: n = 65536, dim 3) over a PACKED UPPER TRIANGLE of Y.
//
// Reference: stress mds.py:92-102, mds_update mds.py:114-144, coincidence
// check mds.py:105-111.  With unit weights (W = 1 - I, cli.py:181) the
// reference update theta_i' = (theta_i (w + zs_i) + sum_j (1 - z_ij) theta_j)
// / (2 w), w = n - 1, z_ij = y_ij / d_ij (0 where y_ij = 0), is rewritten
// with S = sum_j theta_j and C_i = sum_{j != i} z_ij (theta_j - theta_i) as
//     theta_i' = (theta_i (w - 1) + S - C_i) / (2 w)
// (algebraically identical; C_i has no cancellation between zs_i theta_i
// and sum z_ij theta_j).  Stress = sum_{i<j} (y_ij - d_ij)^2.  Every
// unordered pair is visited ONCE: pair (i, j) adds z g to C_i and -z g to
// C_j (g = theta_j - theta_i), so Y is streamed from HBM once per iteration
// as n(n+128)/2 fp32 values -- half of a full-row pass.
//
// Layout: tiles of 128 x 128 points, (I, J) with I <= J, row-major over the
// upper triangle; each tile is 64 KB contiguous (diagonal tiles are stored
// full, entries beyond n are zero).  mmk_mds_tri_pack builds it from full
// rows on the device (and optionally validates symmetry / zero diagonal /
// finiteness / sign, mds.py:40-58).
//
// mds_tri_stage copies theta into a zero-padded [dim][n_pad] workspace copy
// and forms S (fp64, fixed order).  mds_tri_kernel (persistent, one CTA per
// SM, 8 warps): a CTA owns a contiguous range of tiles; each tile and the
// coordinates of its 128 column points arrive by 1-D bulk copies (TMA
// engine, one mbarrier) into a 3-stage ring.  Thread (ty, tx) owns an 8 x 8
// block of the tile: rows ty*8+a, columns {tx*4+b, 64+tx*4+b} (conflict-free
// 16-byte smem reads).  Pair arithmetic runs on packed fp32x2 (FFMA2 / FADD2
// / FMUL2 with the row coordinate as a broadcast scalar operand): 16 packed
// ops + 2 MUFU.RSQ per two pairs; one rsqrt gives z = y rsqrt(d2) and
// d = d2 rsqrt(d2).  d2 starts at 1e-37 so a coincident pair yields a huge
// but finite rsqrt: the per-thread rsqrt sum flags it, and only then the
// exact check (mds.py:105-111: error iff coincident AND y > 0) runs over that
// thread's 64 pairs.  Row accumulators C_i stay in registers across a CTA's
// run of tiles in one tile row; column accumulators are reduced across the
// CTA per tile and written as fp32 partials.  mds_tri_accum sums all
// partials of a point in a fixed order (deterministic, no float atomics) into
// the fp64 reduction buffer red = [n][dim] | stress -- the payload a sharded
// run all-reduces (tiles are split across ranks) -- and mds_tri_finish
// applies the update.
#include "mmk_common.cuh"
#include "tc_common.cuh"

namespace {

using namespace mmk;

constexpr int TB = 128;
constexpr int TILE = TB * TB;
constexpr uint32_t TILE_BYTES = TILE * 4;
constexpr int STAGES = 3;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr float kTiny = 1e-37f;
constexpr float kSuspect = 1e17f;
constexpr int kMaxTriDim = 3;
constexpr uint32_t TH_BYTES = kMaxTriDim * TB * 4;          // column coordinates per stage
constexpr uint32_t STAGE_BYTES = TILE_BYTES + TH_BYTES;

__host__ __device__ inline long long tri_index(long long I, long long J, long long T) {
    return I * T - I * (I - 1) / 2 + (J - I);
}

// tile row of linear tile index t (largest I with tri_index(I, I) <= t)
__host__ __device__ inline int row_of(long long t, int T) {
    int lo = 0, hi = T - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tri_index(mid, mid, T) <= t)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

// CTA c of G owns local tiles [start(c), start(c + 1))
__host__ __device__ inline long long cta_start(long long c, long long ntl, long long G) {
    return c * ntl / G;
}
__host__ __device__ inline int cta_of(long long u, long long ntl, long long G) {
    long long c = u * G / ntl;
    while (c + 1 < G && cta_start(c + 1, ntl, G) <= u) ++c;
    while (c > 0 && cta_start(c, ntl, G) > u) --c;
    return (int)c;
}

__device__ __forceinline__ float rsq(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

// column of slot (p, e) of thread tx: p < 2 -> tx*4 + 2p + e, else 64 + ...
__device__ __forceinline__ int jcol(int tx, int p, int e) {
    return (p < 2 ? tx * 4 + 2 * p : 64 + tx * 4 + 2 * (p - 2)) + e;
}

template <int DIM>
struct Rows {
    float nti[8][DIM];    // -theta_i (a broadcast scalar operand of FFMA2/FADD2)
    float2 C[8][DIM];     // row sums of z (theta_j - theta_i), packed over two j lanes
};

// All 64 pairs of this thread in one tile.  MASK: diagonal / edge tile,
// only pairs with i < j < n count.
template <int DIM, bool MASK>
__device__ __forceinline__ void tile_pairs(const float* __restrict__ ys, Rows<DIM>& R,
                                           const float2 (&tj)[4][DIM], float2 (&CJ)[4][DIM],
                                           float2& st2, float2& rsum, int tx, int ty,
                                           long long ig0, long long jg0, int n) {
    const float2 tiny2 = f2(kTiny, kTiny);
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const int il = ty * 8 + a;
        const float4 y0 = *reinterpret_cast<const float4*>(ys + il * TB + tx * 4);
        const float4 y1 = *reinterpret_cast<const float4*>(ys + il * TB + 64 + tx * 4);
        const float2 Y[4] = {f2(y0.x, y0.y), f2(y0.z, y0.w), f2(y1.x, y1.y), f2(y1.z, y1.w)};
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            float2 g[DIM];
            float2 d2 = tiny2;
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                g[k] = __fadd2_rn(tj[p][k], f2(R.nti[a][k], R.nti[a][k]));
                d2 = __ffma2_rn(g[k], g[k], d2);
            }
            const float2 rs = f2(rsq(d2.x), rsq(d2.y));
            float2 y = Y[p];
            if (MASK) {
                const long long ig = ig0 + il, j0 = jg0 + jcol(tx, p, 0);
                const float2 m = f2((j0 > ig && j0 < n) ? 1.f : 0.f,
                                    (j0 + 1 > ig && j0 + 1 < n) ? 1.f : 0.f);
                y = __fmul2_rn(y, m);
                d2 = __fmul2_rn(d2, m);
                rsum = __ffma2_rn(rs, m, rsum);
            } else {
                rsum = __fadd2_rn(rs, rsum);
            }
            const float2 z = __fmul2_rn(y, rs);
            const float2 r = __ffma2_rn(d2, neg2(rs), y);   // y - d
            st2 = __ffma2_rn(r, r, st2);
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                R.C[a][k] = __ffma2_rn(z, g[k], R.C[a][k]);
                CJ[p][k] = __ffma2_rn(z, g[k], CJ[p][k]);   // negated at the flush
            }
        }
    }
}

// Exact coincidence check (mds.py:105-111) for this thread's pairs; runs only
// when the rsqrt sum flagged a (possible) coincident pair.
template <int DIM>
__device__ __noinline__ void careful(const float* __restrict__ ys, const float* __restrict__ thp,
                                     long long npad, int tx, int ty, long long ig0,
                                     long long jg0, int n, int64_t* err) {
    for (int a = 0; a < 8; ++a) {
        const int il = ty * 8 + a;
        const long long ig = ig0 + il;
        for (int p = 0; p < 4; ++p) {
            for (int e = 0; e < 2; ++e) {
                const int jl = jcol(tx, p, e);
                const long long jg = jg0 + jl;
                if (!(jg > ig && jg < n)) continue;
                const float y = ys[il * TB + jl];
                if (!(y > 0.f)) continue;
                float d2 = 0.f;
                for (int k = 0; k < DIM; ++k) {
                    const float g = thp[k * npad + ig] - thp[k * npad + jg];
                    d2 = fmaf(g, g, d2);
                }
                if (d2 <= 0.f) flag_error(err, MMK_E_NUMERICS, err_at_update(1, ig * n + jg));
            }
        }
    }
}

// row partial of this CTA for a tile-row segment: reduce over the 16 tx lanes
// (one half-warp) sharing ty; lane tx == 0 writes its 8 points
template <int DIM>
__device__ __forceinline__ void flush_rows(const Rows<DIM>& R, float* __restrict__ rowpart,
                                           long long slot, int tx, int ty) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            float v = R.C[a][k].x + R.C[a][k].y;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (tx == 0) rowpart[(slot * DIM + k) * TB + ty * 8 + a] = v;
        }
    }
}

template <int DIM>
__global__ void __launch_bounds__(kThreads, 1)
mds_tri_kernel(const float* __restrict__ Yp, long long t0, long long ntl, int T, int n,
               const float* __restrict__ thp, long long npad, float* __restrict__ colpart,
               float* __restrict__ rowpart, int kmax, double* __restrict__ stpart, int64_t* err) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    float* red = reinterpret_cast<float*>(smem_raw + STAGES * STAGE_BYTES);   // 2 x [warp][DIM][TB]
    __shared__ uint64_t full[STAGES];
    __shared__ double sred[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tid & 15, ty = tid >> 4;
    const long long G = gridDim.x, c = blockIdx.x;
    const long long u0 = cta_start(c, ntl, G), u1 = cta_start(c + 1, ntl, G);
    const int cnt = (int)(u1 - u0);
    if (cnt <= 0) {
        if (tid == 0) stpart[c] = 0.0;
        return;
    }
    // tile coordinates of this CTA's first tile; later tiles advance J
    int I = row_of(t0 + u0, T);
    int J = I + (int)(t0 + u0 - tri_index(I, I, T));
    auto issue = [&](int k, int I_, int J_) {
        const int s = k % STAGES;
        uint8_t* dst = smem_raw + s * STAGE_BYTES;
        tc::mbar_expect_tx(&full[s], TILE_BYTES + DIM * TB * 4);
        tc::bulk_load(dst, Yp + (u0 + k) * (long long)TILE, TILE_BYTES, &full[s]);
        for (int k2 = 0; k2 < DIM; ++k2)
            tc::bulk_load(dst + TILE_BYTES + k2 * TB * 4, thp + k2 * npad + (long long)J_ * TB,
                          TB * 4, &full[s]);
        (void)I_;
    };
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) tc::mbar_init(&full[s], 1);
        tc::fence_barrier_init();
    }
    __syncthreads();
    int pI = I, pJ = J;   // producer's (I, J) of the next tile to issue
    if (tid == 0) {
        for (int k = 0; k < STAGES && k < cnt; ++k) {
            issue(k, pI, pJ);
            if (++pJ == T) pJ = ++pI;
        }
    }
    Rows<DIM> R;
    double st64 = 0.0;
    int curI = -1, Ifirst = I;
    const bool ragged = (n % TB) != 0;
    for (int k = 0; k < cnt; ++k) {
        const long long ig0 = (long long)I * TB, jg0 = (long long)J * TB;
        if (I != curI) {
            if (curI >= 0) flush_rows<DIM>(R, rowpart, c * kmax + (curI - Ifirst), tx, ty);
            curI = I;
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int k2 = 0; k2 < DIM; ++k2) {
                    R.nti[a][k2] = -__ldg(thp + k2 * npad + ig0 + ty * 8 + a);
                    R.C[a][k2] = f2(0.f, 0.f);
                }
        }
        const int s = k % STAGES;
        tc::mbar_wait(&full[s], (k / STAGES) & 1);
        const float* ys = reinterpret_cast<const float*>(smem_raw + s * STAGE_BYTES);
        const float* thj = ys + TILE;
        float2 tj[4][DIM], CJ[4][DIM];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int k2 = 0; k2 < DIM; ++k2) {
                tj[p][k2] = *reinterpret_cast<const float2*>(thj + k2 * TB + jcol(tx, p, 0));
                CJ[p][k2] = f2(0.f, 0.f);
            }
        float2 st2 = f2(0.f, 0.f), rsum = f2(0.f, 0.f);
        if (I == J || (ragged && J == T - 1))
            tile_pairs<DIM, true>(ys, R, tj, CJ, st2, rsum, tx, ty, ig0, jg0, n);
        else
            tile_pairs<DIM, false>(ys, R, tj, CJ, st2, rsum, tx, ty, ig0, jg0, n);
        st64 += (double)st2.x + (double)st2.y;
        if (!(rsum.x + rsum.y <= kSuspect)) careful<DIM>(ys, thp, npad, tx, ty, ig0, jg0, n, err);
        // column partials: lanes l and l ^ 16 hold the two ty of a warp
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int k2 = 0; k2 < DIM; ++k2) {
                CJ[p][k2].x += __shfl_xor_sync(0xffffffffu, CJ[p][k2].x, 16);
                CJ[p][k2].y += __shfl_xor_sync(0xffffffffu, CJ[p][k2].y, 16);
            }
        // red is double-buffered: the readers of this buffer (tile k - 2) are
        // behind the barrier of tile k - 1, so one barrier per tile suffices
        float* rb = red + (k & 1) * (kWarps * kMaxTriDim * TB);
        if (lane < 16) {
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int k2 = 0; k2 < DIM; ++k2)
                    *reinterpret_cast<float2*>(rb + (warp * DIM + k2) * TB + jcol(tx, p, 0)) =
                        CJ[p][k2];
        }
        __syncthreads();   // slot s consumed by every thread; rb complete
        if (tid == 0 && k + STAGES < cnt) {
            issue(k + STAGES, pI, pJ);
            if (++pJ == T) pJ = ++pI;
        }
        float* cp = colpart + (u0 + k) * (long long)(DIM * TB);
        for (int o = tid; o < DIM * TB; o += kThreads) {
            float sum = 0.f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) sum += rb[w * DIM * TB + o];
            cp[o] = -sum;
        }
        if (++J == T) J = ++I;
    }
    flush_rows<DIM>(R, rowpart, c * kmax + (curI - Ifirst), tx, ty);
    const double bs = block_sum(st64, sred);
    if (tid == 0) stpart[c] = bs;
}

// zero-padded theta copy [dim][npad] and S_k = sum_i theta_ki (fp64, fixed
// order) into the tail of red -- written by the rank holding tile 0 only, so
// the all-reduce of red over ranks yields S once
__global__ void __launch_bounds__(256)
mds_tri_stage(const float* __restrict__ theta, float* __restrict__ thp, int n, long long npad,
              int dim, double* __restrict__ part, unsigned int* counter, double* __restrict__ S,
              int owner) {
    __shared__ double sc[32];
    double acc[kMaxTriDim] = {0.0, 0.0, 0.0};
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npad;
         p += (long long)gridDim.x * blockDim.x) {
        for (int k = 0; k < dim; ++k) {
            const float v = p < n ? theta[(long long)k * n + p] : 0.f;
            thp[k * npad + p] = v;
            acc[k] += (double)v;
        }
    }
    for (int k = 0; k < dim; ++k) {
        const double b = block_sum(acc[k], sc);
        if (threadIdx.x == 0) part[blockIdx.x * kMaxTriDim + k] = b;
    }
    if (arrive_last(counter, gridDim.x)) {
        for (int k = 0; k < dim; ++k) {
            double t = 0.0;
            for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
                t += part[b * kMaxTriDim + k];
            t = block_sum(t, sc);
            if (threadIdx.x == 0) S[k] = owner ? t : 0.0;   // summed once across ranks
        }
    }
}

// red[p][.] = fixed-order sum of every partial of point p; red[n*DIM] = stress.
// One CTA per tile column P: 4 groups of 128 threads split the column tiles
// (I = g, g + 4, ...), group 0 adds the row partials, and the 4 group sums
// are combined in a fixed order (deterministic).
constexpr int kAccGroups = 4;
template <int DIM>
__global__ void __launch_bounds__(128 * kAccGroups)
mds_tri_accum(const float* __restrict__ colpart, const float* __restrict__ rowpart, int kmax,
              const double* __restrict__ stpart, int G, long long t0, long long ntl, int T, int n,
              double* __restrict__ red, unsigned int* counter) {
    __shared__ double part[kAccGroups][DIM][TB];
    __shared__ double sc[32];
    const int P = blockIdx.x, pl = threadIdx.x % TB, g = threadIdx.x / TB;
    double acc[DIM];
#pragma unroll
    for (int q = 0; q < DIM; ++q) acc[q] = 0.0;
    // tiles (I, P) of the local range: I in [Ilo, P]
    const long long base = tri_index(0, P, T);   // I = 0
#pragma unroll 4
    for (int I = g; I <= P; I += kAccGroups) {
        const long long u = tri_index(I, P, T) - t0;
        if (u < 0 || u >= ntl) continue;
        const float* cp = colpart + u * (DIM * TB) + pl;
#pragma unroll
        for (int q = 0; q < DIM; ++q) acc[q] += (double)__ldg(cp + q * TB);
    }
    (void)base;
    if (g == 0) {
        long long lo = tri_index(P, P, T) - t0, hi = tri_index(P, T - 1, T) - t0;
        if (lo < 0) lo = 0;
        if (hi > ntl - 1) hi = ntl - 1;
        if (lo <= hi) {
            const int c0 = cta_of(lo, ntl, G), c1 = cta_of(hi, ntl, G);
            for (int c = c0; c <= c1; ++c) {
                const int seg = P - row_of(t0 + cta_start(c, ntl, G), T);
                const float* rp = rowpart + ((long long)c * kmax + seg) * (DIM * TB) + pl;
#pragma unroll
                for (int q = 0; q < DIM; ++q) acc[q] += (double)rp[q * TB];
            }
        }
    }
#pragma unroll
    for (int q = 0; q < DIM; ++q) part[g][q][pl] = acc[q];
    __syncthreads();
    const int p = P * TB + threadIdx.x;
    if (threadIdx.x < TB && p < n) {
#pragma unroll
        for (int q = 0; q < DIM; ++q) {
            double t = part[0][q][threadIdx.x];
#pragma unroll
            for (int k = 1; k < kAccGroups; ++k) t += part[k][q][threadIdx.x];
            red[(long long)p * DIM + q] = t;
        }
    }
    if (arrive_last(counter, gridDim.x)) {
        const double tot = block_sum_array(stpart, G, sc);
        if (threadIdx.x == 0) red[(long long)n * DIM] = tot;
    }
}

template <int DIM>
__global__ void mds_tri_finish(const float* __restrict__ theta, float* __restrict__ out, int n,
                               const double* __restrict__ red, double* f_dev) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const double* S = red + (long long)n * DIM + 1;
    if (f_dev && p == 0) *f_dev = red[(long long)n * DIM];
    if (p >= n || out == nullptr) return;
    const double w = (double)(n - 1);
#pragma unroll
    for (int k = 0; k < DIM; ++k)
        out[(long long)k * n + p] =
            (float)(((double)theta[(long long)k * n + p] * (w - 1.0) + S[k] -
                     red[(long long)p * DIM + k]) /
                    (2.0 * w));
}

// pack (and optionally validate) the tiles of local range [t0, t1) whose tile
// row lies in the given block of full rows [row0, row0 + rows)
__global__ void mds_tri_pack_kernel(const float* __restrict__ Y, long long ldy, int n, int T,
                                    long long row0, long long rows, long long t0, long long t1,
                                    float* __restrict__ packed, int validate, int64_t* err) {
    const long long t = t0 + blockIdx.x;
    if (t >= t1) return;
    const int I = row_of(t, T);
    const int J = I + (int)(t - tri_index(I, I, T));
    const long long ig0 = (long long)I * TB, jg0 = (long long)J * TB;
    if (ig0 < row0 || ig0 >= row0 + rows) return;
    float* dst = packed + (long long)blockIdx.x * TILE;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
        const long long ig = ig0 + e / TB, jg = jg0 + e % TB;
        float v = 0.f;
        if (ig < n && jg < n && ig - row0 < rows) v = Y[(ig - row0) * ldy + jg];
        dst[e] = v;
        if (!validate || ig >= n || jg >= n || ig - row0 >= rows) continue;
        const long long idx = ig * n + jg;
        if (!isfinite(v)) flag_error(err, MMK_E_DOMAIN, err_at(2, idx));
        else if (v < 0.f) flag_error(err, MMK_E_DOMAIN, err_at(3, idx));
        if (ig == jg && v != 0.f) flag_error(err, MMK_E_DOMAIN, err_at(5, idx));
        if (jg >= row0 && jg < row0 + rows && ig != jg) {
            const float vt = Y[(jg - row0) * ldy + ig];
            if (!(vt == v) && isfinite(v)) flag_error(err, MMK_E_DOMAIN, err_at(4, idx));
        }
    }
}

struct TriPlan {
    int T, G, kmax;
    long long ntl;
};

TriPlan tri_plan(long long n, long long t0, long long t1) {
    TriPlan P;
    P.T = (int)((n + TB - 1) / TB);
    P.ntl = t1 - t0;
    P.G = (int)(P.ntl < kNumSMs ? P.ntl : kNumSMs);
    if (P.G < 1) P.G = 1;
    P.kmax = 1;
    for (long long c = 0; c < P.G; ++c) {
        const long long a = cta_start(c, P.ntl, P.G), b = cta_start(c + 1, P.ntl, P.G);
        if (b <= a) continue;
        const int k = row_of(t0 + b - 1, P.T) - row_of(t0 + a, P.T) + 1;
        if (k > P.kmax) P.kmax = k;
    }
    return P;
}

struct TriWs {
    unsigned int* counter;    // [0] accum, [1] stage
    double* stpart;
    double* spart;
    float* thp;
    float* colpart;
    float* rowpart;
    long long npad;
};

constexpr int kStageBlocks = 2 * kNumSMs;

size_t tri_layout(const TriPlan& P, int dim, void* base, TriWs* L) {
    size_t off = 256;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    const long long npad = (long long)P.T * TB;
    const size_t os = take(sizeof(double) * P.G);
    const size_t osp = take(sizeof(double) * kStageBlocks * kMaxTriDim);
    const size_t oth = take(sizeof(float) * (size_t)dim * npad);
    const size_t oc = take(sizeof(float) * (size_t)P.ntl * dim * TB);
    const size_t orow = take(sizeof(float) * (size_t)P.G * P.kmax * dim * TB);
    if (base && L) {
        char* b = reinterpret_cast<char*>(base);
        L->counter = reinterpret_cast<unsigned int*>(b);
        L->stpart = reinterpret_cast<double*>(b + os);
        L->spart = reinterpret_cast<double*>(b + osp);
        L->thp = reinterpret_cast<float*>(b + oth);
        L->colpart = reinterpret_cast<float*>(b + oc);
        L->rowpart = reinterpret_cast<float*>(b + orow);
        L->npad = npad;
    }
    return off;
}

constexpr uint32_t kTriSmem = STAGES * STAGE_BYTES + 2 * kWarps * kMaxTriDim * TB * 4;

int check_tri(long long n, long long dim, long long t0, long long t1) {
    const long long T = (n + TB - 1) / TB;
    if (n < 2 || n > (1LL << 30) || dim < 1 || dim > kMaxTriDim || t0 < 0 || t1 <= t0 ||
        t1 > T * (T + 1) / 2) {
        mmk_host::set_error("bad packed-triangle MDS shape: n=%lld dim=%lld tiles [%lld, %lld) "
                            "(dim <= %d)", n, dim, t0, t1, kMaxTriDim);
        return MMK_E_SHAPE;
    }
    return MMK_OK;
}

template <int DIM>
int tri_a(const float* Yp, long long t0, long long t1, const float* theta, int n, void* ws,
          double* red, int64_t* err, cudaStream_t st) {
    const TriPlan P = tri_plan(n, t0, t1);
    TriWs L;
    tri_layout(P, DIM, ws, &L);
    if (mmk_host::first_on_device(reinterpret_cast<const void*>(mds_tri_kernel<DIM>))) {
        cudaFuncSetAttribute(mds_tri_kernel<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kTriSmem);
    }
    MMK_LAUNCH("mds_tri_stage", st,
               (mds_tri_stage<<<kStageBlocks, 256, 0, st>>>(theta, L.thp, n, L.npad, DIM, L.spart,
                                                            L.counter + 1,
                                                            red + (long long)n * DIM + 1,
                                                            t0 == 0 ? 1 : 0)));
    MMK_LAUNCH("mds_tri", st,
               (mds_tri_kernel<DIM><<<P.G, kThreads, kTriSmem, st>>>(
                   Yp, t0, P.ntl, P.T, n, L.thp, L.npad, L.colpart, L.rowpart, P.kmax, L.stpart,
                   err)));
    MMK_CHECK_LAUNCH("mds_tri_kernel");
    MMK_LAUNCH("mds_tri_accum", st,
               (mds_tri_accum<DIM><<<P.T, 128 * kAccGroups, 0, st>>>(
                   L.colpart, L.rowpart, P.kmax, L.stpart, P.G, t0, P.ntl, P.T, n, red,
                   L.counter)));
    MMK_CHECK_LAUNCH("mds_tri_accum");
    return MMK_OK;
}

template <int DIM>
int tri_b(const float* theta, float* out, int n, const double* red, double* f_dev,
          cudaStream_t st) {
    MMK_LAUNCH("mds_tri_finish", st,
               (mds_tri_finish<DIM><<<ceil_div(n, 256), 256, 0, st>>>(theta, out, n, red, f_dev)));
    MMK_CHECK_LAUNCH("mds_tri_finish");
    return MMK_OK;
}

}  // namespace

extern "C" int64_t mmk_mds_tri_ntiles(int64_t n) {
    const int64_t T = (n + TB - 1) / TB;
    return T * (T + 1) / 2;
}

// [C (n dim) | stress | S (dim) | device-error flag]
extern "C" int64_t mmk_mds_tri_reduce_len(int64_t n, int64_t dim) { return n * dim + 1 + dim + 1; }

extern "C" int mmk_mds_tri_ws_bytes(int64_t n, int64_t dim, int64_t t0, int64_t t1, size_t* out) {
    int rc = check_tri(n, dim, t0, t1);
    if (rc) return rc;
    *out = tri_layout(tri_plan(n, t0, t1), (int)dim, nullptr, nullptr);
    return MMK_OK;
}

extern "C" int mmk_mds_tri_pack(const float* Y, int64_t ldy, int64_t n, int64_t row0, int64_t rows,
                                float* packed, int64_t t0, int64_t t1, int validate,
                                int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_mds_tri_pack");
    int rc = check_tri(n, 1, t0, t1);
    if (rc) return rc;
    if (row0 < 0 || row0 % TB || rows < 1 || row0 + rows > n || ldy < n) {
        mmk_host::set_error("pack rows [%lld, +%lld) must start on a 128-row boundary inside n=%lld",
                            (long long)row0, (long long)rows, (long long)n);
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int T = (int)((n + TB - 1) / TB);
    MMK_LAUNCH("mds_tri_pack", st,
               (mds_tri_pack_kernel<<<(unsigned)(t1 - t0), 256, 0, st>>>(
                   Y, ldy, (int)n, T, row0, rows, t0, t1, packed, validate, err_dev)));
    MMK_CHECK_LAUNCH("mds_tri_pack_kernel");
    return MMK_OK;
}

extern "C" int mmk_mds_tri_iter_a(const float* packed, int64_t t0, int64_t t1, const float* theta,
                                  int64_t dim, int64_t n, void* ws, size_t ws_bytes, double* red,
                                  int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_mds_tri_iter_a");
    int rc = check_tri(n, dim, t0, t1);
    if (rc) return rc;
    const size_t need = tri_layout(tri_plan(n, t0, t1), (int)dim, nullptr, nullptr);
    if (ws_bytes < need) {
        mmk_host::set_error("packed MDS workspace too small: %zu < %zu", ws_bytes, need);
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (dim) {
        case 1: rc = tri_a<1>(packed, t0, t1, theta, (int)n, ws, red, err_dev, st); break;
        case 2: rc = tri_a<2>(packed, t0, t1, theta, (int)n, ws, red, err_dev, st); break;
        default: rc = tri_a<3>(packed, t0, t1, theta, (int)n, ws, red, err_dev, st); break;
    }
    if (rc) return rc;
    mmk_host::err_flag(err_dev, red + mmk_mds_tri_reduce_len(n, dim) - 1, st);
    return MMK_OK;
}

extern "C" int mmk_mds_tri_iter_b(const float* theta, float* theta_out, int64_t dim, int64_t n,
                                  const double* red, double* f_dev, int64_t* err_dev,
                                  void* stream) {
    MMK_NVTX("mmk_mds_tri_iter_b");
    if (dim < 1 || dim > kMaxTriDim || n < 2) {
        mmk_host::set_error("bad packed-triangle MDS shape: n=%lld dim=%lld", (long long)n,
                            (long long)dim);
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    mmk_host::peer_err(red + mmk_mds_tri_reduce_len(n, dim) - 1, err_dev, st);
    switch (dim) {
        case 1: return tri_b<1>(theta, theta_out, (int)n, red, f_dev, st);
        case 2: return tri_b<2>(theta, theta_out, (int)n, red, f_dev, st);
        default: return tri_b<3>(theta, theta_out, (int)n, red, f_dev, st);
    }
}

extern "C" int mmk_mds_tri_iter(const float* packed, int64_t t0, int64_t t1, const float* theta,
                                float* theta_out, int64_t dim, int64_t n, void* ws,
                                size_t ws_bytes, double* red, double* f_dev, int64_t* err_dev,
                                void* stream) {
    MMK_NVTX("mmk_mds_tri_iter");
    mmk_host::NoFlag one_gpu;   // no collective between the phases
    int rc = mmk_mds_tri_iter_a(packed, t0, t1, theta, dim, n, ws, ws_bytes, red, err_dev, stream);
    if (rc) return rc;
    return mmk_mds_tri_iter_b(theta, theta_out, dim, n, red, f_dev, err_dev, stream);
}
