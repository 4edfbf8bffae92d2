// mds_votes.cu -- roll-call votes -> packed-triangle dissimilarities on the
// tensor cores (reference votes_to_dissimilarity,
// mds.py:260-283).
//
// For a q x m vote matrix V (entries 1 / -1 / 0) with presence P = (V != 0),
// shared S = P P^T counts the roll calls two voters both attended and
// N = V V^T = agreements - disagreements on them, so the dissimilarity is
// D = (S - N) / (2 S) off the diagonal (0 on it).  Both products are exact in
// fp16 x fp16 -> fp32 (small integers, sums < 2^24).  One MMA stream gives
// both: with A_i = [p_i | v_i] and B rows [p_j | -v_j] (-> S - N) stacked on
// [p_j | 0] (-> S) along N, a kind::f16 M128 x N256 MMA over K = 2m fills the
// two halves of a 256-column TMEM accumulator.  The epilogue writes D
// straight into the packed upper-triangle tile layout of mds_tri.cu (tiles
// (I <= J) of 128 x 128, 64 KB each), so an n x n matrix never exists: the
// q = 65536 ingestion makes 8.6 GB of packed fp32 tiles from a 90 MB vote
// matrix.
//
//   mds_votes_prep  votes (fp32/fp64) -> A [q_pad][2 m_pad] and
//                   B [2 q_pad][2 m_pad] fp16 (blocks of 128 [p|-v] rows then
//                   128 [p|0] rows); validates the entries (DomainError).
//   mds_votes_tri   persistent, one CTA per SM: warp 0 TMA (A tile 128 x 64
//                   and B tile 256 x 64 per K chunk, 4-stage ring), warp 1
//                   one thread issues 4 SS MMAs per chunk into one of two
//                   TMEM accumulators, warps 2-5 epilogue (TMEM -> D ->
//                   packed tile, shared-no-roll-call check).
#include <cuda_fp16.h>

#include "mmk_common.cuh"
#include "tc_common.cuh"

namespace {

using namespace mmk;

constexpr int TB = 128;                 // tile side (points), = mds_tri.cu
constexpr int KC = 64;                  // K per stage (fp16: one 128-byte row)
constexpr uint32_t SA = TB * KC * 2;    // 16 KB
constexpr uint32_t SB = 2 * TB * KC * 2;   // 32 KB
constexpr int NST = 4;
constexpr uint32_t SMEM = NST * (SA + SB) + 1024;
constexpr int kThreads = 32 * 6;        // TMA, MMA, 4 epilogue warps
constexpr int NACC = 2;                 // TMEM accumulators (256 columns each)

__host__ __device__ inline long long tri_index(long long I, long long J, long long T) {
    return I * T - I * (I - 1) / 2 + (J - I);
}
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

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// A[i] = [p_i | v_i], B[block J] = 128 rows [p_j | -v_j] then 128 rows [p_j | 0]
template <typename T>
__global__ void mds_votes_prep_kernel(const T* __restrict__ votes, long long q, long long m,
                                      long long qpad, long long mpad, __half* __restrict__ A,
                                      __half* __restrict__ B, int64_t* err) {
    const long long K2 = 2 * mpad;
    const long long total = qpad * mpad;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / mpad, k = e % mpad;
        float v = 0.f;
        if (i < q && k < m) {
            const T x = votes[i * m + k];
            if (!(x == T(1) || x == T(-1) || x == T(0)))
                flag_error(err, MMK_E_DOMAIN, err_at(6, i * m + k));
            else
                v = (float)x;
        }
        const float p = v != 0.f ? 1.f : 0.f;
        A[i * K2 + k] = __float2half_rn(p);
        A[i * K2 + mpad + k] = __float2half_rn(v);
        const long long blk = i / TB, r = i % TB;
        __half* b1 = B + (blk * 2 * TB + r) * K2;
        __half* b2 = B + (blk * 2 * TB + TB + r) * K2;
        b1[k] = __float2half_rn(p);
        b1[mpad + k] = __float2half_rn(-v);
        b2[k] = __float2half_rn(p);
        b2[mpad + k] = __float2half_rn(0.f);
    }
}

struct Bars {
    uint64_t full[NST], empty[NST], dfull[NACC], dempty[NACC];
};

__global__ void __launch_bounds__(kThreads, 1)
mds_votes_tri_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                     long long q, long long K2, long long t0, long long ntl, int T,
                     float* __restrict__ packed, int64_t* err) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ Bars B;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long G = gridDim.x, c = blockIdx.x;
    const long long u0 = c * ntl / G, u1 = (c + 1) * ntl / G;
    const int cnt = (int)(u1 - u0);
    const int nk = (int)(K2 / KC);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            tc::mbar_init(&B.full[s], 1);
            tc::mbar_init(&B.empty[s], 1);
        }
        for (int a = 0; a < NACC; ++a) {
            tc::mbar_init(&B.dfull[a], 1);
            tc::mbar_init(&B.dempty[a], 128);
        }
        tc::fence_barrier_init();
        tc::tma_prefetch(&mA);
        tc::tma_prefetch(&mB);
    }
    if (warp == 1) tc::tmem_alloc<512>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    auto tile_ij = [&](int k, int& I, int& J) {
        const long long t = t0 + u0 + k;
        I = row_of(t, T);
        J = I + (int)(t - tri_index(I, I, T));
    };
    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int k = 0; k < cnt; ++k) {
                int I, J;
                tile_ij(k, I, J);
                for (int kc = 0; kc < nk; ++kc, ++it) {
                    const int s = it % NST;
                    tc::mbar_wait(&B.empty[s], ((it / NST) & 1) ^ 1);
                    tc::mbar_expect_tx(&B.full[s], SA + SB);
                    uint8_t* dst = base + s * (SA + SB);
                    tc::tma_load_2d(dst, &mA, &B.full[s], kc * KC, I * TB);
                    tc::tma_load_2d(dst + SA, &mB, &B.full[s], kc * KC, J * 2 * TB);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id = idesc_f16(TB, 2 * TB);
            int it = 0;
            for (int k = 0; k < cnt; ++k) {
                const int a = k % NACC;
                if (k >= NACC) tc::mbar_wait(&B.dempty[a], ((k / NACC) - 1) & 1);
                tc::tc_fence_after();
                const uint32_t d = tmem + a * 2 * TB;
                for (int kc = 0; kc < nk; ++kc, ++it) {
                    const int s = it % NST;
                    tc::mbar_wait(&B.full[s], (it / NST) & 1);
                    tc::tc_fence_after();
                    const uint8_t* st = base + s * (SA + SB);
                    const uint64_t da = tc::sdesc_sw128(st, 16, 1024);
                    const uint64_t db = tc::sdesc_sw128(st + SA, 16, 1024);
#pragma unroll
                    for (int ks = 0; ks < KC / 16; ++ks)
                        tc::mma_f16ss(d, da + ks * 2, db + ks * 2, id, (kc | ks) ? 1u : 0u);
                    tc::mma_commit(&B.empty[s]);
                }
                tc::mma_commit(&B.dfull[a]);
            }
        }
    } else {
        const int quarter = warp & 3;   // warps 2..5 -> quarters 2, 3, 0, 1
        for (int k = 0; k < cnt; ++k) {
            int I, J;
            tile_ij(k, I, J);
            const int a = k % NACC;
            tc::mbar_wait(&B.dfull[a], (k / NACC) & 1);
            tc::tc_fence_after();
            const long long il = quarter * 32 + lane;
            const long long i = (long long)I * TB + il;
            float* row = packed + (u0 + k) * (long long)(TB * TB) + il * TB;
            const uint32_t ta = tmem + a * 2 * TB + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
            for (int h = 0; h < TB / 32; ++h) {
                float sn[32], sh[32];
                tc::tmem_ld32(ta + h * 32, sn);
                tc::tmem_ld32(ta + TB + h * 32, sh);
                float out[32];
#pragma unroll
                for (int c2 = 0; c2 < 32; ++c2) {
                    const long long j = (long long)J * TB + h * 32 + c2;
                    float dv = 0.f;
                    if (i < q && j < q && i != j) {
                        if (sh[c2] == 0.f) {
                            const long long lo = i < j ? i : j, hi = i < j ? j : i;
                            flag_error(err, MMK_E_DOMAIN, err_at(7, lo * q + hi));
                        } else {
                            // exact integers in fp32; the reference divides in fp64
                            dv = (float)(((double)sn[c2]) / (2.0 * (double)sh[c2]));
                        }
                    }
                    out[c2] = dv;
                }
                float4* o = reinterpret_cast<float4*>(row + h * 32);
#pragma unroll
                for (int c4 = 0; c4 < 8; ++c4)
                    o[c4] = make_float4(out[4 * c4], out[4 * c4 + 1], out[4 * c4 + 2],
                                        out[4 * c4 + 3]);
            }
            tc::tc_fence_before();
            tc::mbar_arrive(&B.dempty[a]);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free<512>(tmem);
}

}  // namespace

extern "C" int mmk_mds_votes_bytes(int64_t q, int64_t m, size_t* out) {
    const long long qpad = (q + TB - 1) / TB * TB, mpad = (m + 31) / 32 * 32;
    *out = (size_t)(3 * qpad) * (size_t)(2 * mpad) * 2;   // A + B fp16
    return MMK_OK;
}

extern "C" int mmk_mds_votes_tri(int dtype, const void* votes, int64_t q, int64_t m,
                                 float* packed, int64_t t0, int64_t t1, void* ws,
                                 size_t ws_bytes, int64_t* err_dev, void* stream) {
    MMK_NVTX("mmk_mds_votes_tri");
    const long long T = (q + TB - 1) / TB;
    if (q < 2 || m < 1 || t0 < 0 || t1 <= t0 || t1 > T * (T + 1) / 2 || (m + 31) / 32 * 32 * 2 >= (1LL << 20)) {
        mmk_host::set_error("bad vote matrix %lld x %lld or tile range [%lld, %lld)",
                            (long long)q, (long long)m, (long long)t0, (long long)t1);
        return MMK_E_SHAPE;
    }
    size_t need = 0;
    mmk_mds_votes_bytes(q, m, &need);
    if (ws_bytes < need) {
        mmk_host::set_error("votes workspace too small: %zu < %zu", ws_bytes, need);
        return MMK_E_SHAPE;
    }
    const long long qpad = T * TB, mpad = (m + 31) / 32 * 32, K2 = 2 * mpad;
    __half* A = reinterpret_cast<__half*>(ws);
    __half* Bm = A + qpad * K2;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int grid = 4 * kNumSMs;
    if (dtype == MMK_F32)
        MMK_LAUNCH("mds_votes_prep", st,
                   (mds_votes_prep_kernel<float><<<grid, 256, 0, st>>>(
                       (const float*)votes, q, m, qpad, mpad, A, Bm, err_dev)));
    else
        MMK_LAUNCH("mds_votes_prep", st,
                   (mds_votes_prep_kernel<double><<<grid, 256, 0, st>>>(
                       (const double*)votes, q, m, qpad, mpad, A, Bm, err_dev)));
    MMK_CHECK_LAUNCH("mds_votes_prep_kernel");
    CUtensorMap mA, mB;
    int rc;
    if ((rc = mmk_host::make_map_f16(&mA, A, qpad, K2, K2, TB))) return rc;
    if ((rc = mmk_host::make_map_f16(&mB, Bm, 2 * qpad, K2, K2, 2 * TB))) return rc;
    if (mmk_host::first_on_device(reinterpret_cast<const void*>(mds_votes_tri_kernel))) {
        cudaFuncSetAttribute(mds_votes_tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM);
    }
    const long long ntl = t1 - t0;
    const int G = (int)(ntl < kNumSMs ? ntl : kNumSMs);
    MMK_LAUNCH("mds_votes_tri", st,
               (mds_votes_tri_kernel<<<G, kThreads, SMEM, st>>>(mA, mB, q, K2, t0, ntl, (int)T,
                                                                 packed, err_dev)));
    MMK_CHECK_LAUNCH("mds_votes_tri_kernel");
    return MMK_OK;
}
