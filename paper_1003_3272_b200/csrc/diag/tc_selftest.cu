// tc_selftest.cu -- known-answer check of the tcgen05 building blocks the
// NNMF tensor-core kernels rely on (TMA 128B-swizzled tiles, K-major and
// MN-major UMMA descriptors, kind::tf32 MMA, TMEM loads).  One CTA computes
//   D1[128x64] = A[128x64] . B[64x64]^T     (A, B K-major; the V-step's Q)
//   D2[128x32] = A . B[:, 0:32]             (B MN-major;   the V-step residual)
//   D3[128x64] = X[32x128]^T . V[32x64]     (A, B MN-major; the W-step's P^T)
// in single-pass TF32; tests compare against fp64 products with a TF32
// tolerance.
#include "../mmk_common.cuh"
#include "../tc_common.cuh"

namespace {

constexpr uint32_t kA = 2 * 16384, kB = 2 * 8192, kX = 4 * 4096, kV = 2 * 4096, kB32 = 8192;

__global__ void __launch_bounds__(128)
tc_selftest_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                   const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mV,
                   const __grid_constant__ CUtensorMap mB32,
                   float* D1, float* D2, float* D3, int mode, int* diag) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = sA + kA;
    uint8_t* sX = sB + kB;
    uint8_t* sV = sX + kX;
    uint8_t* sB32 = sV + kV;
    __shared__ uint64_t bar_tma, bar_mma;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        tc::mbar_init(&bar_tma, 1);
        tc::mbar_init(&bar_mma, 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<256>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tm = tmem_base;
    if (tid == 0) {
        tc::mbar_expect_tx(&bar_tma, kA + kB + kX + kV + kB32);
        tc::tma_load_2d(sB32, &mB32, &bar_tma, 0, 0);
        for (int b = 0; b < 2; ++b) tc::tma_load_2d(sA + b * 16384, &mA, &bar_tma, b * 32, 0);
        for (int b = 0; b < 2; ++b) tc::tma_load_2d(sB + b * 8192, &mB, &bar_tma, b * 32, 0);
        for (int b = 0; b < 4; ++b) tc::tma_load_2d(sX + b * 4096, &mX, &bar_tma, b * 32, 0);
        for (int b = 0; b < 2; ++b) tc::tma_load_2d(sV + b * 4096, &mV, &bar_tma, b * 32, 0);
    }
    if (!tc::mbar_wait_bounded(&bar_tma, 0)) {
        if (tid == 0) atomicOr(diag, 1);
    }
    if (mode & 1) {  // dump the raw (swizzled) A tile, X tile and B (32B-atom) tile
        const float* f = reinterpret_cast<const float*>(sA);
        for (int i = tid; i < 128 * 64; i += 128) D1[i] = f[i];
        const float* fx = reinterpret_cast<const float*>(sX);
        for (int i = tid; i < 128 * 32; i += 128) D3[i] = fx[i];
        const float* fb = reinterpret_cast<const float*>(sB32);
        for (int i = tid; i < 64 * 32; i += 128) D3[128 * 32 + i] = fb[i];
    }
    if (tid == 0 && (mode & 14)) {
        tc::tc_fence_after();
        // D1: K = 64 as 2 swizzle-atom columns x 4 K-steps of 8
        for (int ks = 0; ks < 8 && (mode & 2); ++ks) {
            const int kb = ks >> 2, sub = ks & 3;
            uint64_t a = tc::sdesc_sw128(sA + kb * 16384 + sub * 32, 16, 1024);
            uint64_t b = tc::sdesc_sw128(sB + kb * 8192 + sub * 32, 16, 1024);
            tc::mma_tf32(tm + 0, a, b, tc::idesc_tf32(128, 64, 0, 0), ks > 0);
        }
        // D2: B = first 32 columns of B viewed MN-major (k = row of B)
        for (int ks = 0; ks < 8 && (mode & 4); ++ks) {
            const int kb = ks >> 2, sub = ks & 3;
            uint64_t a = tc::sdesc_sw128(sA + kb * 16384 + sub * 32, 16, 1024);
            uint64_t b = tc::sdesc_sw128_32b(sB32 + ks * 1024, 8192, 512);
            tc::mma_tf32(tm + 64, a, b, tc::idesc_tf32(128, 32, 0, 1), ks > 0);
        }
        // D3: A = X^T (MN-major, 4 groups of 32 columns 4 KB apart), B = V (MN-major)
        for (int ks = 0; ks < 4 && (mode & 8); ++ks) {
            uint64_t a = tc::sdesc_sw128_32b(sX + ks * 1024, 4096, 512);
            uint64_t b = tc::sdesc_sw128_32b(sV + ks * 1024, 4096, 512);
            tc::mma_tf32(tm + 128, a, b, tc::idesc_tf32(128, 64, 1, 1), ks > 0);
        }
        tc::mma_commit(&bar_mma);
    }
    if (mode & 14) {
        if (!tc::mbar_wait_bounded(&bar_mma, 0)) {
            if (tid == 0) atomicOr(diag, 2);
        }
    }
    tc::tc_fence_after();
    if (!(mode & 1)) {
        const int row = warp * 32 + lane;
        const uint32_t lane_addr = tm + ((uint32_t)(warp * 32) << 16);
        float v[32];
        for (int c = 0; c < 2; ++c) {
            tc::tmem_ld32(lane_addr + 0 + c * 32, v);
            for (int i = 0; i < 32; ++i) D1[row * 64 + c * 32 + i] = v[i];
        }
        tc::tmem_ld32(lane_addr + 64, v);
        for (int i = 0; i < 32; ++i) D2[row * 32 + i] = v[i];
        for (int c = 0; c < 2; ++c) {
            tc::tmem_ld32(lane_addr + 128 + c * 32, v);
            for (int i = 0; i < 32; ++i) D3[row * 64 + c * 32 + i] = v[i];
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<256>(tm);
}

}  // namespace


extern "C" int mmk_selftest_tc(const float* A, const float* B, const float* X, const float* V,
                               float* D1, float* D2, float* D3, int mode, int* diag,
                               void* stream) {
    CUtensorMap mA, mB, mX, mV, mB32;
    int rc;
    if ((rc = mmk_host::make_map_f32(&mA, A, 128, 64, 64, 128))) return rc;
    if ((rc = mmk_host::make_map_f32(&mB, B, 64, 64, 64, 64))) return rc;
    if ((rc = mmk_host::make_map_f32(&mX, X, 32, 128, 128, 32, 32))) return rc;
    if ((rc = mmk_host::make_map_f32(&mV, V, 32, 64, 64, 32, 32))) return rc;
    if ((rc = mmk_host::make_map_f32(&mB32, B, 64, 64, 64, 64, 32))) return rc;
    const size_t smem = 1024 + kA + kB + kX + kV + kB32;
    cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    tc_selftest_kernel<<<1, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(mA, mB, mX, mV, mB32,
                                                                                D1, D2, D3, mode,
                                                                                diag);
    MMK_CHECK_LAUNCH("tc_selftest_kernel");
    return MMK_OK;
}

// ---------------------------------------------------------------------------
// MMA issue-rate microbenchmark (tuning aid): one CTA, one thread issues
// `iters` back-to-back tcgen05.mma of one shape on zeroed operands, commits,
// waits; out[0] = cycles.  mode: 0 SS tf32 N128, 1 TS tf32 N128, 2 TS tf32
// N64, 3 SS tf32 N256, 4 SS f16 N128 K16, 5 SS tf32 N64, 6 TS f16 N256,
// 7 SS f16 N256.
namespace {
__global__ void __launch_bounds__(128) tc_mma_bench_kernel(int mode, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 64 * 1024 / 4; i += 128) reinterpret_cast<float*>(base)[i] = 0.f;
    tc::fence_async_smem();
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tm = tmem_base;
    if (tid == 0) {
        const uint64_t da = tc::sdesc_sw128(base, 16, 1024);
        const uint64_t db = tc::sdesc_sw128(base + 16384, 16, 1024);
        // f16: a fmt 0 (F16), b fmt 0, c F32
        const uint32_t id_f16_128 = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t id_f16_256 = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t acc = i ? 1u : 0u;
            switch (mode) {
                case 0: tc::mma_tf32(tm, da, db, tc::idesc_tf32(128, 128, 0, 0), acc); break;
                case 1: tc::mma_tf32_ts(tm, tm + 256, db, tc::idesc_tf32(128, 128, 0, 0), acc); break;
                case 2: tc::mma_tf32_ts(tm, tm + 256, db, tc::idesc_tf32(128, 64, 0, 0), acc); break;
                case 3: tc::mma_tf32(tm, da, db, tc::idesc_tf32(128, 256, 0, 0), acc); break;
                case 4: tc::mma_f16ss(tm, da, db, id_f16_128, acc); break;
                case 5: tc::mma_tf32(tm, da, db, tc::idesc_tf32(128, 64, 0, 0), acc); break;
                case 6: tc::mma_f16ts(tm, tm + 256, db, id_f16_256, acc); break;
                case 7: tc::mma_f16ss(tm, da, db, id_f16_256, acc); break;
                // independent accumulators (D rotates over 4 / 2 regions)
                case 8: tc::mma_tf32(tm + (i & 3) * 128, da, db, tc::idesc_tf32(128, 128, 0, 0), i >= 4); break;
                case 9: tc::mma_tf32_ts(tm + (i & 3) * 64, tm + 256, db, tc::idesc_tf32(128, 64, 0, 0), i >= 4); break;
                case 10: tc::mma_tf32(tm + (i & 1) * 128, da, db, tc::idesc_tf32(128, 128, 0, 0), i >= 2); break;
                case 11: tc::mma_tf32_ts(tm + (i & 1) * 128, tm + 256 + 64 * (i & 1), db, tc::idesc_tf32(128, 128, 0, 0), i >= 2); break;
                default: tc::mma_f16ss(tm + (i & 1) * 256, da, db, id_f16_256, i >= 2); break;
            }
        }
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 0);
        out[0] = clock64() - t0;
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tm);
}
}  // namespace

extern "C" int mmk_tc_mma_bench(int mode, int iters, long long* out, void* stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaFuncSetAttribute(tc_mma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    tc_mma_bench_kernel<<<1, 128, 70 * 1024, st>>>(mode, iters, out);
    MMK_CHECK_LAUNCH("tc_mma_bench_kernel");
    return MMK_OK;
}

// ---------------------------------------------------------------------------
// 2-CTA (cta_group::2) issue-rate microbenchmark: a cluster of two CTAs (one
// TPC), the leader issues `iters` back-to-back kind::f16 MMAs of M = 256
// (128 rows per SM) x N x K16, all SS from zeroed shared memory, then one
// multicast commit; cycles of the leader into out[0], a timeout flag into
// out[1] (bounded waits: a wrong encoding cannot hang the GPU).
namespace {
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
tc_mma2_bench_kernel(int ncols, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = cluster_rank();
    for (int i = tid; i < 64 * 1024 / 4; i += 128) reinterpret_cast<float*>(base)[i] = 0.f;
    tc::fence_async_smem();
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            tc::smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc::tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc::tc_fence_after();
    const uint32_t tm = tmem_base;
    if (rank == 0 && tid == 0) {
        const uint64_t da = tc::sdesc_sw128(base, 16, 1024);
        const uint64_t db = tc::sdesc_sw128(base + 32768, 16, 1024);
        // kind::f16: a/b F16, c F32; N >> 3 at bit 17, M >> 4 at bit 24 (M = 256)
        const int nc = ncols < 0 ? -ncols : ncols;
        const uint32_t idesc = (1u << 4) | ((uint32_t)(nc >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
        long long t0 = clock64();
        const bool ts = ncols < 0;
        for (int i = 0; i < iters; ++i) {
            if (ts)   // A from TMEM (columns 256..): the TS form the NNMF kernels use
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                    "r"(tm + 256), "l"(db), "r"(idesc), "r"(i ? 1u : 0u)
                    : "memory");
            else
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                    "l"(da), "l"(db), "r"(idesc), "r"(i ? 1u : 0u)
                    : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
            "[%0], %1;" ::"r"(tc::smem_u32(&bar)),
            "h"((unsigned short)3)
            : "memory");
        const bool ok = tc::mbar_wait_bounded(&bar, 0);
        out[0] = clock64() - t0;
        out[1] = ok ? 0 : 1;
    }
    if (rank == 1 && tid == 0) {
        if (!tc::mbar_wait_bounded(&bar, 0)) out[2] = 1;
    }
    tc::tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
}  // namespace

extern "C" int mmk_tc_mma2_bench(int ncols, int iters, long long* out, void* stream) {
    const int nc = ncols < 0 ? -ncols : ncols;   // negative: A from TMEM (TS form)
    if (nc < 16 || nc > 256 || (nc % 16)) {
        mmk_host::set_error("mma2 bench: N must be a multiple of 16 in [16, 256]");
        return MMK_E_SHAPE;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaFuncSetAttribute(tc_mma2_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         70 * 1024);
    tc_mma2_bench_kernel<<<2, 128, 70 * 1024, st>>>(ncols, iters, out);
    MMK_CHECK_LAUNCH("tc_mma2_bench_kernel");
    return MMK_OK;
}

// ---------------------------------------------------------------------------
// Cross-CTA hand-off latency in a CTA pair: `iters` round trips in which CTA 0
// arrives (release.cluster) on CTA 1's mbarrier and waits on its own, and
// CTA 1 answers in kind; out[0] = CTA 0 cycles per round trip.  A second
// phase measures a commit-multicast round trip: CTA 0 issues an empty
// tcgen05.commit.cta_group::2 multicast to both barriers and CTA 1 answers
// with a remote arrive; out[1] = cycles per round trip.
namespace {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32)
tc_pingpong_kernel(int iters, long long* out) {
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t rank = tc::cluster_rank();
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_barrier_init();
    }
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        tc::smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    __syncwarp();
    tc::cluster_sync();
    if (threadIdx.x == 0) {
        const uint32_t peer = tc::map_to_rank(&bar, rank ^ 1u);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (rank == 0) {
                tc::mbar_arrive_cluster(peer);
                if (!tc::mbar_wait_bounded(&bar, i & 1)) { out[2] = 1; break; }
            } else {
                if (!tc::mbar_wait_bounded(&bar, i & 1)) { out[3] = 1; break; }
                tc::mbar_arrive_cluster(peer);
            }
        }
        if (rank == 0) out[0] = (clock64() - t0) / iters;
    }
    __syncwarp();
    tc::cluster_sync();
    // phase 2: commit multicast (leader) -> both barriers; peer answers
    if (threadIdx.x == 0) {
        const uint32_t leader = tc::map_to_rank(&bar, 0);
        uint32_t ph = (uint32_t)iters;   // phases completed in phase 1 (both barriers)
        const int rounds = iters / 2 > 0 ? iters / 2 : 1;
        long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            if (rank == 0) {
                tc::mma_commit_pair(&bar);   // arrives on both CTAs' barriers
                if (!tc::mbar_wait_bounded(&bar, ph & 1)) { out[2] = 2; break; }
                ++ph;
                if (!tc::mbar_wait_bounded(&bar, ph & 1)) { out[2] = 3; break; }
                ++ph;
            } else {
                if (!tc::mbar_wait_bounded(&bar, ph & 1)) { out[3] = 2; break; }
                ++ph;
                tc::mbar_arrive_cluster(leader);
            }
        }
        if (rank == 0) out[1] = (clock64() - t0) / rounds;
    }
    __syncwarp();
    tc::cluster_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" ::"r"(tmem_base));
}
}  // namespace

extern "C" int mmk_tc_pingpong(int iters, long long* out, void* stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    tc_pingpong_kernel<<<2, 32, 0, st>>>(iters, out);
    MMK_CHECK_LAUNCH("tc_pingpong_kernel");
    return MMK_OK;
}
