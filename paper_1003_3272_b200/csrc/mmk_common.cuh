// mmk_common.cuh -- shared device helpers for the MM iteration kernels.
//
// Conventions (see include/mmk.h):
//  * every launch goes on the caller's stream; no allocation in the hot loop
//  * reductions are deterministic: fixed-shape warp/block trees, per-block
//    partials in workspace, and a fixed-order final pass (no float atomics)
//  * data-dependent invariant violations are recorded in a device error
//    record {code, index} (first offending index via atomicMin) and mapped
//    to the reference's exception classes on the host after the per-iteration
//    scalar read
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include "../../include/mmk.h"

namespace mmk {

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;

// ---- error record ----------------------------------------------------------
// err[0] = status code (first writer wins), err[1] = smallest offending index
__device__ __forceinline__ void flag_error(int64_t* err, int code, long long index) {
    if (err == nullptr) return;
    unsigned long long* e = reinterpret_cast<unsigned long long*>(err);
    atomicCAS(e, 0ull, (unsigned long long)code);
    atomicMin(e + 1, (unsigned long long)index);
}

// index = site << 48 | offending index; sites distinguish checks that share a
// status code (e.g. PET zero-mean ray vs negative discriminant)
__device__ __forceinline__ long long err_at(int site, long long index) {
    return ((long long)site << 48) | index;
}
// Sites 16..31 (site + kUpdateSite) mark errors the reference raises only from
// the UPDATE (its step()): MDS coincident pairs, PET negative discriminant /
// non-positive intensities, the Poisson update's zero mean.  A fused pass
// evaluates f(state) and the update together, so such an error at a state the
// reference would not step from (converged, or the iteration cap) must not
// stop the run: the stopping rule checks them last (mm_step) and the host
// defers them to step() (_engine.DeviceMm).  Objective-class errors have the
// smaller sites, so atomicMin keeps them first.
constexpr int kUpdateSite = 16;
__device__ __forceinline__ long long err_at_update(int site, long long index) {
    return err_at(site + kUpdateSite, index);
}
__host__ __device__ __forceinline__ bool err_update_only(long long index) {
    const long long s = index >> 48;
    return s >= kUpdateSite && s < 2 * kUpdateSite;
}
// 0: no error, 1: objective-class error, 2: update-only error
__device__ __forceinline__ int err_class(const void* err) {
    const volatile long long* e = reinterpret_cast<const volatile long long*>(err);
    if (e[0] == 0) return 0;
    return err_update_only(e[1]) ? 2 : 1;
}

// ---- reductions ------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum, result valid in every thread.  `scratch` needs
// blockDim.x/32 entries.  Fixed tree => deterministic for a fixed blockDim.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    T t = (lane < nw) ? scratch[lane] : T(0);
    t = warp_sum(t);
    return t;
}

// "Last block finishes" protocol: each block publishes a partial, the last
// block to arrive (device-scope counter) sums all partials in index order and
// re-arms the counter for the next launch.  Returns true in the last block.
__device__ __forceinline__ bool arrive_last(unsigned int* counter, unsigned int nblocks) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int prev = atomicAdd(counter, 1u);
        last = (prev == nblocks - 1);
        if (last) *counter = 0u;   // re-arm
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// Deterministic sum of `n` doubles by one block (fixed striding + tree).
__device__ __forceinline__ double block_sum_array(const double* a, long long n, double* scratch) {
    double s = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) s += a[i];
    return block_sum(s, scratch);
}

// ---- dtype traits ----------------------------------------------------------
template <typename T> struct num;
// Epilogues run in fp64 for both storage types, so the NNMF denominator guard
// keeps the reference's 1e-300 (nnmf.py:32).  The PET intensity floor
// (pet.py:36) must survive the store: 1e-300 flushes to 0 in fp32, so fp32
// storage floors at the smallest normal float instead.
template <> struct num<float> {
    static __device__ __forceinline__ double floor() { return 1.1754943508222875e-38; }
};
template <> struct num<double> {
    static __device__ __forceinline__ double floor() { return 1e-300; }
};
constexpr double kDenomGuard = 1e-300;

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace mmk

// host-side error plumbing shared by the ABI translation units
namespace mmk_host {
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
bool prof_on();
// 2-D fp32 row-major TMA map: box = 32 columns (128 B) x box_rows, 128B swizzle
int make_map_f32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                 uint64_t row_stride_elems, uint32_t box_rows, int swizzle = 128);
// 2-D fp16 row-major TMA map: box = 64 columns (128 B) x box_rows, 128B swizzle
int make_map_f16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                 uint64_t row_stride_elems, uint32_t box_rows);
void prof_start(const char* name, cudaStream_t s);
void prof_stop(cudaStream_t s);
// true the first time `key` (e.g. a kernel's address) is seen on the current
// device -- for once-per-device kernel attributes (thread-safe)
bool first_on_device(const void* key);
// Device errors of sharded runs (one collective per iteration):
// phase A writes 1.0 into the last slot of its all-reduce payload when this
// rank's error record is set (err_flag); phase B, after the all-reduce, marks
// a clean rank whose summed flag is > 0 with MMK_E_PEER (peer_err), so every
// rank stops at the same iteration.  The host then recovers the first
// offender with one (rare, slow-path) reduction of the records.
void err_flag(const int64_t* err, double* flag, cudaStream_t st);
void peer_err(const double* flag, int64_t* err, cudaStream_t st);
// Single-GPU iterations (phases A and B back to back, no collective between
// them) skip both launches: a NoFlag scope around them turns them off.
struct NoFlag {
    explicit NoFlag(bool active = true);
    ~NoFlag();
    bool prev;
};
}  // namespace mmk_host

namespace mmk_host {
// NVTX range over a C-ABI entry point (named ranges on an Nsight Systems
// timeline; a pointer check when no tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace mmk_host
#define MMK_NVTX(name) const mmk_host::NvtxRange _mmk_nvtx_range(name)

// Bracket one kernel launch for the opt-in profiler (mmk_prof_enable), in an
// NVTX range named after the kernel (the launch call on the host timeline;
// launches replayed from a CUDA graph do not pass through here).
#define MMK_LAUNCH(name, st, ...)                                           \
    do {                                                                    \
        const mmk_host::NvtxRange _nvtx(name);                              \
        const bool _p = mmk_host::prof_on();                                \
        if (_p) mmk_host::prof_start(name, st);                             \
        __VA_ARGS__;                                                        \
        if (_p) mmk_host::prof_stop(st);                                    \
    } while (0)

#define MMK_CHECK_LAUNCH(what)                                              \
    do {                                                                    \
        cudaError_t _e = cudaGetLastError();                                \
        if (_e != cudaSuccess) return mmk_host::cuda_status(_e, what);      \
    } while (0)
