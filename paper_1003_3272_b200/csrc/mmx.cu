// mmx.cu -- device side of the MMX1 matrix loader (reference io.py:90-106:
// "MMX1" magic, two little-endian u64 dims, row-major f8 payload).  The host
// streams the payload through pinned buffers; this kernel narrows each
// landed fp64 chunk to the fp32 storage of a single-precision run with
// round-to-nearest-even, i.e. exactly numpy's astype(float32).
#include "mmk_common.cuh"

namespace {

__global__ void __launch_bounds__(256)
f64_to_f32_kernel(const double* __restrict__ src, float* __restrict__ dst, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long pairs = n / 2;
    const double2* s2 = reinterpret_cast<const double2*>(src);
    float2* d2 = reinterpret_cast<float2*>(dst);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < pairs; t += stride) {
        const double2 v = s2[t];
        d2[t] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) dst[n - 1] = __double2float_rn(src[n - 1]);
}

}  // namespace

extern "C" int mmk_f64_to_f32(const double* src, float* dst, int64_t n, void* stream) {
    MMK_NVTX("mmk_f64_to_f32");
    if (n < 0 || ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)) {
        mmk_host::set_error("f64->f32: n=%lld, buffers must be 16-byte aligned", (long long)n);
        return MMK_E_SHAPE;
    }
    if (n == 0) return MMK_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const long long blocks = mmk::ceil_div((n + 1) / 2, 256);
    const int grid = (int)(blocks < 8 * mmk::kNumSMs ? blocks : 8 * mmk::kNumSMs);
    MMK_LAUNCH("mmx_f64_to_f32", st, (f64_to_f32_kernel<<<grid, 256, 0, st>>>(src, dst, n)));
    MMK_CHECK_LAUNCH("f64_to_f32_kernel");
    return MMK_OK;
}
