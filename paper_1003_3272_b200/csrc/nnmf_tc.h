// nnmf_tc.h -- host interface of the tensor-core NNMF path (nnmf_tc.cu).
#pragma once

#include <cuda_runtime.h>

namespace mmk_tc {

// dtype / shape admit the tensor-core path (fp32, ranks 17..128 on rank tiles
// of 64 and 128, m and n multiples
// of 8, >= 128, the pre-split copy of X within its memory cap)
bool shape_ok(int dtype, long long m, long long n, long long r);
// ... and this X (row stride, alignment; MMK_NNMF_TC=0 disables the path)
bool eligible(int dtype, long long m, long long n, long long r, long long ldx, const void* X);
size_t ws_bytes(long long m, long long n, long long r);
// r = 64 / 128, or 17..127 on the rank-64 / rank-128 kernels with zero-padded V / W
int iter_a(const float* X, long long ldx, const float* V, const float* W, float* V_out,
           long long m, long long n, long long r, void* tcws, double* GW, double* red,
           cudaStream_t st);

// Per-X preparation (sum x^2 / scale exponent, the pre-split copy): iter_a
// launches it every iteration (a key check after the first); a device-loop
// engine runs it once before its first batch (prepare_x) and captures its
// loop with set_x_prepared(true), which leaves those launches out.
int prepare_x(const float* X, long long ldx, long long m, long long n, void* tcws,
              cudaStream_t st);
void set_x_prepared(bool on);
// while an engine captures: ctl[MMK_CTL_LAST] for the W-half kernels (nullptr
// otherwise); last_flag() is what the capture passes to them
void set_last_flag(const int64_t* p);
const long long* last_flag();
// [begin, end) of the pre-split copy of X in the tensor-core workspace
void presplit_span(long long m, long long n, size_t* begin, size_t* end);
// the NNMF workspace's tensor-core part for (dtype, m, n, r), or nullptr when
// the tensor-core path does not apply (nnmf.cu)
void* engine_tc_ws(int dtype, const void* X, long long ldx, long long m, long long n, long long r,
                   void* ws);

}  // namespace mmk_tc
