// nnmf_tc.h -- host interface of the tensor-core NNMF path (nnmf_tc.cu).
#pragma once

#include <cuda_runtime.h>

namespace mmk_tc {

bool eligible(int dtype, long long m, long long n, long long r, long long ldx, const void* X);
size_t ws_bytes(long long m, long long n);
int iter_a(const float* X, long long ldx, const float* V, const float* W, float* V_out,
           long long m, long long n, void* tcws, double* GW, double* red,
           cudaStream_t st);

}  // namespace mmk_tc
