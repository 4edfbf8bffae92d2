// nnmf_tile.h -- host interface of the register-blocked NNMF kernels
// (nnmf_tile.cu): ranks 17..128, fp64 at any shape and the fp32 shapes the
// tensor-core path does not take.
#pragma once

#include <cuda_runtime.h>

namespace mmk_tile {

bool applies(long long r);
long long vstep_blocks(long long m);   // CTAs (= partial slots) of vstep
// the fused V step: flags as nnmf.cu VSTEP_UPDATE / VSTEP_RESID / VSTEP_GRAD
template <typename T>
void vstep(const T* X, long long ldx, const T* V, const T* W, const double* GW, T* Vout,
           long long m, long long n, int r, int flags, double* respart, unsigned int* counter,
           double* res_out, cudaStream_t st);
// P = V^T X split over S row ranges -> out[S][r][n] (S = 1: the final P)
template <typename T>
int wpart_splits(long long m, long long n, int max_splits);
// fp64 (DMMA) Frobenius W part: S chosen by wave efficiency over the
// resident CTA slots plus the partial traffic, S <= max_splits
int wpart_splits_dmma(long long m, long long n, int r, int max_splits);
constexpr int kDmmaMaxSplits = 16;
template <typename T>
void wpart(const T* X, long long ldx, const T* V, long long m, long long n, int r, int S,
           double* out, cudaStream_t st);

// Poisson loss (ranks 17..128): the fused V step (objective x ln b - b, ratio
// x / b, v' = v sqrt(q / wsum)) and P = V'^T (X / (V' W)) over S row splits
template <typename T>
void pois_vstep(const T* X, long long ldx, const T* V, const T* W, const double* wsum, T* Vout,
                long long m, long long n, int r, double* fpart, unsigned int* counter,
                double* f_out, int64_t* err, cudaStream_t st);
template <typename T>
void pois_wpart(const T* X, long long ldx, const T* V, const T* W, long long m, long long n,
                int r, int S, double* out, int64_t* err, cudaStream_t st);

}  // namespace mmk_tile
