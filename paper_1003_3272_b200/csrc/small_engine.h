// small_engine.h -- host interface of the persistent small-problem engines.
//
// For the paper-shape problems one MM iteration is a few microseconds of GPU
// work spread over several dependent kernels, so a graph of per-phase kernels
// is launch- and drain-bound.  A persistent engine instead runs a whole batch
// of iterations inside ONE cooperative kernel: the phases of an iteration are
// separated by software grid barriers (mm_control.cuh), and the run_mm
// stopping rule is applied on the device after every iteration exactly as the
// graph engine's control kernel does (same ctl / trace / slot protocol, so
// mmk_engine_run and the Python driver are unchanged).
#pragma once
#include <cuda_runtime.h>

#include <functional>

#include "../../include/mmk.h"

namespace mmk_small {

struct Launch {
    std::function<int(cudaStream_t)> fn;   // one launch = one batch (or until stop)
    void* scratch = nullptr;               // cudaMalloc'd, freed by mmk_engine_destroy
};

// Frobenius NNMF (nnmf.py:84-110, 143-159) or, with poisson, the Poisson
// log fit (nnmf.py:178-265): r <= 16, small m x n.
// MMK_SMALL_ENGINE=0 in the environment disables the persistent engines.
// Scratch buffers of destroyed persistent engines are kept for reuse:
// cudaFree synchronises the device and costs milliseconds, which is most of
// a short run.  scratch_take returns a zeroed-header buffer of >= bytes.
void* scratch_take(size_t bytes, size_t zero_bytes);
void scratch_give(void* p);

bool nnmf_eligible(int dtype, long long m, long long n, long long r, long long ldx);
int nnmf_prepare(int dtype, const void* X, long long ldx, void* VA, void* WA, void* VB, void* WB,
                 long long m, long long n, int r, const mmk_stop_rule* rule, double* trace,
                 int64_t* tstamp, int64_t* ctl, int64_t* err, Launch* out, bool poisson = false);

// Penalized PET with the sparse projector (pet.py:363-417 on CSR + CSC):
// ratios and intensities staged in shared memory (d doubles + p values).
bool pet_eligible(int dtype, long long d, long long p);
int pet_prepare(int dtype, const int32_t* rptr, const int32_t* ridx, const void* rval,
                const int32_t* cptr, const int32_t* cidx, const void* cval, const void* y,
                void* lamA, void* lamB, long long d, long long p, const int32_t* nbr_ptr,
                const int32_t* nbr_idx, double mu, const mmk_stop_rule* rule, double* trace,
                int64_t* tstamp, int64_t* ctl, int64_t* err, Launch* out);

// MDS stress majorization, full rows (mds.py:114-144), n <= 8192, dim <= 10.
bool mds_eligible(int dtype, long long n, long long dim, bool weighted);
int mds_prepare(int dtype, const void* Y, const void* Wt, long long ldy, const double* wsum,
                void* thetaA, void* thetaB, long long dim, long long n,
                const mmk_stop_rule* rule, double* trace, int64_t* tstamp, int64_t* ctl,
                int64_t* err, Launch* out);

}  // namespace mmk_small
