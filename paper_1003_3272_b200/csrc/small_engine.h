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

// Frobenius NNMF (nnmf.py:84-110, 143-159): r <= 16, small m x n.
// MMK_SMALL_ENGINE=0 in the environment disables the persistent engines.
bool nnmf_eligible(int dtype, long long m, long long n, long long r, long long ldx);
int nnmf_prepare(int dtype, const void* X, long long ldx, void* VA, void* WA, void* VB, void* WB,
                 long long m, long long n, int r, const mmk_stop_rule* rule, double* trace,
                 int64_t* tstamp, int64_t* ctl, int64_t* err, Launch* out);

}  // namespace mmk_small
