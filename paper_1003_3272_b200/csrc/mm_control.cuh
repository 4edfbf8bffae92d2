// mm_control.cuh -- the run_mm stopping rule (driver.py:101-149) applied on the
// device after each iteration, shared by the graph engine's control kernel
// (engine.cu) and the persistent small-problem kernels (nnmf_small.cu), and
// the software grid barrier those persistent kernels use.
//
// Barrier design note: a single arrival counter costs ~30 cycles per CTA of
// serialised same-address L2 atomics (~4.5k cycles at 148 CTAs); per-CTA
// flag slots polled by one warp per CTA have no serialisation, so a barrier
// costs about two L2 round trips after the last arrival.
#pragma once
#include "mmk_common.cuh"

namespace mmk {

enum { kMmContinue = 0, kMmStop = 1, kMmPause = 2 };

__device__ __forceinline__ double ctl_f64(long long b) { return __longlong_as_double(b); }
__device__ __forceinline__ long long ctl_bits(double d) { return __double_as_longlong(d); }

// Records f of iteration ctl[IT] (trace + device timestamp) and decides:
// non-finite, monotone slack monotone_tol * (1 + |f_prev|), relative change
// |f - f_prev| / (|f_prev| + 1) < epsilon, the max_iters cap -> kMmStop with
// ctl[REASON] and ctl[SLOT] = half (the slot holding the returned state);
// otherwise advances ctl[IT]; after half 1 pauses every rule.batch iterations
// (-> kMmPause) so the host can drain the trace.  Single thread.
__device__ __forceinline__ int mm_control(int half, long long* ctl, double* trace,
                                          long long* tstamp, const long long* err,
                                          const mmk_stop_rule& rule, double f) {
    const long long it = ctl[MMK_CTL_IT];
    const long long k = it - ctl[MMK_CTL_BATCH_START];
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    trace[k] = f;
    tstamp[k] = (long long)now;
    int reason = 0;
    if (*(volatile const long long*)err != 0) {
        reason = MMK_STOP_DEVICE_ERROR;
    } else if (!isfinite(f)) {
        reason = MMK_STOP_NONFINITE;
    } else if (it > 0) {
        const double fp = ctl_f64(ctl[MMK_CTL_FPREV]);
        if (rule.check_monotone && rule.sign * (f - fp) < -rule.monotone_tol * (1.0 + fabs(fp))) {
            reason = MMK_STOP_MONOTONE;
        } else {
            const double rel = fabs(f - fp) / (fabs(fp) + 1.0);
            ctl[MMK_CTL_REL] = ctl_bits(rel);
            if (rel < rule.epsilon) reason = MMK_STOP_CONVERGED;
        }
    }
    if (!reason && it >= rule.max_iters) reason = MMK_STOP_CAP;
    if (reason) {
        ctl[MMK_CTL_REASON] = reason;
        ctl[MMK_CTL_SLOT] = half;
        return kMmStop;
    }
    ctl[MMK_CTL_FPREV] = ctl_bits(f);
    ctl[MMK_CTL_IT] = it + 1;
    if (half == 1 && it + 1 - ctl[MMK_CTL_BATCH_START] >= rule.batch) {
        ctl[MMK_CTL_BATCH_START] = it + 1;
        return kMmPause;
    }
    return kMmContinue;
}

// Flag barrier: CTA b publishes `epoch` in its own 128-byte slot
// flags[32 b] (no atomics, no serialisation), then warp 0 of every CTA polls
// all slots until each holds an epoch >= its own.  Epochs only grow (the
// caller derives them from a per-launch sequence number), so slots never
// need resetting.
__device__ __forceinline__ void grid_sync_flags(unsigned int* flags, unsigned int epoch) {
    __syncthreads();
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
            __threadfence();
            *(volatile unsigned int*)(flags + 32 * blockIdx.x) = epoch;
        }
        for (;;) {
            bool ok = true;
            for (unsigned int b = threadIdx.x; b < gridDim.x; b += 32)
                ok &= (int)(*(volatile unsigned int*)(flags + 32 * b) - epoch) >= 0;
            if (__all_sync(0xffffffffu, ok)) break;
            __nanosleep(16);
        }
        __threadfence();
    }
    __syncthreads();
}

}  // namespace mmk
