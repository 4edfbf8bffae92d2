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

// Loop state of the stopping rule (the ctl fields it reads and advances).
struct MmState {
    long long it, bstart;
    double fprev, rel;
    bool has_rel;
};

// The stopping rule proper: non-finite, monotone slack
// monotone_tol * (1 + |f_prev|), relative change |f - f_prev| / (|f_prev| + 1)
// < epsilon, the max_iters cap -> kMmStop (reason in *reason); otherwise
// advances the state and, after half 1, pauses every rule.batch iterations
// (-> kMmPause) so the host can drain the trace.  Pure function of its
// inputs, so every CTA of a persistent kernel can evaluate it redundantly.
// err: err_class of the pass's error record -- an objective-class error (1)
// stops first, as the reference raises it while evaluating f; an update-only
// one (2) only when the run would go on to step from this state.
__device__ __forceinline__ int mm_step(MmState& st, int half, double f, int err,
                                       const mmk_stop_rule& rule, int* reason) {
    int why = 0;
    st.has_rel = false;
    if (err == 1) {
        why = MMK_STOP_DEVICE_ERROR;
    } else if (!isfinite(f)) {
        why = MMK_STOP_NONFINITE;
    } else if (st.it > 0) {
        const double fp = st.fprev;
        if (rule.check_monotone && rule.sign * (f - fp) < -rule.monotone_tol * (1.0 + fabs(fp))) {
            why = MMK_STOP_MONOTONE;
        } else {
            st.rel = fabs(f - fp) / (fabs(fp) + 1.0);
            st.has_rel = true;
            if (st.rel < rule.epsilon) why = MMK_STOP_CONVERGED;
        }
    }
    if (!why && st.it >= rule.max_iters) why = MMK_STOP_CAP;
    if (!why && err == 2) why = MMK_STOP_DEVICE_ERROR;
    *reason = why;
    if (why) return kMmStop;
    st.fprev = f;
    st.it += 1;
    if (half == 1 && st.it - st.bstart >= rule.batch) {
        st.bstart = st.it;
        return kMmPause;
    }
    return kMmContinue;
}

__device__ __forceinline__ MmState mm_load(const long long* ctl) {
    MmState st;
    st.it = ctl[MMK_CTL_IT];
    st.bstart = ctl[MMK_CTL_BATCH_START];
    st.fprev = ctl_f64(ctl[MMK_CTL_FPREV]);
    st.rel = 0.0;
    st.has_rel = false;
    return st;
}

// Records f of iteration st.it (trace + device timestamp) and writes the
// outcome of mm_step back to ctl: ctl[REASON] and ctl[SLOT] = half (the slot
// holding the returned state) on a stop.  `st` is the state BEFORE the step.
__device__ __forceinline__ void mm_record(long long* ctl, double* trace, long long* tstamp,
                                          const MmState& before, const MmState& after, int half,
                                          double f, int decision, int reason) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    const long long k = before.it - before.bstart;
    trace[k] = f;
    tstamp[k] = (long long)now;
    ctl[MMK_CTL_FCUR] = ctl_bits(f);
    if (after.has_rel) ctl[MMK_CTL_REL] = ctl_bits(after.rel);
    if (decision == kMmStop) {
        ctl[MMK_CTL_REASON] = reason;
        ctl[MMK_CTL_SLOT] = half;
        return;
    }
    ctl[MMK_CTL_FPREV] = ctl_bits(after.fprev);
    ctl[MMK_CTL_IT] = after.it;
    ctl[MMK_CTL_BATCH_START] = after.bstart;
}

// Single-thread form used by the graph engine's control kernel and the NNMF
// persistent kernel: state from ctl, step, record.
__device__ __forceinline__ int mm_control(int half, long long* ctl, double* trace,
                                          long long* tstamp, const long long* err,
                                          const mmk_stop_rule& rule, double f) {
    const MmState before = mm_load(ctl);
    MmState after = before;
    int reason = 0;
    const int d = mm_step(after, half, f, err_class(err), rule, &reason);
    mm_record(ctl, trace, tstamp, before, after, half, f, d, reason);
    // the next pass evaluates f at the iteration cap: nothing after its
    // objective is used (run_mm never steps from the final state)
    ctl[MMK_CTL_LAST] = (d != kMmStop && after.it >= rule.max_iters) ? 1 : 0;
    return d;
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
