/* mmk_diag.h -- libmmk_diag.so: tcgen05 self-test and tuning
 * microbenchmarks.  NOT part of the solver ABI (include/mmk.h); built next to
 * libmmk.so by paper_1003_3272_b200/build.py from csrc/diag/. */
#ifndef MMK_DIAG_H_
#define MMK_DIAG_H_

#ifdef __cplusplus
extern "C" {
#endif

/* Known-answer self-test of the tcgen05 building blocks (TMA 128B-swizzle
 * tiles, K-/MN-major UMMA descriptors, kind::tf32 MMA, TMEM loads):
 *   D1[128x64] = A[128x64] B[64x64]^T,  D2[128x32] = A B[:, :32],
 *   D3[128x64] = X[32x128]^T V[32x64]   (device fp32, row-major).
 * mode bits: 1 dump the raw swizzled A tile into D1, 2/4/8 run D1/D2/D3;
 * diag (device int) gets bit 1 if the TMA barrier timed out, 2 for MMA. */
int mmk_selftest_tc(const float *A, const float *B, const float *X, const float *V, float *D1,
                    float *D2, float *D3, int mode, int *diag, void *stream);

/* Tuning aid: cycles for `iters` back-to-back tcgen05.mma of one shape
 * (mode 0 SS tf32 N128, 1 TS tf32 N128, 2 TS tf32 N64, 3 SS tf32 N256,
 * 4 SS f16 N128, 5 SS tf32 N64, 6 TS f16 N256, 7 SS f16 N256; M = 128) into
 * out[0] (device int64). */
int mmk_tc_mma_bench(int mode, int iters, long long *out, void *stream);

/* Tuning aid: the same for cta_group::2 (a 2-CTA cluster, M = 256, kind::f16,
 * N = |ncols|, A from TMEM when ncols < 0): leader cycles into out[0],
 * timeout flags into out[1], out[2]. */
int mmk_tc_mma2_bench(int ncols, int iters, long long *out, void *stream);

/* Tuning aid: cross-CTA hand-off latency in a CTA pair: out[0] cycles per
 * remote-arrive round trip, out[1] per commit-multicast + remote-arrive round
 * trip, out[2..3] timeout flags. */
int mmk_tc_pingpong(int iters, long long *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MMK_DIAG_H_ */
