/*
 * mmk.h -- C ABI of libmmk.so, the sm_100a MM-iteration kernels.
 *
 * The reference package (mmkit 0.1.0, /root/reference/pkg/src/mmkit) has no
 * FFI: its "native" boundary is the numba-compiled kernel layer called from
 * the solver modules (kernels.py:92-310, pet.py:204-210).  This header is the
 * drop-in replacement for that boundary; the Python solver modules in
 * paper_1003_3272_b200/ bind it with ctypes.  Each entry
 * point names the reference operation(s) it replaces.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller (PyTorch
 *    tensors).  Row-major, C-contiguous unless a leading dimension is given.
 *  - `dtype` selects the storage/compute precision of the state arrays:
 *    MMK_F32 or MMK_F64.  Objectives, Gram matrices and cross-block
 *    reductions are always accumulated in fp64.
 *  - `ws` is a caller-allocated workspace of at least *_ws_bytes() bytes,
 *    zero-initialised ONCE at allocation (it carries re-armed counters).
 *  - `red` is the caller-allocated fp64 "reduction buffer" (*_reduce_len()
 *    doubles).  Phase A writes this rank's partial sums into it; a
 *    multi-GPU caller all-reduces it (NCCL, sum) before phase B.  The fused
 *    single-GPU entry points run A and B back to back.
 *  - `f_dev` receives the fp64 objective at the INPUT state; `err_dev` is a
 *    two-int64 device record {status code, site << 48 | first offending index}
 *    that the
 *    kernels set on data-dependent invariant violations (never cleared by the
 *    library; the caller zeroes it).  Launch/shape problems are returned
 *    synchronously as the function's status.
 *  - Every launch is enqueued on `stream` (a cudaStream_t); no call
 *    synchronises the host, allocates, or keeps global mutable state except
 *    the thread-local error string.
 */
#ifndef MMK_H_
#define MMK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMK_ABI_VERSION 1

/* status codes -> paper_1003_3272_b200.errors (errors.py:10-48 taxonomy) */
enum {
    MMK_OK = 0,
    MMK_E_SHAPE = 1,     /* ShapeError */
    MMK_E_DOMAIN = 2,    /* DomainError */
    MMK_E_NUMERICS = 3,  /* NumericsError */
    MMK_E_NONFINITE = 4, /* NonFiniteError */
    MMK_E_CUDA = 5,      /* DeviceError (launch / runtime failure) */
    MMK_E_PEER = 6       /* error-record code only: another rank of a sharded run
                            flagged a device error (its record names it) */
};

enum { MMK_F32 = 0, MMK_F64 = 1 };

int mmk_abi_version(void);
const char *mmk_last_error(void);

/* Opt-in launch profiler (bench.py): when enabled, every kernel launch is
 * bracketed by CUDA events on its stream; mmk_prof_report() synchronises
 * them and writes "name\tlaunches\ttotal_ms\n" lines (returns the length).
 * Launches recorded into a CUDA graph are not profiled. */
int mmk_prof_enable(int on);
int mmk_prof_report(char *buf, size_t len);

/* ------------------------------------------------------------------------
 * NNMF, Frobenius loss.  X is m x n (leading dim ldx), V m x r, W r x n.
 * Replaces nnmf_objective / nnmf_update_v / nnmf_update_w (nnmf.py:75-110)
 * and their matmul/elementwise/tree_reduce_sum calls (kernels.py:143-310).
 *
 *   iter_a : f-partial(V,W) = sum (X - VW)^2 over the local rows,
 *            V' = V * (X W^T) / (V (W W^T) + guard)             -> V_out
 *            red = [ V'^T X (r x n) | V'^T V' (r x r) | f-partial ]
 *   iter_b : W' = W * P / (G W + guard) from the (all-reduced) red -> W_out,
 *            f_dev = red[f]
 * The row range is the caller's shard of X/V (rows are independent in the
 * V step; the W step is a sum over rows, hence the all-reduce of `red`).
 * Ranks 1..128 (MMK_E_SHAPE above).  fp32 ranks 17..128 with m, n multiples
 * of 8 run on the tensor cores (rank tiles of 64 and 128); fp64 ranks 17..128
 * on the FP64 tensor cores (DMMA tiles); ranks <= 16 on warp-per-row kernels.
 * The workspace (prepared by mmk_nnmf_ws_clear, or zero-filled, before first
 * use) caches per-X data of the fp32 tensor-core path (ranks 17..128) -- the
 * scale exponent and the pre-split fp16 hi / lo copy of X (4 bytes per
 * element, row-major; shapes whose copy would pass 96 GiB take the SIMT
 * path) -- keyed by (X, m, n, ldx): clear it again, or use a fresh one, if
 * the contents of X change in place.  mmk_nnmf_ws_clear zeroes everything
 * but the pre-split copy (written before it is read), on `stream`.
 * mmk_nnmf_ws_bytes sizes the workspace of iter / iter_a / the engine;
 * mmk_nnmf_op_ws_bytes the smaller one of the single operations below (they
 * run the SIMT kernels and never touch the tensor-core region).
 * ---------------------------------------------------------------------- */
int mmk_nnmf_ws_bytes(int dtype, int64_t m, int64_t n, int64_t r, size_t *out);
int mmk_nnmf_op_ws_bytes(int dtype, int64_t m, int64_t n, int64_t r, size_t *out);
int mmk_nnmf_ws_clear(int dtype, int64_t m, int64_t n, int64_t r, void *ws, size_t ws_bytes,
                      void *stream);
/* the per-X preparation of the tensor-core path enqueued on `stream` (a no-op
 * when the path does not apply or X is already prepared in `ws`); call it
 * before mmk_nnmf_engine_create so the GPU overlaps the graph construction */
int mmk_nnmf_prepare(int dtype, const void *X, int64_t ldx, int64_t m, int64_t n, int64_t r,
                     void *ws, size_t ws_bytes, void *stream);
int64_t mmk_nnmf_reduce_len(int64_t n, int64_t r);
int mmk_nnmf_iter_a(int dtype, const void *X, int64_t ldx, const void *V, const void *W,
                    void *V_out, int64_t m, int64_t n, int64_t r, void *ws, size_t ws_bytes,
                    double *red, int64_t *err_dev, void *stream);
int mmk_nnmf_iter_b(int dtype, const void *W, void *W_out, int64_t n, int64_t r,
                    const double *red, double *f_dev, int64_t *err_dev, void *stream);
/* single-GPU fused iteration: f(V,W) -> f_dev, (V', W') -> (V_out, W_out) */
int mmk_nnmf_iter(int dtype, const void *X, int64_t ldx, const void *V, const void *W,
                  void *V_out, void *W_out, int64_t m, int64_t n, int64_t r, void *ws,
                  size_t ws_bytes, double *red, double *f_dev, int64_t *err_dev, void *stream);
/* public single operations (nnmf.py:75-81, 84-96, 99-110) */
int mmk_nnmf_objective(int dtype, const void *X, int64_t ldx, const void *V, const void *W,
                       int64_t m, int64_t n, int64_t r, void *ws, size_t ws_bytes,
                       double *f_dev, int64_t *err_dev, void *stream);
int mmk_nnmf_update_v(int dtype, const void *X, int64_t ldx, const void *V, const void *W,
                      void *V_out, int64_t m, int64_t n, int64_t r, void *ws, size_t ws_bytes,
                      int64_t *err_dev, void *stream);
int mmk_nnmf_update_w(int dtype, const void *X, int64_t ldx, const void *V, const void *W,
                      void *W_out, int64_t m, int64_t n, int64_t r, void *ws, size_t ws_bytes,
                      double *red, int64_t *err_dev, void *stream);
/* Gradient of ||X - VW||^2 (nnmf_gradient, nnmf.py:113-119):
 * GV = 2 (V W - X) W^T (m x r), GW = 2 V^T (V W - X) (r x n); red as for
 * mmk_nnmf_update_w (reduce_len doubles). */
int mmk_nnmf_gradient(int dtype, const void *X, int64_t ldx, const void *V, const void *W,
                      void *GV, void *GW, int64_t m, int64_t n, int64_t r, void *ws,
                      size_t ws_bytes, double *red, int64_t *err_dev, void *stream);

/* ------------------------------------------------------------------------
 * NNMF, Poisson log fit (nnmf.py:178-265), rank <= 128.  Square-root
 * multiplicative MM: V' = V sqrt((R W^T) / (rowsum W + guard)) with
 * R = X / (VW) masked to x > 0, then W' = W sqrt((V'^T R') / (colsum V' +
 * guard)) with R' = X / (V'W).
 *   iter_a : f-partial(V, W) = sum x ln(VW) - VW (fp64) over the local rows,
 *            V -> V_out, red = [ V'^T R' (r x n) | colsum V' (r) | f-partial ]
 *   iter_b : W' from the (all-reduced) red -> W_out, f_dev = red[f]
 * A positive count over a zero reconstruction sets NUMERICS at site 1
 * (state's objective / V half) or 2 (W half), index i * n + j.
 * ---------------------------------------------------------------------- */
int mmk_nnmf_poisson_ws_bytes(int dtype, int64_t m, int64_t n, int64_t r, size_t *out);
int64_t mmk_nnmf_poisson_reduce_len(int64_t n, int64_t r);
int mmk_nnmf_poisson_iter_a(int dtype, const void *X, int64_t ldx, const void *V, const void *W,
                            void *V_out, int64_t m, int64_t n, int64_t r, void *ws,
                            size_t ws_bytes, double *red, int64_t *err_dev, void *stream);
int mmk_nnmf_poisson_iter_b(int dtype, const void *W, void *W_out, int64_t n, int64_t r,
                            const double *red, double *f_dev, int64_t *err_dev, void *stream);
int mmk_nnmf_poisson_iter(int dtype, const void *X, int64_t ldx, const void *V, const void *W,
                          void *V_out, void *W_out, int64_t m, int64_t n, int64_t r, void *ws,
                          size_t ws_bytes, double *red, double *f_dev, int64_t *err_dev,
                          void *stream);

/* ------------------------------------------------------------------------
 * PET penalized Poisson MM.  E is d x p (leading dim lde), y d, lam p.
 * Neighbourhoods as int32 CSR (nbr_ptr p+1, nbr_idx).  Replaces
 * pet_update / pet_penalized_objective / pet_loglik (pet.py:288-417) with the
 * forward matvec, count ratio, back-projection, neighbour sums and root.
 *
 *   iter_a : m = E lam over the local rays; ratio; loglik partial;
 *            red = [ E^T ratio (p) | loglik-partial ]
 *   iter_b : c = lam * red[b]; EM (mu = 0) or positive-root update with
 *            floor -> lam_out; f_dev = loglik - mu/2 * penalty(lam)
 * flags: MMK_PET_UPDATE (write lam_out), MMK_PET_OBJECTIVE (write f_dev),
 *        MMK_PET_CHECK_POSITIVE (flag DOMAIN at the first lam_j <= 0).
 * ---------------------------------------------------------------------- */
enum { MMK_PET_UPDATE = 1, MMK_PET_OBJECTIVE = 2, MMK_PET_CHECK_POSITIVE = 4 };
int mmk_pet_ws_bytes(int dtype, int64_t d, int64_t p, size_t *out);
int64_t mmk_pet_reduce_len(int64_t p);
int mmk_pet_iter_a(int dtype, const void *E, int64_t lde, const void *y, const void *lam,
                   int64_t d, int64_t p, void *ws, size_t ws_bytes, double *red,
                   int64_t *err_dev, void *stream);
int mmk_pet_iter_b(int dtype, const void *lam, void *lam_out, int64_t p,
                   const int32_t *nbr_ptr, const int32_t *nbr_idx, double mu, int flags,
                   const double *red, void *ws, size_t ws_bytes, double *f_dev,
                   int64_t *err_dev, void *stream);
int mmk_pet_iter(int dtype, const void *E, int64_t lde, const void *y, const void *lam,
                 void *lam_out, int64_t d, int64_t p, const int32_t *nbr_ptr,
                 const int32_t *nbr_idx, double mu, int flags, void *ws, size_t ws_bytes,
                 double *red, double *f_dev, int64_t *err_dev, void *stream);
/* Gradient of the penalized loglikelihood (pet_penalized_gradient,
 * pet.py:349-360) from red = [b | loglik] left by mmk_pet_iter_a /
 * mmk_pet_sparse_iter_a at lam:  grad_j = b_j - colsum_j
 * - mu (deg_j lam_j - sum_{k in N(j)} lam_k);  colsum fp64 (p). */
int mmk_pet_gradient(int dtype, const void *lam, void *grad, int64_t p, const int32_t *nbr_ptr,
                     const int32_t *nbr_idx, double mu, const double *colsum, const double *red,
                     void *stream);

/* Sparse system matrix variant (the Siddon matrix is ~1 % nonzero): E as
 * CSR by rays (rptr d+1, ridx, rval) for the forward projection and CSC by
 * pixels (cptr p+1, cidx, cval) for the back-projection, int32 indices,
 * values in `dtype`.  Same red layout and phase B as the dense path (a
 * sharded caller passes its rays' CSR rows and the CSC of its ray block). */
int mmk_pet_sparse_ws_bytes(int dtype, int64_t d, int64_t p, size_t *out);
int mmk_pet_sparse_iter_a(int dtype, const int32_t *rptr, const int32_t *ridx, const void *rval,
                          const int32_t *cptr, const int32_t *cidx, const void *cval,
                          const void *y, const void *lam, int64_t d, int64_t p, void *ws,
                          size_t ws_bytes, double *red, int64_t *err_dev, void *stream);
int mmk_pet_sparse_iter(int dtype, const int32_t *rptr, const int32_t *ridx, const void *rval,
                        const int32_t *cptr, const int32_t *cidx, const void *cval, const void *y,
                        const void *lam, void *lam_out, int64_t d, int64_t p,
                        const int32_t *nbr_ptr, const int32_t *nbr_idx, double mu, int flags,
                        void *ws, size_t ws_bytes, double *red, double *f_dev, int64_t *err_dev,
                        void *stream);

/* Siddon system matrix on the device (pet.py:69-132): detector positions
 * det (n_det x 2 fp64, detector_positions()), grid lines (side + 1 fp64,
 * np.linspace(-1, 1, side + 1)); one row per detector pair in the
 * reference's loop order, written as ELL: idx / val [n_rays][cap] (cap >=
 * 2 side + 3), cnt[n_rays].  Unnormalised chord lengths. */
int mmk_pet_siddon(const double *det, int n_det, int side, const double *lines, int cap,
                   int *idx, double *val, int *cnt, void *stream);

/* ------------------------------------------------------------------------
 * MDS stress majorization, full-row tiling.  theta is dim x n (SoA: row k =
 * coordinate k of every point).  Y/Wt point at row `row0` of the n x n
 * dissimilarity / weight matrices (leading dim ldy); Wt == NULL means unit
 * off-diagonal weights (1 - I, the CLI's choice, cli.py:181).  wsum = row
 * sums of the weights (fp64, n).  Replaces stress / mds_update
 * (mds.py:79-144): no n x n temporary is formed.
 *
 * Computes, for the `rows` points starting at row0,
 *   theta_out[:, i - row0] (leading dim ldo) = the MM update of point i
 *   f_dev = sum_{i in rows, j > i} w_ij (y_ij - d_ij)^2   (stress partial)
 * flags: MMK_MDS_UPDATE, MMK_MDS_OBJECTIVE.  Coupled coincident points
 * (d_ij = 0, w_ij y_ij > 0) set NUMERICS with index i*n + j.
 * MMK_MDS_GRADIENT instead writes the stress gradient (stress_gradient,
 * mds.py:147-167) 2 (theta_i (w_i. - z_i.) - sum_j (w_ij - z_ij) theta_j)
 * to theta_out; coincident points with w_ij > 0 set NUMERICS.
 * ---------------------------------------------------------------------- */
enum { MMK_MDS_UPDATE = 1, MMK_MDS_OBJECTIVE = 2, MMK_MDS_GRADIENT = 4 };
int mmk_mds_ws_bytes(int dtype, int64_t n, int64_t dim, int64_t rows, size_t *out);
int mmk_mds_iter(int dtype, const void *Y, const void *Wt, int64_t ldy, const double *wsum,
                 const void *theta, void *theta_out, int64_t ldo, int64_t dim, int64_t n,
                 int64_t row0, int64_t rows, int flags, void *ws, size_t ws_bytes,
                 double *f_dev, int64_t *err_dev, void *stream);

/* ------------------------------------------------------------------------
 * MDS for large unit-weight problems (W = 1 - I, cli.py:181) over a PACKED
 * UPPER TRIANGLE of Y: 128 x 128 tiles (I <= J) stored row-major over the
 * triangle, 64 KB each (fp32 only, dim <= 3).  Every unordered pair is
 * visited once per iteration (half the bytes of a full-row pass).
 * Replaces stress / mds_update / _coincidence_error (mds.py:92-144) for the
 * BASELINE config-5 shape.  [t0, t1) is this rank's range of linear tile
 * indices (all tiles on one GPU; a balanced split when sharded).
 *
 *   pack   : tiles of [t0, t1) whose tile row lies in full rows
 *            [row0, row0 + rows) of Y (leading dim ldy) -> packed
 *            (packed[u] = tile t0 + u); validate != 0 also checks finite,
 *            nonnegative, zero diagonal and exact symmetry (DOMAIN sites
 *            2, 3, 5, 4) where the transposed row is inside the block.
 *   iter_a : red = [ per point C_i[dim] = sum_j z_ij (theta_j - theta_i) |
 *            stress partial | S = sum_i theta_i (from the rank holding
 *            tile 0 only) ] (fp64, n*dim + 1 + dim); the sharded caller
 *            all-reduces it.
 *   iter_b : theta_out = MM update from red, f_dev = stress.
 * Coupled coincident points set NUMERICS with index i*n + j (site 1).
 * ---------------------------------------------------------------------- */
/* Roll-call votes (q x m, entries 1 / -1 / 0, fp32 or fp64 `dtype`) straight
 * into packed-triangle fp32 dissimilarity tiles [t0, t1) on the tensor cores
 * (votes_to_dissimilarity, mds.py:260-283: D = (S - N) / (2 S) with S = P P^T,
 * N = V V^T, exact in fp16 x fp16 -> fp32).  ws >= mmk_mds_votes_bytes.
 * DOMAIN errors: site 6 bad vote entry (index i*m + k), site 7 a pair sharing
 * no roll call (index i*q + j, i < j). */
int mmk_mds_votes_bytes(int64_t q, int64_t m, size_t *out);
int mmk_mds_votes_tri(int dtype, const void *votes, int64_t q, int64_t m, float *packed,
                      int64_t t0, int64_t t1, void *ws, size_t ws_bytes, int64_t *err_dev,
                      void *stream);
int64_t mmk_mds_tri_ntiles(int64_t n);
int64_t mmk_mds_tri_reduce_len(int64_t n, int64_t dim);
int mmk_mds_tri_ws_bytes(int64_t n, int64_t dim, int64_t t0, int64_t t1, size_t *out);
int mmk_mds_tri_pack(const float *Y, int64_t ldy, int64_t n, int64_t row0, int64_t rows,
                     float *packed, int64_t t0, int64_t t1, int validate, int64_t *err_dev,
                     void *stream);
int mmk_mds_tri_iter_a(const float *packed, int64_t t0, int64_t t1, const float *theta,
                       int64_t dim, int64_t n, void *ws, size_t ws_bytes, double *red,
                       int64_t *err_dev, void *stream);
int mmk_mds_tri_iter_b(const float *theta, float *theta_out, int64_t dim, int64_t n,
                       const double *red, double *f_dev, int64_t *err_dev, void *stream);
int mmk_mds_tri_iter(const float *packed, int64_t t0, int64_t t1, const float *theta,
                     float *theta_out, int64_t dim, int64_t n, void *ws, size_t ws_bytes,
                     double *red, double *f_dev, int64_t *err_dev, void *stream);

/* ------------------------------------------------------------------------
 * Sharded-layout helper: gathered [G][dim][rows_pad] -> theta [dim][n]
 * (the coordinate all-gather of the row-sharded MDS path).
 * ---------------------------------------------------------------------- */
int mmk_mds_unpack(int dtype, const void *gathered, void *theta, int64_t dim, int64_t n,
                   int64_t rows_pad, void *stream);

/* ------------------------------------------------------------------------
 * Collectives over the process's NCCL (torch.distributed's communicator,
 * passed as ProcessGroupNCCL._comm_ptr()).  Sum all-reduce of the fp64
 * phase-A buffers; all-gather of state slices.  Resolved at run time with
 * dlsym, so libmmk.so has no link-time NCCL dependency.
 * ---------------------------------------------------------------------- */
int mmk_nccl_available(void);
int mmk_allreduce_f64(double *buf, int64_t count, void *comm, void *stream);
int mmk_allgather(const void *send, void *recv, int64_t count, int dtype, void *comm,
                  void *stream);

/* ------------------------------------------------------------------------
 * Device-side MM loop (replaces the host loop of run_mm, driver.py:101-149,
 * with identical stopping / monotonicity / non-finite semantics).
 *
 * An engine is ONE CUDA graph: a conditional WHILE node whose body runs one
 * fused iteration A -> B (f(A) into ctl[MMK_CTL_FCUR]) and a control kernel
 * that applies the stopping rule, then -- inside a conditional IF node --
 * the iteration B -> A and its control kernel: two iterations per body,
 * no state copies.  Each mmk_engine_run() launch advances until the run
 * stops or `batch` (even) iterations were recorded.  trace[k] / tstamp[k]
 * (k = it - batch start) receive f(S_it) and the device globaltimer (ns).
 * When the run stops at iteration `it`, S_it is in slot A if
 * ctl[MMK_CTL_SLOT] == 0, else in slot B; after a pause it is in slot A.  ctl (16 int64, zeroed by the caller
 * before the first launch) holds the loop state.  With comm != NULL the
 * body also all-reduces the phase-A buffer (NNMF, PET) or the stress
 * partial + coordinate all-gather (MDS) over NCCL.
 * ---------------------------------------------------------------------- */
typedef struct {
    double epsilon;
    double monotone_tol;
    double sign;          /* +1 maximize, -1 minimize */
    int64_t max_iters;
    int64_t batch;
    int32_t check_monotone;
    int32_t pad_;
} mmk_stop_rule;

enum {
    MMK_CTL_IT = 0,          /* index of the state whose objective was recorded last */
    MMK_CTL_REASON = 1,      /* MMK_STOP_* (0 while running / paused) */
    MMK_CTL_BATCH_START = 2, /* iteration index stored at trace[0] of the current batch */
    MMK_CTL_FPREV = 3,       /* fp64 bits */
    MMK_CTL_FCUR = 4,        /* fp64 bits: f_dev of the iteration kernels */
    MMK_CTL_REL = 5,         /* fp64 bits: last relative change */
    MMK_CTL_SLOT = 6,        /* after a stop: 0 -> state in slot A, 1 -> slot B */
    MMK_CTL_LAST = 7,        /* 1: the next pass is the last (iteration cap) and only its f
                                is recorded -- the fp32 tensor-core NNMF engine skips the
                                W half of that pass */
    MMK_CTL_LEN = 16
};
enum {
    MMK_STOP_RUNNING = 0,
    MMK_STOP_CONVERGED = 1,
    MMK_STOP_CAP = 2,
    MMK_STOP_NONFINITE = 3,
    MMK_STOP_MONOTONE = 4,
    MMK_STOP_DEVICE_ERROR = 5
};

int mmk_nnmf_engine_create(int dtype, const void *X, int64_t ldx, void *VA, void *WA, void *VB,
                           void *WB, int64_t m, int64_t n, int64_t r, void *ws, size_t ws_bytes,
                           double *red, void *comm, const mmk_stop_rule *rule, double *trace,
                           int64_t *tstamp, int64_t *ctl, int64_t *err_dev, void **engine);
int mmk_nnmf_poisson_engine_create(int dtype, const void *X, int64_t ldx, void *VA, void *WA,
                                   void *VB, void *WB, int64_t m, int64_t n, int64_t r, void *ws,
                                   size_t ws_bytes, double *red, void *comm,
                                   const mmk_stop_rule *rule, double *trace, int64_t *tstamp,
                                   int64_t *ctl, int64_t *err_dev, void **engine);
int mmk_pet_engine_create(int dtype, const void *E, int64_t lde, const void *y, void *lamA,
                          void *lamB, int64_t d, int64_t p, const int32_t *nbr_ptr,
                          const int32_t *nbr_idx, double mu, void *ws, size_t ws_bytes,
                          double *red, void *comm, const mmk_stop_rule *rule, double *trace,
                          int64_t *tstamp, int64_t *ctl, int64_t *err_dev, void **engine);
int mmk_pet_sparse_engine_create(int dtype, const int32_t *rptr, const int32_t *ridx,
                                 const void *rval, const int32_t *cptr, const int32_t *cidx,
                                 const void *cval, const void *y, void *lamA, void *lamB,
                                 int64_t d, int64_t p, const int32_t *nbr_ptr,
                                 const int32_t *nbr_idx, double mu, void *ws, size_t ws_bytes,
                                 double *red, void *comm, const mmk_stop_rule *rule,
                                 double *trace, int64_t *tstamp, int64_t *ctl, int64_t *err_dev,
                                 void **engine);
int mmk_mds_engine_create(int dtype, const void *Y, const void *Wt, int64_t ldy,
                          const double *wsum, void *thetaA, void *thetaB, void *local_out,
                          void *gathered, int64_t dim, int64_t n, int64_t row0, int64_t rows,
                          int64_t rows_pad, void *ws, size_t ws_bytes, void *comm,
                          const mmk_stop_rule *rule, double *trace, int64_t *tstamp,
                          int64_t *ctl, int64_t *err_dev, void **engine);
int mmk_mds_tri_engine_create(const float *packed, int64_t t0, int64_t t1, float *thetaA,
                              float *thetaB, int64_t dim, int64_t n, void *ws, size_t ws_bytes,
                              double *red, void *comm, const mmk_stop_rule *rule, double *trace,
                              int64_t *tstamp, int64_t *ctl, int64_t *err_dev, void **engine);
int mmk_engine_run(void *engine, void *stream);
void mmk_engine_destroy(void *engine);

/* MMX1 loader (replaces the host decode of io.py:90-106 `_load_binary` for
 * device runs): narrow n landed fp64 values to fp32, round-to-nearest-even
 * (numpy astype(float32)); src/dst 16-byte aligned device buffers. */
int mmk_f64_to_f32(const double *src, float *dst, int64_t n, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MMK_H_ */
