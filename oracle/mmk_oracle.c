/*
 * mmk_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * CPU restatement of the reference's deterministic dense kernels
 * (/root/reference/pkg/src/mmkit/kernels.py).  Only tests/, the smoke check
 * in __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs
 * may load this library; the product path never does.
 *
 * Association order is reproduced exactly so that results are bitwise equal
 * to the reference's numba loops (compiled here with -ffp-contract=off so no
 * multiply-add is fused, as LLVM does not fuse without fast-math):
 *
 *   ora_collapse  <- _pairwise_collapse  kernels.py:112-130
 *                    (pairwise halving, odd tail carried to the next level)
 *   ora_matmul    <- _mm_nn/_mm_nt/_mm_tn/_mm_tt  kernels.py:143-204
 *                    (first halving level fused with the products)
 *   ora_tree_sum  <- tree_reduce_sum  kernels.py:259-282 (serial and
 *                    level-parallel paths share one association order)
 *   ora_neighbor_sums <- pet._neighbor_sums  pet.py:204-210
 *
 * Parallelism partitions disjoint output rows over pthreads, the same
 * decomposition as run_partitioned (kernels.py:92-109), so any thread
 * count gives identical bits.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

static double collapse(double *buf, int64_t n) {
    if (n == 0) return 0.0;
    while (n > 1) {
        int64_t half = n / 2;
        for (int64_t t = 0; t < half; ++t) buf[t] = buf[2 * t] + buf[2 * t + 1];
        if (n & 1) {
            buf[half] = buf[n - 1];
            n = half + 1;
        } else {
            n = half;
        }
    }
    return buf[0];
}

double ora_collapse(double *buf, int64_t n) { return collapse(buf, n); }

double ora_tree_sum(const double *v, int64_t n) {
    if (n == 0) return 0.0;
    double *buf = (double *)malloc(sizeof(double) * (size_t)n);
    memcpy(buf, v, sizeof(double) * (size_t)n);
    double s = collapse(buf, n);
    free(buf);
    return s;
}

/* op(A) is rows x inner, op(B) is inner x cols; A, B, C row-major contiguous.
 * A stored as (ta ? inner x rows : rows x inner), B as (tb ? cols x inner :
 * inner x cols). */
typedef struct {
    const double *a, *b;
    double *c;
    int64_t rows, inner, cols, lo, hi;
    int ta, tb;
} mm_job;

static void *mm_rows(void *arg) {
    const mm_job *J = (const mm_job *)arg;
    const int64_t inner = J->inner, rows = J->rows, cols = J->cols;
    const int64_t half = inner / 2;
    const int64_t m = (inner & 1) ? half + 1 : half;
    const double *a = J->a, *b = J->b;
    const int ta = J->ta, tb = J->tb;
    double *buf = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    for (int64_t i = J->lo; i < J->hi; ++i) {
        for (int64_t j = 0; j < cols; ++j) {
#define A_(r, k) (ta ? a[(k) * rows + (r)] : a[(r) * inner + (k)])
#define B_(k, cc) (tb ? b[(cc) * inner + (k)] : b[(k) * cols + (cc)])
            for (int64_t t = 0; t < half; ++t)
                buf[t] = A_(i, 2 * t) * B_(2 * t, j) + A_(i, 2 * t + 1) * B_(2 * t + 1, j);
            if (inner & 1) buf[half] = A_(i, inner - 1) * B_(inner - 1, j);
            J->c[i * cols + j] = inner > 0 ? collapse(buf, m) : 0.0;
#undef A_
#undef B_
        }
    }
    free(buf);
    return NULL;
}

/* Contiguous row chunks, the first (rows % parts) one row longer: the
 * partition of kernels._partition (kernels.py:79-89). */
int ora_matmul(const double *a, const double *b, double *c, int64_t rows,
               int64_t inner, int64_t cols, int ta, int tb, int threads) {
    if (threads < 1) threads = 1;
    if (threads > rows) threads = rows > 0 ? (int)rows : 1;
    if (threads > 256) threads = 256;
    mm_job jobs[256];
    pthread_t tid[256];
    int64_t base = rows / threads, extra = rows % threads, lo = 0;
    for (int p = 0; p < threads; ++p) {
        int64_t hi = lo + base + (p < extra ? 1 : 0);
        mm_job J = {a, b, c, rows, inner, cols, lo, hi, ta, tb};
        jobs[p] = J;
        lo = hi;
    }
    if (threads == 1) {
        mm_rows(&jobs[0]);
        return 0;
    }
    for (int p = 1; p < threads; ++p) pthread_create(&tid[p], NULL, mm_rows, &jobs[p]);
    mm_rows(&jobs[0]);
    for (int p = 1; p < threads; ++p) pthread_join(tid[p], NULL);
    return 0;
}

void ora_neighbor_sums(const int64_t *indptr, const int64_t *indices,
                       const double *lam, double *out, int64_t n) {
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t t = indptr[j]; t < indptr[j + 1]; ++t) s += lam[indices[t]];
        out[j] = s;
    }
}

int ora_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
