// nnmf_ref.cu -- the fp64 single operations of the Frobenius NNMF in the
// reference's own arithmetic order, so they are bitwise equal to mmkit's
// nnmf_objective / nnmf_update_v / nnmf_update_w / nnmf_gradient
// (nnmf.py:75-119) -- including its fixed point: X = VW (computed by its
// matmul) leaves V and W unchanged bit for bit (test_nnmf.py:46-52).
//
// The reference matmul (kernels.py:139-215) forms every inner product as a
// pairwise tree: the products a_k b_k rounded separately, summed in pairs
// (2t, 2t+1), an odd tail carried to the next level, repeated to one value
// (_pairwise_collapse).  A thread here streams the K products of its output
// through a stack of partial sums -- push a product at level 0, merge the two
// top entries while their levels agree, at the end fold the stack from the
// top (right to left).  That reproduces the halving tree exactly: the merged
// entries are the perfect subtrees over aligned power-of-two blocks, and the
// leftover blocks of the binary decomposition of K meet in the order the
// carried tails do.  tree_reduce_sum (kernels.py:261-285) over the m n
// squared residuals is the same tree over a flattened array: blocks of 2048
// aligned elements reduce to their subtree sums (a partial last block by
// halving with carry, which is exactly what the global tree does to it), and
// the block sums are reduced again the same way.  Every add / multiply /
// divide is explicitly rounded (__dadd_rn, __dmul_rn, __ddiv_rn): no FMA
// contraction, as in the reference's numba kernels (the C oracle, compiled
// with -ffp-contract=off, is bitwise pinned to them).
//
// These are single operations (not the iteration hot path): one thread per
// output element, O(m n r) work, the reconstruction V W materialised once.
#include "mmk_common.cuh"

namespace {

constexpr int kLevels = 40;   // stack depth: K < 2^39

struct Tree {
    double val[kLevels];
    int lvl[kLevels];
    int top = 0;
    __device__ __forceinline__ void push(double p) {
        val[top] = p;
        lvl[top] = 0;
        ++top;
        while (top >= 2 && lvl[top - 1] == lvl[top - 2]) {
            val[top - 2] = __dadd_rn(val[top - 2], val[top - 1]);
            lvl[top - 2] += 1;
            --top;
        }
    }
    __device__ __forceinline__ double fold() {
        if (top == 0) return 0.0;
        double s = val[top - 1];
        for (int t = top - 2; t >= 0; --t) s = __dadd_rn(val[t], s);
        return s;
    }
};

// C[i][j] = tree_k A(i, k) B(k, j) with A(i, k) = A[i sai + k sak],
// B(k, j) = B[k sbk + j sbj]; SCALE multiplies the result (2.0: the gradient)
__global__ void tree_mm_kernel(const double* __restrict__ A, long long sai, long long sak,
                               const double* __restrict__ B, long long sbk, long long sbj,
                               double* __restrict__ C, long long ldc, long long M, long long N,
                               long long K, double scale) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long i = blockIdx.y;
    if (j >= N || i >= M) return;
    Tree t;
    for (long long k = 0; k < K; ++k) t.push(__dmul_rn(A[i * sai + k * sak], B[k * sbk + j * sbj]));
    const double s = t.fold();
    C[i * ldc + j] = scale == 1.0 ? s : __dmul_rn(scale, s);
}

// out = f * (num / (den + 1e-300)), elementwise (nnmf.py:95, 109)
__global__ void tree_update_kernel(const double* __restrict__ f, const double* __restrict__ num,
                                   const double* __restrict__ den, double* __restrict__ out,
                                   long long len) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= len) return;
    out[t] = __dmul_rn(f[t], __ddiv_rn(num[t], __dadd_rn(den[t], mmk::kDenomGuard)));
}

// recon - x, elementwise (nnmf.py:116); ldx is X's row stride
__global__ void tree_resid_kernel(const double* __restrict__ recon, const double* __restrict__ X,
                                  long long ldx, double* __restrict__ out, long long m,
                                  long long n) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m * n) return;
    const long long i = t / n, j = t - i * n;
    out[t] = __dsub_rn(recon[t], X[i * ldx + j]);
}

constexpr int kChunk = 2048;   // elements per block of the tree reduction
constexpr int kRedThreads = 256;

// halving with carry over s[0..len) in shared memory (ping-pong with d),
// returns the single value in thread 0
__device__ double halve_block(double* s, double* d, int len) {
    while (len > 1) {
        const int half = len >> 1;
        for (int t = threadIdx.x; t < half; t += blockDim.x) d[t] = __dadd_rn(s[2 * t], s[2 * t + 1]);
        if ((len & 1) && threadIdx.x == 0) d[half] = s[len - 1];
        __syncthreads();
        double* tmp = s;
        s = d;
        d = tmp;
        len = half + (len & 1);
    }
    return s[0];
}

// SQ: element e of the flattened m x n array is (x_ij - recon_ij)^2 with
// recon read from `recon` (nnmf.py:80); else element e is src[e]
template <bool SQ>
__global__ void __launch_bounds__(kRedThreads)
tree_chunk_kernel(const double* __restrict__ src, const double* __restrict__ X, long long ldx,
                  long long n, long long len, double* __restrict__ out) {
    __shared__ double s[kChunk], d[kChunk / 2 + 1];
    const long long e0 = (long long)blockIdx.x * kChunk;
    const int cnt = (int)(len - e0 < kChunk ? len - e0 : kChunk);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const long long e = e0 + t;
        double v;
        if (SQ) {
            const long long i = e / n, j = e - i * n;
            const double diff = __dsub_rn(X[i * ldx + j], src[e]);
            v = __dmul_rn(diff, diff);
        } else {
            v = src[e];
        }
        s[t] = v;
    }
    __syncthreads();
    // the first level writes into d (size kChunk / 2 + 1); later levels ping-pong
    const double r = halve_block(s, d, cnt);
    if (threadIdx.x == 0) out[blockIdx.x] = r;
}

}  // namespace

namespace mmk_ref {

static int status(const char* what) {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MMK_OK : mmk_host::cuda_status(e, what);
}

// workspace: recon (m n) | num (max(m r, r n)) | den (same) | two partial buffers
static size_t take(size_t& off, size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
}

size_t ws_bytes(long long m, long long n, long long r) {
    size_t off = 0;
    const long long mn = m * n, big = (m * r > r * n ? m * r : r * n);
    const long long p1 = (mn + kChunk - 1) / kChunk + 1;
    take(off, sizeof(double) * (size_t)(mn > 0 ? mn : 1));
    take(off, sizeof(double) * (size_t)big);
    take(off, sizeof(double) * (size_t)big);
    take(off, sizeof(double) * (size_t)p1);
    take(off, sizeof(double) * (size_t)p1);
    return off;
}

struct L {
    double *recon, *num, *den, *p1, *p2;
};

static L layout(long long m, long long n, long long r, void* ws) {
    size_t off = 0;
    const long long mn = m * n, big = (m * r > r * n ? m * r : r * n);
    const long long p1 = (mn + kChunk - 1) / kChunk + 1;
    char* c = reinterpret_cast<char*>(ws);
    L l;
    l.recon = reinterpret_cast<double*>(c + take(off, sizeof(double) * (size_t)(mn > 0 ? mn : 1)));
    l.num = reinterpret_cast<double*>(c + take(off, sizeof(double) * (size_t)big));
    l.den = reinterpret_cast<double*>(c + take(off, sizeof(double) * (size_t)big));
    l.p1 = reinterpret_cast<double*>(c + take(off, sizeof(double) * (size_t)p1));
    l.p2 = reinterpret_cast<double*>(c + take(off, sizeof(double) * (size_t)p1));
    return l;
}

static void mm(const double* A, long long sai, long long sak, const double* B, long long sbk,
               long long sbj, double* C, long long ldc, long long M, long long N, long long K,
               cudaStream_t st, double scale = 1.0) {
    if (M <= 0 || N <= 0) return;
    dim3 grid((unsigned)((N + 127) / 128), (unsigned)M);
    MMK_LAUNCH("nnmf_tree_mm", st,
               (tree_mm_kernel<<<grid, 128, 0, st>>>(A, sai, sak, B, sbk, sbj, C, ldc, M, N, K,
                                                     scale)));
}

// recon = V W (m x n, K = r): matmul(v, w) (nnmf.py:77, 93, 107, 115)
static void recon(const double* V, const double* W, long long m, long long n, long long r,
                  double* out, cudaStream_t st) {
    mm(V, r, 1, W, n, 1, out, n, m, n, r, st);
}

int objective(const double* X, long long ldx, const double* V, const double* W, long long m,
              long long n, long long r, void* ws, double* f_dev, cudaStream_t st) {
    L l = layout(m, n, r, ws);
    const long long mn = m * n;
    if (mn == 0) {
        cudaMemsetAsync(f_dev, 0, sizeof(double), st);
        return status("nnmf_tree_objective");
    }
    recon(V, W, m, n, r, l.recon, st);
    long long len = (mn + kChunk - 1) / kChunk;
    MMK_LAUNCH("nnmf_tree_sum", st,
               (tree_chunk_kernel<true><<<(unsigned)len, kRedThreads, 0, st>>>(l.recon, X, ldx, n,
                                                                               mn, l.p1)));
    double *src = l.p1, *dst = l.p2;
    while (len > 1) {
        const long long next = (len + kChunk - 1) / kChunk;
        MMK_LAUNCH("nnmf_tree_sum", st,
                   (tree_chunk_kernel<false><<<(unsigned)next, kRedThreads, 0, st>>>(
                       src, nullptr, 0, 1, len, dst)));
        double* t = src;
        src = dst;
        dst = t;
        len = next;
    }
    cudaMemcpyAsync(f_dev, src, sizeof(double), cudaMemcpyDeviceToDevice, st);
    return status("nnmf_tree_objective");
}

// v <- v * (X W^T) / ((V W) W^T + 1e-300)   (nnmf.py:84-96)
int update_v(const double* X, long long ldx, const double* V, const double* W, double* Vout,
             long long m, long long n, long long r, void* ws, cudaStream_t st) {
    L l = layout(m, n, r, ws);
    mm(X, ldx, 1, W, 1, n, l.num, r, m, r, n, st);        // matmul(x, w, transpose_b)
    recon(V, W, m, n, r, l.recon, st);
    mm(l.recon, n, 1, W, 1, n, l.den, r, m, r, n, st);    // matmul(recon, w, transpose_b)
    const long long len = m * r;
    if (len > 0)
        MMK_LAUNCH("nnmf_tree_update", st,
                   (tree_update_kernel<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(
                       V, l.num, l.den, Vout, len)));
    return status("nnmf_tree_update_v");
}

// w <- w * (V^T X) / (V^T (V W) + 1e-300)   (nnmf.py:99-110)
int update_w(const double* X, long long ldx, const double* V, const double* W, double* Wout,
             long long m, long long n, long long r, void* ws, cudaStream_t st) {
    L l = layout(m, n, r, ws);
    mm(V, 1, r, X, ldx, 1, l.num, n, r, n, m, st);        // matmul(v, x, transpose_a)
    recon(V, W, m, n, r, l.recon, st);
    mm(V, 1, r, l.recon, n, 1, l.den, n, r, n, m, st);    // matmul(v, recon, transpose_a)
    const long long len = r * n;
    if (len > 0)
        MMK_LAUNCH("nnmf_tree_update", st,
                   (tree_update_kernel<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(
                       W, l.num, l.den, Wout, len)));
    return status("nnmf_tree_update_w");
}

// grad_v = 2 (V W - X) W^T, grad_w = 2 V^T (V W - X)   (nnmf.py:113-119)
int gradient(const double* X, long long ldx, const double* V, const double* W, double* GV,
             double* GW, long long m, long long n, long long r, void* ws, cudaStream_t st) {
    L l = layout(m, n, r, ws);
    recon(V, W, m, n, r, l.recon, st);
    const long long mn = m * n;
    if (mn > 0)   // resid = recon - x, in place
        MMK_LAUNCH("nnmf_tree_resid", st,
                   (tree_resid_kernel<<<(unsigned)((mn + 255) / 256), 256, 0, st>>>(
                       l.recon, X, ldx, l.recon, m, n)));
    mm(l.recon, n, 1, W, 1, n, GV, r, m, r, n, st, 2.0);  // 2 * matmul(resid, w, transpose_b)
    mm(V, 1, r, l.recon, n, 1, GW, n, r, n, m, st, 2.0);  // 2 * matmul(v, resid, transpose_a)
    return status("nnmf_tree_gradient");
}

}  // namespace mmk_ref
