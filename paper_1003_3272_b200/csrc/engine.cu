// engine.cu -- the MM driver loop on the device.
//
// The reference driver (driver.py:101-149) reads one objective per iteration
// on the host to apply its stopping rule.  For the paper-shape problems the
// whole iteration is a few microseconds of GPU work, so a host round trip per
// iteration would dominate.  The engine instead records ONE CUDA graph
//
//     WHILE (w) {  iteration(A -> B, f(A)) ; control(f)  ->  w, i
//                  IF (i) { iteration(B -> A, f(B)) ; control(f) -> w } }
//
// using conditional WHILE and IF nodes: two iterations per body with the
// state slots swapped, so no state copy is needed.  The control kernel applies exactly the
// reference's rules -- non-finite check, monotone slack
// monotone_tol * (1 + |f_prev|), relative change |f - f_prev| / (|f_prev| + 1)
// < epsilon, the max_iters cap -- records the objective trace and a device
// timestamp per iteration, and clears the condition to stop, or to pause
// every `batch` iterations so the host can drain the trace buffer.  When the
// loop stops at iteration k, slot A holds state k (the reference returns the
// state whose objective was the last one recorded).
//
// Multi-GPU engines additionally capture the NCCL all-reduce of the phase-A
// buffer inside the body (ncclAllReduce resolved from the process's NCCL, the
// one torch.distributed loaded), so a sharded run is also one graph launch
// per batch.
#include <dlfcn.h>

#include <functional>
#include <mutex>
#include <vector>

#include "mm_control.cuh"
#include "nnmf_tc.h"
#include "small_engine.h"

namespace {

using namespace mmk;

struct Engine {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cap = nullptr;
    mmk_small::Launch persistent;   // set: one persistent-kernel launch per batch
    std::function<int(cudaStream_t)> prologue;   // once, before the first batch
    bool prologue_done = false;
};

// half 0 follows iteration A -> B (its objective is f(A)), half 1 follows
// B -> A.  A stop records which slot holds the returned state (the input of
// the last recorded objective, as run_mm returns it); batch pauses happen only
// after half 1, so every launch starts from slot A.
__global__ void control_kernel(cudaGraphConditionalHandle h, cudaGraphConditionalHandle hif,
                               int half, long long* ctl, double* trace, long long* tstamp,
                               const long long* err, mmk_stop_rule rule) {
    if (threadIdx.x != 0) return;
    const int d = mm_control(half, ctl, trace, tstamp, err, rule, ctl_f64(ctl[MMK_CTL_FCUR]));
    if (d == kMmStop) {
        cudaGraphSetConditional(h, 0);
        if (half == 0) cudaGraphSetConditional(hif, 0);
    } else if (half == 0) {
        cudaGraphSetConditional(hif, 1);
    } else if (d == kMmPause) {
        cudaGraphSetConditional(h, 0);
    }
}

#define ENG_CHECK(call, what)                                          \
    do {                                                               \
        cudaError_t _e = (call);                                       \
        if (_e != cudaSuccess) {                                       \
            rc = mmk_host::cuda_status(_e, what);                      \
            goto fail;                                                 \
        }                                                              \
    } while (0)

using IterFn = std::function<int(cudaStream_t, int /* 0: A -> B, 1: B -> A */)>;

// capture `iter(dir)` + control(half = dir) into `g`; returns the last node
int capture_half(Engine* e, cudaGraph_t g, const IterFn& iter, int dir,
                 cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi,
                 const mmk_stop_rule* rule, double* trace, int64_t* tstamp, int64_t* ctl,
                 int64_t* err, cudaGraphNode_t* last) {
    int rc = MMK_OK;
    cudaGraph_t captured;
    cudaError_t ce = cudaStreamBeginCaptureToGraph(e->cap, g, nullptr, nullptr, 0,
                                                   cudaStreamCaptureModeThreadLocal);
    if (ce != cudaSuccess) return mmk_host::cuda_status(ce, "cudaStreamBeginCaptureToGraph");
    rc = iter(e->cap, dir);
    if (rc == MMK_OK) {
        control_kernel<<<1, 32, 0, e->cap>>>(hw, hi, dir, reinterpret_cast<long long*>(ctl), trace,
                                             reinterpret_cast<long long*>(tstamp),
                                             reinterpret_cast<const long long*>(err), *rule);
        cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) rc = mmk_host::cuda_status(le, "control_kernel");
    }
    if (rc == MMK_OK && last) {
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        ce = cudaStreamGetCaptureInfo(e->cap, &cs, nullptr, nullptr, &deps, &nd);
        if (ce != cudaSuccess || nd != 1) rc = mmk_host::cuda_status(
            ce != cudaSuccess ? ce : cudaErrorInvalidValue, "cudaStreamGetCaptureInfo");
        else
            *last = deps[0];
    }
    ce = cudaStreamEndCapture(e->cap, &captured);
    if (rc == MMK_OK && ce != cudaSuccess) rc = mmk_host::cuda_status(ce, "EndCapture");
    return rc;
}

int build(const IterFn& iter, const mmk_stop_rule* rule, double* trace, int64_t* tstamp,
          int64_t* ctl, int64_t* err, void** out) {
    int rc = MMK_OK;
    Engine* e = new Engine();
    cudaGraphConditionalHandle hw, hi;
    cudaGraphNodeParams np = {}, ip = {};
    cudaGraphNode_t node, ifnode, last = nullptr;
    cudaGraph_t body;
    if (rule->batch < 2 || (rule->batch & 1)) {
        mmk_host::set_error("engine batch must be an even number >= 2");
        rc = MMK_E_SHAPE;
        goto fail;
    }
    ENG_CHECK(cudaGraphCreate(&e->graph, 0), "cudaGraphCreate");
    ENG_CHECK(cudaGraphConditionalHandleCreate(&hw, e->graph, 1, cudaGraphCondAssignDefault),
              "cudaGraphConditionalHandleCreate(while)");
    ENG_CHECK(cudaGraphConditionalHandleCreate(&hi, e->graph, 0, 0),
              "cudaGraphConditionalHandleCreate(if)");
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = hw;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    ENG_CHECK(cudaGraphAddNode(&node, e->graph, nullptr, 0, &np), "cudaGraphAddNode(while)");
    body = np.conditional.phGraph_out[0];
    ENG_CHECK(cudaStreamCreateWithFlags(&e->cap, cudaStreamNonBlocking), "cudaStreamCreate");
    rc = capture_half(e, body, iter, 0, hw, hi, rule, trace, tstamp, ctl, err, &last);
    if (rc != MMK_OK) goto fail;
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    ENG_CHECK(cudaGraphAddNode(&ifnode, body, &last, 1, &ip), "cudaGraphAddNode(if)");
    rc = capture_half(e, ip.conditional.phGraph_out[0], iter, 1, hw, hi, rule, trace, tstamp, ctl,
                      err, nullptr);
    if (rc != MMK_OK) goto fail;
    ENG_CHECK(cudaGraphInstantiate(&e->exec, e->graph, 0), "cudaGraphInstantiate");
    *out = e;
    return MMK_OK;
fail:
    if (e->exec) cudaGraphExecDestroy(e->exec);
    if (e->graph) cudaGraphDestroy(e->graph);
    if (e->cap) cudaStreamDestroy(e->cap);
    delete e;
    *out = nullptr;
    return rc;
}

// ncclAllReduce from the NCCL already loaded into the process (torch's).
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
constexpr int kNcclDouble = 8, kNcclFloat = 7, kNcclSum = 0;

template <typename F>
F nccl_sym(const char* name) {
    void* s = dlsym(RTLD_DEFAULT, name);
    if (!s) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (h) s = dlsym(h, name);
    }
    return reinterpret_cast<F>(s);
}

}  // namespace

extern "C" int mmk_nccl_available(void) {
    return nccl_sym<nccl_allreduce_fn>("ncclAllReduce") != nullptr ? 1 : 0;
}

extern "C" int mmk_allreduce_f64(double* buf, int64_t count, void* comm, void* stream) {
    auto fn = nccl_sym<nccl_allreduce_fn>("ncclAllReduce");
    if (!fn) {
        mmk_host::set_error("ncclAllReduce not found in the process (is torch.distributed "
                            "initialised with the nccl backend?)");
        return MMK_E_CUDA;
    }
    int r = fn(buf, buf, (size_t)count, kNcclDouble, kNcclSum, comm,
               reinterpret_cast<cudaStream_t>(stream));
    if (r != 0) {
        mmk_host::set_error("ncclAllReduce failed with ncclResult %d", r);
        return MMK_E_CUDA;
    }
    return MMK_OK;
}

extern "C" int mmk_allgather(const void* send, void* recv, int64_t count, int dtype, void* comm,
                             void* stream) {
    auto fn = nccl_sym<nccl_allgather_fn>("ncclAllGather");
    if (!fn) {
        mmk_host::set_error("ncclAllGather not found in the process");
        return MMK_E_CUDA;
    }
    int r = fn(send, recv, (size_t)count, dtype == MMK_F32 ? kNcclFloat : kNcclDouble, comm,
               reinterpret_cast<cudaStream_t>(stream));
    if (r != 0) {
        mmk_host::set_error("ncclAllGather failed with ncclResult %d", r);
        return MMK_E_CUDA;
    }
    return MMK_OK;
}

extern "C" int mmk_engine_run(void* eng, void* stream) {
    MMK_NVTX("mmk_engine_run");
    Engine* e = reinterpret_cast<Engine*>(eng);
    if (!e) {
        mmk_host::set_error("null engine");
        return MMK_E_SHAPE;
    }
    if (e->persistent.fn) return e->persistent.fn(reinterpret_cast<cudaStream_t>(stream));
    if (e->prologue && !e->prologue_done) {
        const int rc = e->prologue(reinterpret_cast<cudaStream_t>(stream));
        if (rc) return rc;
        e->prologue_done = true;
    }
    cudaError_t ce = cudaGraphLaunch(e->exec, reinterpret_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return mmk_host::cuda_status(ce, "cudaGraphLaunch");
    return MMK_OK;
}

extern "C" void mmk_engine_destroy(void* eng) {
    Engine* e = reinterpret_cast<Engine*>(eng);
    if (!e) return;
    if (e->exec) cudaGraphExecDestroy(e->exec);
    if (e->graph) cudaGraphDestroy(e->graph);
    if (e->cap) cudaStreamDestroy(e->cap);
    if (e->persistent.scratch) mmk_small::scratch_give(e->persistent.scratch);
    delete e;
}

static size_t esize(int dtype) { return dtype == MMK_F32 ? 4 : 8; }

extern "C" int mmk_nnmf_engine_create(int dtype, const void* X, int64_t ldx, void* VA, void* WA,
                                      void* VB, void* WB, int64_t m, int64_t n, int64_t r,
                                      void* ws, size_t ws_bytes, double* red, void* comm,
                                      const mmk_stop_rule* rule, double* trace, int64_t* tstamp,
                                      int64_t* ctl, int64_t* err_dev, void** engine) {
    MMK_NVTX("mmk_nnmf_engine_create");
    if (!comm && mmk_small::nnmf_eligible(dtype, m, n, r, ldx)) {
        // small problems: the whole loop in one persistent kernel per batch
        Engine* e = new Engine();
        int rc = mmk_small::nnmf_prepare(dtype, X, ldx, VA, WA, VB, WB, m, n, (int)r, rule, trace,
                                         tstamp, ctl, err_dev, &e->persistent);
        if (rc) {
            delete e;
            *engine = nullptr;
            return rc;
        }
        *engine = e;
        return MMK_OK;
    }
    double* f_dev = reinterpret_cast<double*>(ctl + MMK_CTL_FCUR);
    const int64_t rl = mmk_nnmf_reduce_len(n, r);
    auto iter = [=](cudaStream_t s, int dir) -> int {
        mmk_host::NoFlag one_gpu(comm == nullptr);   // error flag only around a collective
        void *Vi = dir ? VB : VA, *Vo = dir ? VA : VB, *Wi = dir ? WB : WA, *Wo = dir ? WA : WB;
        int rc = mmk_nnmf_iter_a(dtype, X, ldx, Vi, Wi, Vo, m, n, r, ws, ws_bytes, red, err_dev, s);
        if (rc) return rc;
        if (comm) {
            rc = mmk_allreduce_f64(red, rl, comm, s);
            if (rc) return rc;
        }
        return mmk_nnmf_iter_b(dtype, Wi, Wo, n, r, red, f_dev, err_dev, s);
    };
    // tensor-core path: the per-X preparation runs once (engine prologue, on
    // the run's stream) instead of as a key check in every captured iteration
    // and the W half of a pass that only needs its objective (the iteration
    // cap, ctl[MMK_CTL_LAST] set by the control kernel) exits at launch
    void* tcws = mmk_tc::engine_tc_ws(dtype, X, ldx, m, n, r, ws);
    if (tcws) {
        mmk_tc::set_x_prepared(true);
        mmk_tc::set_last_flag(ctl + MMK_CTL_LAST);
    }
    const int rc = build(iter, rule, trace, tstamp, ctl, err_dev, engine);
    mmk_tc::set_x_prepared(false);
    mmk_tc::set_last_flag(nullptr);
    if (rc == MMK_OK && tcws) {
        const float* Xf = reinterpret_cast<const float*>(X);
        reinterpret_cast<Engine*>(*engine)->prologue = [=](cudaStream_t s) {
            return mmk_tc::prepare_x(Xf, ldx, m, n, tcws, s);
        };
    }
    return rc;
}

extern "C" int mmk_pet_engine_create(int dtype, const void* E, int64_t lde, const void* y,
                                     void* lamA, void* lamB, int64_t d, int64_t p,
                                     const int32_t* nbr_ptr, const int32_t* nbr_idx, double mu,
                                     void* ws, size_t ws_bytes, double* red, void* comm,
                                     const mmk_stop_rule* rule, double* trace, int64_t* tstamp,
                                     int64_t* ctl, int64_t* err_dev, void** engine) {
    MMK_NVTX("mmk_pet_engine_create");
    double* f_dev = reinterpret_cast<double*>(ctl + MMK_CTL_FCUR);
    const int64_t rl = mmk_pet_reduce_len(p);
    auto iter = [=](cudaStream_t s, int dir) -> int {
        mmk_host::NoFlag one_gpu(comm == nullptr);   // error flag only around a collective
        void *Li = dir ? lamB : lamA, *Lo = dir ? lamA : lamB;
        int rc = mmk_pet_iter_a(dtype, E, lde, y, Li, d, p, ws, ws_bytes, red, err_dev, s);
        if (rc) return rc;
        if (comm) {
            rc = mmk_allreduce_f64(red, rl, comm, s);
            if (rc) return rc;
        }
        return mmk_pet_iter_b(dtype, Li, Lo, p, nbr_ptr, nbr_idx, mu,
                              MMK_PET_UPDATE | MMK_PET_OBJECTIVE, red, ws, ws_bytes, f_dev,
                              err_dev, s);
    };
    return build(iter, rule, trace, tstamp, ctl, err_dev, engine);
}

extern "C" int mmk_mds_engine_create(int dtype, const void* Y, const void* Wt, int64_t ldy,
                                     const double* wsum, void* thetaA, void* thetaB,
                                     void* local_out, void* gathered, int64_t dim, int64_t n,
                                     int64_t row0, int64_t rows, int64_t rows_pad, void* ws,
                                     size_t ws_bytes, void* comm, const mmk_stop_rule* rule,
                                     double* trace, int64_t* tstamp, int64_t* ctl,
                                     int64_t* err_dev, void** engine) {
    MMK_NVTX("mmk_mds_engine_create");
    if (!comm && row0 == 0 && rows == n && mmk_small::mds_eligible(dtype, n, dim, Wt != nullptr)) {
        // small problems: the whole loop in one persistent kernel per batch
        Engine* e = new Engine();
        int rc = mmk_small::mds_prepare(dtype, Y, Wt, ldy, wsum, thetaA, thetaB, dim, n, rule,
                                        trace, tstamp, ctl, err_dev, &e->persistent);
        if (rc) {
            delete e;
            *engine = nullptr;
            return rc;
        }
        *engine = e;
        return MMK_OK;
    }
    double* f_dev = reinterpret_cast<double*>(ctl + MMK_CTL_FCUR);
    auto iter = [=](cudaStream_t s, int dir) -> int {
        mmk_host::NoFlag one_gpu(comm == nullptr);   // error flag only around a collective
        void *Ti = dir ? thetaB : thetaA, *To = dir ? thetaA : thetaB;
        if (!comm) {
            return mmk_mds_iter(dtype, Y, Wt, ldy, wsum, Ti, To, n, dim, n, 0, n,
                                MMK_MDS_UPDATE | MMK_MDS_OBJECTIVE, ws, ws_bytes, f_dev, err_dev,
                                s);
        }
        // sharded: own rows -> local_out [dim x rows_pad]; all-gather into
        // gathered [rank][dim][rows_pad]; unpack to the output slot [dim x n];
        // the stress partial is all-reduced in place
        int rc = mmk_mds_iter(dtype, Y, Wt, ldy, wsum, Ti, local_out, rows_pad, dim, n, row0,
                              rows, MMK_MDS_UPDATE | MMK_MDS_OBJECTIVE, ws, ws_bytes, f_dev,
                              err_dev, s);
        if (rc) return rc;
        rc = mmk_allreduce_f64(f_dev, 1, comm, s);
        if (rc) return rc;
        rc = mmk_allgather(local_out, gathered, dim * rows_pad, dtype, comm, s);
        if (rc) return rc;
        return mmk_mds_unpack(dtype, gathered, To, dim, n, rows_pad, s);
    };
    return build(iter, rule, trace, tstamp, ctl, err_dev, engine);
}

extern "C" int mmk_mds_tri_engine_create(const float* packed, int64_t t0, int64_t t1,
                                         float* thetaA, float* thetaB, int64_t dim, int64_t n,
                                         void* ws, size_t ws_bytes, double* red, void* comm,
                                         const mmk_stop_rule* rule, double* trace,
                                         int64_t* tstamp, int64_t* ctl, int64_t* err_dev,
                                         void** engine) {
    MMK_NVTX("mmk_mds_tri_engine_create");
    double* f_dev = reinterpret_cast<double*>(ctl + MMK_CTL_FCUR);
    const int64_t rl = mmk_mds_tri_reduce_len(n, dim);
    auto iter = [=](cudaStream_t s, int dir) -> int {
        mmk_host::NoFlag one_gpu(comm == nullptr);   // error flag only around a collective
        float *Ti = dir ? thetaB : thetaA, *To = dir ? thetaA : thetaB;
        int rc = mmk_mds_tri_iter_a(packed, t0, t1, Ti, dim, n, ws, ws_bytes, red, err_dev, s);
        if (rc) return rc;
        if (comm) {
            rc = mmk_allreduce_f64(red, rl, comm, s);
            if (rc) return rc;
        }
        return mmk_mds_tri_iter_b(Ti, To, dim, n, red, f_dev, err_dev, s);
    };
    return build(iter, rule, trace, tstamp, ctl, err_dev, engine);
}

extern "C" int mmk_nnmf_poisson_engine_create(int dtype, const void* X, int64_t ldx, void* VA,
                                              void* WA, void* VB, void* WB, int64_t m, int64_t n,
                                              int64_t r, void* ws, size_t ws_bytes, double* red,
                                              void* comm, const mmk_stop_rule* rule,
                                              double* trace, int64_t* tstamp, int64_t* ctl,
                                              int64_t* err_dev, void** engine) {
    MMK_NVTX("mmk_nnmf_poisson_engine_create");
    if (!comm && mmk_small::nnmf_eligible(dtype, m, n, r, ldx)) {
        Engine* e = new Engine();
        int rc = mmk_small::nnmf_prepare(dtype, X, ldx, VA, WA, VB, WB, m, n, (int)r, rule, trace,
                                         tstamp, ctl, err_dev, &e->persistent, true);
        if (rc) {
            delete e;
            *engine = nullptr;
            return rc;
        }
        *engine = e;
        return MMK_OK;
    }
    double* f_dev = reinterpret_cast<double*>(ctl + MMK_CTL_FCUR);
    const int64_t rl = mmk_nnmf_poisson_reduce_len(n, r);
    auto iter = [=](cudaStream_t s, int dir) -> int {
        mmk_host::NoFlag one_gpu(comm == nullptr);   // error flag only around a collective
        void *Vi = dir ? VB : VA, *Vo = dir ? VA : VB, *Wi = dir ? WB : WA, *Wo = dir ? WA : WB;
        int rc = mmk_nnmf_poisson_iter_a(dtype, X, ldx, Vi, Wi, Vo, m, n, r, ws, ws_bytes, red,
                                         err_dev, s);
        if (rc) return rc;
        if (comm) {
            rc = mmk_allreduce_f64(red, rl, comm, s);
            if (rc) return rc;
        }
        return mmk_nnmf_poisson_iter_b(dtype, Wi, Wo, n, r, red, f_dev, err_dev, s);
    };
    return build(iter, rule, trace, tstamp, ctl, err_dev, engine);
}

extern "C" int mmk_pet_sparse_engine_create(int dtype, const int32_t* rptr, const int32_t* ridx,
                                            const void* rval, const int32_t* cptr,
                                            const int32_t* cidx, const void* cval, const void* y,
                                            void* lamA, void* lamB, int64_t d, int64_t p,
                                            const int32_t* nbr_ptr, const int32_t* nbr_idx,
                                            double mu, void* ws, size_t ws_bytes, double* red,
                                            void* comm, const mmk_stop_rule* rule, double* trace,
                                            int64_t* tstamp, int64_t* ctl, int64_t* err_dev,
                                            void** engine) {
    MMK_NVTX("mmk_pet_sparse_engine_create");
    if (!comm && mmk_small::pet_eligible(dtype, d, p)) {
        // small problems: the whole loop in one persistent kernel per batch
        Engine* e = new Engine();
        int rc = mmk_small::pet_prepare(dtype, rptr, ridx, rval, cptr, cidx, cval, y, lamA, lamB,
                                        d, p, nbr_ptr, nbr_idx, mu, rule, trace, tstamp, ctl,
                                        err_dev, &e->persistent);
        if (rc) {
            delete e;
            *engine = nullptr;
            return rc;
        }
        *engine = e;
        return MMK_OK;
    }
    double* f_dev = reinterpret_cast<double*>(ctl + MMK_CTL_FCUR);
    const int64_t rl = mmk_pet_reduce_len(p);
    auto iter = [=](cudaStream_t s, int dir) -> int {
        mmk_host::NoFlag one_gpu(comm == nullptr);   // error flag only around a collective
        void *Li = dir ? lamB : lamA, *Lo = dir ? lamA : lamB;
        if (!comm)   // one GPU: fused back-projection + pixel update
            return mmk_pet_sparse_iter(dtype, rptr, ridx, rval, cptr, cidx, cval, y, Li, Lo, d,
                                       p, nbr_ptr, nbr_idx, mu,
                                       MMK_PET_UPDATE | MMK_PET_OBJECTIVE, ws, ws_bytes, red,
                                       f_dev, err_dev, s);
        int rc = mmk_pet_sparse_iter_a(dtype, rptr, ridx, rval, cptr, cidx, cval, y, Li, d, p,
                                       ws, ws_bytes, red, err_dev, s);
        if (rc) return rc;
        if (comm) {
            rc = mmk_allreduce_f64(red, rl, comm, s);
            if (rc) return rc;
        }
        return mmk_pet_iter_b(dtype, Li, Lo, p, nbr_ptr, nbr_idx, mu,
                              MMK_PET_UPDATE | MMK_PET_OBJECTIVE, red, ws, ws_bytes, f_dev,
                              err_dev, s);
    };
    return build(iter, rule, trace, tstamp, ctl, err_dev, engine);
}

namespace mmk_small {

namespace {
struct Pooled {
    void* p;
    size_t bytes;
};
std::mutex g_pool_mu;
std::vector<Pooled> g_free, g_live;
constexpr size_t kPoolKeep = 8;
}  // namespace

void* scratch_take(size_t bytes, size_t zero_bytes) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    void* p = nullptr;
    size_t got = 0;
    for (size_t i = 0; i < g_free.size(); ++i) {
        if (g_free[i].bytes >= bytes) {
            p = g_free[i].p;
            got = g_free[i].bytes;
            g_free.erase(g_free.begin() + i);
            break;
        }
    }
    if (!p) {
        if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
        got = bytes;
    }
    g_live.push_back({p, got});
    if (zero_bytes) {
        // barrier slots must read 0 before the first launch on any stream
        cudaMemset(p, 0, zero_bytes);
        cudaDeviceSynchronize();
    }
    return p;
}

void scratch_give(void* p) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (size_t i = 0; i < g_live.size(); ++i) {
        if (g_live[i].p == p) {
            g_free.push_back(g_live[i]);
            g_live.erase(g_live.begin() + i);
            break;
        }
    }
    while (g_free.size() > kPoolKeep) {
        cudaFree(g_free.front().p);
        g_free.erase(g_free.begin());
    }
}

}  // namespace mmk_small
