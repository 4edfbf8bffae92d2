// mmk_abi.cu -- library-wide ABI plumbing: version, thread-local error text.
#include <stdarg.h>
#include <stdio.h>

#include "mmk_common.cuh"

static thread_local char g_err[512] = "";

namespace mmk_host {
void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
int cuda_status(cudaError_t e, const char* what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return MMK_E_CUDA;
}
}  // namespace mmk_host

namespace {
// The flag rides in the all-reduced payload (summed over ranks): 1 for an
// objective-class error, 2^-10 for an update-only one (mmk_common.cuh), so
// the sum tells every rank whether any error is of the objective class.
__global__ void err_flag_kernel(const int64_t* err, double* flag) {
    double v = 0.0;
    if (err != nullptr && err[0] != 0) v = mmk::err_update_only(err[1]) ? 1.0 / 1024.0 : 1.0;
    *flag = v;
}
__global__ void peer_err_kernel(const double* flag, int64_t* err) {
    if (*flag > 0.0 && err[0] == 0) {
        err[0] = MMK_E_PEER;
        // objective class: the index stays at its reset value; update-only:
        // an update-class site, so this rank's stopping rule defers it too
        if (*flag < 0.5) err[1] = (int64_t)mmk::kUpdateSite << 48;
    }
}
}  // namespace

static thread_local bool t_no_flag = false;

namespace mmk_host {
NoFlag::NoFlag(bool active) : prev(t_no_flag) {
    if (active) t_no_flag = true;
}
NoFlag::~NoFlag() { t_no_flag = prev; }
void err_flag(const int64_t* err, double* flag, cudaStream_t st) {
    if (t_no_flag) return;
    MMK_LAUNCH("mmk_err_flag", st, (err_flag_kernel<<<1, 1, 0, st>>>(err, flag)));
}
void peer_err(const double* flag, int64_t* err, cudaStream_t st) {
    if (t_no_flag || err == nullptr) return;
    MMK_LAUNCH("mmk_peer_err", st, (peer_err_kernel<<<1, 1, 0, st>>>(flag, err)));
}
}  // namespace mmk_host

// ---- opt-in launch profiler --------------------------------------------------
// Off by default.  When enabled (bench.py), every kernel launch site brackets
// its launch with CUDA events recorded on the launch stream; mmk_prof_report
// synchronises those events and returns per-kernel launch counts and total
// device milliseconds.  Not used while a graph is being captured.
#include <mutex>
#include <string>
#include <vector>

namespace {
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_pool;   // recycled events (no create/destroy per launch)

cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

namespace mmk_host {
bool first_on_device(const void* key) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> seen;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : seen)
        if (e.first == key && e.second == dev) return false;
    seen.emplace_back(key, dev);
    return true;
}
bool prof_on() { return g_prof_on; }
void prof_start(const char* name, cudaStream_t s) {
    if (!g_prof_on) return;
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    ProfRec r{name, take_event(), take_event()};
    cudaEventRecord(r.a, s);
    g_prof.push_back(r);
}
void prof_stop(cudaStream_t s) {
    if (!g_prof_on) return;
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof.empty()) cudaEventRecord(g_prof.back().b, s);
}
}  // namespace mmk_host

extern "C" int mmk_prof_enable(int on) {
    g_prof_on = on != 0;
    return MMK_OK;
}

extern "C" int mmk_prof_report(char* buf, size_t len) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    std::vector<std::pair<std::string, std::pair<long long, double>>> agg;
    for (ProfRec& r : g_prof) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        bool found = false;
        for (auto& kv : agg)
            if (kv.first == r.name) {
                kv.second.first += 1;
                kv.second.second += ms;
                found = true;
            }
        if (!found) agg.push_back({r.name, {1, (double)ms}});
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_prof.clear();
    std::string out;
    for (auto& kv : agg) {
        char line[256];
        snprintf(line, sizeof(line), "%s\t%lld\t%.6f\n", kv.first.c_str(), kv.second.first,
                 kv.second.second);
        out += line;
    }
    if (buf && len) {
        snprintf(buf, len, "%s", out.c_str());
    }
    return (int)out.size();
}

extern "C" int mmk_abi_version(void) { return MMK_ABI_VERSION; }
extern "C" const char* mmk_last_error(void) { return g_err; }
