"""Fixed per-run cost of nnmf_run at C4: wall/event time of runs of K
iterations (K = 1, 5, 20, 100) on X resident in HBM, and the kernels a
1-iteration run launches (library launch profiler)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib
m, n, r = 131072, 16384, 64
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(1)
x = torch.rand(m, n, generator=g, device=dev)
v0 = torch.rand(m, r, generator=g, device=dev); w0 = torch.rand(r, n, generator=g, device=dev)
be = M.Backend(dtype="fp32", device=0)
prob = M.NnmfProblem(x=x, rank=r)
def run(k):
    cfg = M.MmConfig(max_iters=k, epsilon=1e-300, monotone_tol=1e-6)
    return M.nnmf_run(prob, cfg, be, state0=M.FactorPair(v0, w0))
run(3)
for k in (1, 5, 20, 100):
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); s.record(); st, tr = run(k); e.record(); torch.cuda.synchronize()
    print(f"K={k:4d} event_ms={s.elapsed_time(e):8.2f} wall_ms={1e3*(time.perf_counter()-t0):8.2f} loop_wall_ms={1e3*tr.wall_time:8.2f}")
lib = _lib.load(); _lib.prof_report(); lib.mmk_prof_enable(1)
run(1); torch.cuda.synchronize(); lib.mmk_prof_enable(0)
for k_, (c, ms) in sorted(_lib.prof_report().items(), key=lambda t: -t[1][1]):
    print(f"  {k_:28s} {c:3d} {ms:8.3f} ms")
import torch.profiler as P
with P.profile(activities=[P.ProfilerActivity.CPU, P.ProfilerActivity.CUDA]) as prof:
    run(1); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=12))
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=12))
