"""C4 end-to-end probe: nnmf_run on a pinned host X split into its phases
(upload of X, solver object incl. workspace, fused device loop), synchronised
between phases.  MMK_TC_PRESPLIT=0/1 selects the kernels."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import nnmf as N
from paper_1003_3272_b200.driver import run_mm
m, n, r = 131072, 16384, 64
g = torch.Generator(device="cuda").manual_seed(0)
xd = torch.rand(m, n, device="cuda", generator=g)
xh = torch.empty(m, n, pin_memory=True); xh.copy_(xd); del xd
vh = torch.rand(m, r, generator=torch.Generator().manual_seed(1)).pin_memory()
wh = torch.rand(r, n, generator=torch.Generator().manual_seed(2)).pin_memory()
prob = M.NnmfProblem(x=xh, rank=r)
cfg = M.MmConfig(max_iters=100, epsilon=1e-300, monotone_tol=1e-6)
be = M.Backend(dtype="fp32")
for i in range(4):
    prob._dev.clear(); torch.cuda.synchronize()
    t = [time.perf_counter()]
    prob.device_x(be, torch); torch.cuda.synchronize(); t.append(time.perf_counter())
    mm = N._GpuNnmf(prob, be); torch.cuda.synchronize(); t.append(time.perf_counter())
    s0 = mm.device_state(M.FactorPair(vh, wh)); torch.cuda.synchronize(); t.append(time.perf_counter())
    st, tr = run_mm(mm, s0, cfg); torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"run {i}: upload {d[0]:.1f} ms, solver+ws {d[1]:.1f}, state {d[2]:.1f}, loop {d[3]:.1f} "
          f"(iters {1e3 * tr.cumulative_seconds[-1]:.1f}); mem {torch.cuda.memory_reserved() / 2**30:.1f} GiB")
    del st, tr, mm, s0
