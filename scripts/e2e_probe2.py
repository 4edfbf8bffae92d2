"""Mimic bench.py's e2e (device X of the kernel benchmark still resident) and time phases."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _arrays as A
import paper_1003_3272_b200.nnmf as NN

m, n, r = 131072, 16384, 64
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
x = torch.rand((m, n), device=dev, generator=g)
v0 = torch.rand((m, r), device=dev, generator=g)
w0 = torch.rand((r, n), device=dev, generator=g)
xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True); xh.copy_(x)
vh = v0.cpu().pin_memory(); wh = w0.cpu().pin_memory()
be = M.Backend(dtype="fp32")
prob = M.NnmfProblem(x=xh, rank=r)
cfg = M.MmConfig(max_iters=100, epsilon=1e-300, monotone_tol=1e-6)
T = {}
def wrap(obj, name, tag):
    f = getattr(obj, name)
    def w(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter(); out = f(*a, **k); torch.cuda.synchronize()
        T[tag] = T.get(tag, 0) + time.perf_counter() - t
        return out
    setattr(obj, name, w)
wrap(A, "to_device", "to_device")
wrap(A, "to_user", "to_user")
wrap(NN, "run_mm", "run_mm")
for rep in range(3):
    T.clear()
    prob._dev.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st, tr = M.nnmf_run(prob, cfg, be, state0=M.FactorPair(vh, wh))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"rep {rep}: total {1e3*dt:.1f} ms -> {100/dt:.1f} it/s; " + ", ".join(f"{k} {1e3*v:.1f}" for k, v in T.items()))
    del st, tr
