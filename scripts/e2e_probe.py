"""Break the nnmf-large e2e run into phases (upload, setup, engine build, device loop, readback)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _arrays as A, _lib
from paper_1003_3272_b200.nnmf import _GpuNnmf
from paper_1003_3272_b200.driver import run_mm

m, n, r = 131072, 16384, 64
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(1)
x = torch.rand((m, n), device=dev, generator=g)
xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True); xh.copy_(x)
v0 = torch.rand((m, r), device=dev, generator=g).cpu().pin_memory()
w0 = torch.rand((r, n), device=dev, generator=g).cpu().pin_memory()
del x; torch.cuda.empty_cache()

# raw H2D bandwidth
xd = torch.empty((m, n), device=dev)
for k in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    xd.copy_(xh, non_blocking=True); torch.cuda.synchronize()
    print(f"raw H2D single copy: {xh.numel()*4/(time.perf_counter()-t0)/1e9:.1f} GB/s")
ss = [torch.cuda.Stream() for _ in range(4)]
rows = m // 16
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(16):
    with torch.cuda.stream(ss[i % 4]):
        xd[i*rows:(i+1)*rows].copy_(xh[i*rows:(i+1)*rows], non_blocking=True)
torch.cuda.synchronize()
print(f"raw H2D 16 chunks / 4 streams: {xh.numel()*4/(time.perf_counter()-t0)/1e9:.1f} GB/s")
del xd; torch.cuda.empty_cache()

be = M.Backend(dtype="fp32")
orig = _GpuNnmf._engine_create
def timed_create(self, *a):
    torch.cuda.synchronize(); t = time.perf_counter()
    orig(self, *a)
    torch.cuda.synchronize(); print(f"   engine_create {1e3*(time.perf_counter()-t):.1f} ms")
_GpuNnmf._engine_create = timed_create
for rep in range(2):
    prob = M.NnmfProblem(x=xh, rank=r)
    cfg = M.MmConfig(max_iters=100, epsilon=1e-300, monotone_tol=1e-6)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    xd = prob.device_x(be, torch); torch.cuda.synchronize(); t1 = time.perf_counter()
    tt = [time.perf_counter()]
    mm = _GpuNnmf(prob, be); torch.cuda.synchronize(); t2 = time.perf_counter()
    s0 = mm.device_state(M.FactorPair(v0, w0)); torch.cuda.synchronize(); t3 = time.perf_counter()
    st, tr = run_mm(mm, s0, cfg); torch.cuda.synchronize(); t4 = time.perf_counter()
    v = A.to_user(st.v, v0); w = A.to_user(st.w, w0); t5 = time.perf_counter()
    print(f"rep {rep}: upload {1e3*(t1-t0):.1f} ms ({xh.numel()*4/(t1-t0)/1e9:.1f} GB/s), "
          f"setup {1e3*(t2-t1):.1f}, state {1e3*(t3-t2):.1f}, run_mm {1e3*(t4-t3):.1f} "
          f"({tr.iters} it; device trace {1e3*tr.cumulative_seconds[-1]:.1f} ms), readback {1e3*(t5-t4):.1f}; "
          f"total {1e3*(t5-t0):.1f} ms -> {tr.iters/(t5-t0):.1f} it/s")
    del xd, mm, s0, st, prob
    torch.cuda.empty_cache()

# inside _run_fused
import paper_1003_3272_b200._engine as E
src = open(E.__file__).read()
marks = []
def mark(tag):
    torch.cuda.synchronize(); marks.append((tag, time.perf_counter()))
E.mark = mark
code = src[src.index("    def _run_fused"):src.index("        return final, trace_obj")] + "        return final, trace_obj\n"
code = code.replace("        a = self._alloc_like(state0)", "        mark('start')\n        a = self._alloc_like(state0)")
code = code.replace("        eng = ctypes.c_void_p()", "        mark('allocs')\n        eng = ctypes.c_void_p()")
code = code.replace("        values, stamps = [], []", "        mark('engine')\n        values, stamps = [], []")
code = code.replace("                if reason:\n                    break", "                mark('batch')\n                if reason:\n                    break")
code = code.replace("        it = len(values) - 1", "        mark('destroyed')\n        it = len(values) - 1")
ns = {}
exec("import ctypes, math, time\nimport numpy as np\nfrom paper_1003_3272_b200._engine import *\nfrom paper_1003_3272_b200._engine import _as_f64, StopRule\nfrom paper_1003_3272_b200 import _lib\nfrom paper_1003_3272_b200.errors import *\nclass X:\n" + code, {**E.__dict__, 'mark': mark}, ns)
E.DeviceMm._run_fused = ns['X']._run_fused
prob = M.NnmfProblem(x=xh, rank=r)
cfg = M.MmConfig(max_iters=100, epsilon=1e-300, monotone_tol=1e-6)
xd = prob.device_x(be, torch)
mm = _GpuNnmf(prob, be)
mm.run_fused = mm._run_fused
s0 = mm.device_state(M.FactorPair(v0, w0))
for rep in range(2):
    marks.clear()
    st, tr = run_mm(mm, s0, cfg)
    t0 = marks[0][1]
    print("run_fused marks:", ", ".join(f"{k} {1e3*(t-t0):.1f}" for k, t in marks))
torch.cuda.synchronize(); t = time.perf_counter(); v = A.to_user(st.v, v0); print(f"to_user V {1e3*(time.perf_counter()-t):.1f} ms")
hb = torch.empty(st.v.shape, dtype=st.v.dtype, pin_memory=True)
torch.cuda.synchronize(); t = time.perf_counter(); hb.copy_(st.v); vv = hb.numpy().astype("float64"); print(f"pinned copy + astype {1e3*(time.perf_counter()-t):.1f} ms")

# setup pieces
prob = M.NnmfProblem(x=xh, rank=r)
xd = prob.device_x(be, torch); torch.cuda.synchronize()
for what, fn in [("ws zeros", lambda: torch.zeros(_lib.ws_bytes("mmk_nnmf_ws_bytes", 0, m, n, r), dtype=torch.uint8, device=dev)),
                 ("status", lambda: _lib.StatusBlock(torch, dev)),
                 ("GpuNnmf", lambda: _GpuNnmf(prob, be))]:
    for k in range(2):
        torch.cuda.synchronize(); t = time.perf_counter(); o = fn(); torch.cuda.synchronize()
        print(f"   {what}: {1e3*(time.perf_counter()-t):.2f} ms"); del o
