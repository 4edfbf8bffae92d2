"""Per-kernel times of the tensor-core NNMF iteration at C4 (library launch
profiler: CUDA events around every launch), no result checks -- for A/B of
kernel variants (scripts/tc_variants.sh) including ones whose results are
wrong by construction."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import test_nnmf_tc_gpu as T
from paper_1003_3272_b200 import _lib

m, n = int(os.environ.get("M", 131072)), int(os.environ.get("N", 16384))
r = int(os.environ.get("R", 64))
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(m, n, device="cuda", generator=g)
v = torch.rand(m, r, device="cuda", generator=g)
w = torch.rand(r, n, device="cuda", generator=g)
for _ in range(2):
    T.one_iter(x, v, w, False)
torch.cuda.synchronize()
lib = _lib.load()
lib.mmk_prof_enable(1)
for _ in range(int(os.environ.get("ITERS", 8))):
    T.one_iter(x, v, w, False)
torch.cuda.synchronize()
lib.mmk_prof_enable(0)
rep = _lib.prof_report()
for k in sorted(rep, key=lambda k: -rep[k][1]):
    cnt, ms = rep[k]
    if os.environ.get("ALL") or k in ("nnmf_vstep_tc", "nnmf_wstep_tc"):
        print(os.environ.get("TAG", ""), os.environ.get("MMK_TC_PAIR", ""), f"r={r}", k,
              "avg_ms %.4f" % (ms / cnt))
