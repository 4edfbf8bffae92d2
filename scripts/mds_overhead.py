"""Fixed per-run cost of mds_run on the packed C5 problem (n = 65536, dim 3):
event time of runs of K = 1, 5, 20 iterations with the tiles resident in HBM."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import datasets as D
from paper_1003_3272_b200.mds import PackedMdsProblem
n, dim = 65536, 3
be = M.Backend(dtype="fp32", device=0)
prob = PackedMdsProblem.from_rows(D.distance_rows(n, seed=0), n, dim, be)
theta0 = np.random.default_rng(0).uniform(-1, 1, size=(dim, n))
def run(k):
    return M.mds_run(prob, M.MmConfig(max_iters=k, epsilon=1e-300), be, theta0=theta0)
run(3)
for k in (1, 5, 20):
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); run(k); e.record(); torch.cuda.synchronize()
    print(f"K={k:3d} event_ms={s.elapsed_time(e):8.2f}")
