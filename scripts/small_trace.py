"""Phase timestamps (clock64, CTA 0) of the persistent NNMF kernel at C1."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
dbg = torch.zeros(64 * 12, dtype=torch.int64, device="cuda")
os.environ["MMK_SMALL_TRACE"] = str(dbg.data_ptr())
import paper_1003_3272_b200 as M
x = np.random.default_rng(0).random((2429, 361)).astype(np.float32).astype(np.float64)
g = np.random.default_rng(1)
s0 = M.FactorPair(g.random((2429, 10)), g.random((10, 361)))
cfg = M.MmConfig(max_iters=40, epsilon=1e-300, monotone_tol=1e-6)
M.nnmf_run(M.NnmfProblem(x=x, rank=10), cfg, M.Backend(dtype="fp32"), state0=s0)
torch.cuda.synchronize()
d = dbg.cpu().numpy().reshape(64, 12)[5:35]
d = d[:, [0, 1, 2, 3, 4, 5, 6, 8, 9, 10, 7]]
names = ["Gw", "rows", "partials", "B1", "P2", "B2", "decision", "Pt load", "Gv", "W update"]
med = np.median(np.diff(d, axis=1), axis=0)
print("median cycles per phase:", dict(zip(names, med.astype(int))), "total", int(np.median(d[1:, 0] - d[:-1, 0])))
