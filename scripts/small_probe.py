import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1003_3272_b200 as M
x = np.random.default_rng(0).random((2429, 361)).astype(np.float32).astype(np.float64)
g = np.random.default_rng(1)
s0 = M.FactorPair(g.random((2429, 10)), g.random((10, 361)))
cfg = M.MmConfig(max_iters=200, epsilon=1e-300, monotone_tol=1e-6)
M.nnmf_run(M.NnmfProblem(x=x, rank=10), cfg, M.Backend(dtype="fp32"), state0=s0)
