import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import Backend, MmConfig
rng = np.random.default_rng(0)
xt = rng.random((520, 392)).astype(np.float32).astype(np.float64)
st0 = M.FactorPair(rng.random((520, 64)), rng.random((64, 392)))
cfg = MmConfig(max_iters=3, epsilon=1e-300, monotone_tol=1e-6)
M.nnmf_run(M.NnmfProblem(x=xt, rank=64), cfg, Backend(dtype="fp32", fused=sys.argv[1] == "1"), state0=st0)
print("ok")
