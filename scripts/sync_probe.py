"""One small tensor-core NNMF run at rank R (env), for compute-sanitizer probes."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import paper_1003_3272_b200 as M
r = int(os.environ.get("R", 64))
rng = np.random.default_rng(0)
x = rng.random((520, 392)).astype(np.float32)
st = M.FactorPair(rng.random((520, r)).astype(np.float32), rng.random((r, 392)).astype(np.float32))
M.nnmf_run(M.NnmfProblem(x=x, rank=r), M.MmConfig(max_iters=2, epsilon=1e-300),
           M.Backend(dtype="fp32", fused=False), state0=st)
print("probe done", r)
