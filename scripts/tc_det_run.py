"""Run-to-run determinism of nnmf_run (fused engine / per-iteration) at C4."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_1003_3272_b200 as M

m, n, r = int(sys.argv[1]), int(sys.argv[2]), 64
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(m, n, device="cuda", generator=g)
v0 = torch.rand(m, r, device="cuda", generator=g)
w0 = torch.rand(r, n, device="cuda", generator=g)
prob = M.NnmfProblem(x=x, rank=r)
cfg = M.MmConfig(max_iters=20, epsilon=1e-300, monotone_tol=1e-6)
for fused in (True, False):
    runs = [M.nnmf_run(prob, cfg, M.Backend(dtype="fp32", device=0, fused=fused), state0=M.FactorPair(v0, w0)) for _ in range(3)]
    t0 = runs[0][1].objective_values
    for s, t in runs[1:]:
        d = np.nonzero(t.objective_values != t0)[0]
        print("fused", fused, "differ at", d[:10], "max rel", np.max(np.abs(t.objective_values - t0) / t0),
              "V eq", torch.equal(s.v, runs[0][0].v))
