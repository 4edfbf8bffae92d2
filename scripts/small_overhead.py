import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import datasets as D
e = D.build_system_matrix(D.PetGeometry(64, 64))
y = D.simulate_counts(D.default_phantom(64), e, 20260811)
pp = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=D.build_neighborhoods(64))
x = np.random.default_rng(0).random((2429, 361)).astype(np.float32).astype(np.float64)
g = np.random.default_rng(1)
s0 = M.FactorPair(g.random((2429, 10)), g.random((10, 361)))
nn = M.NnmfProblem(x=x, rank=10)
be = M.Backend(dtype="fp32")
for name, fn in [("pet-c2", lambda k: M.pet_run(pp, M.MmConfig(max_iters=k, epsilon=1e-300, monotone_tol=1e-6), be)),
                 ("nnmf-c1", lambda k: M.nnmf_run(nn, M.MmConfig(max_iters=k, epsilon=1e-300, monotone_tol=1e-6), be, state0=s0))]:
    fn(10)
    for k in (10, 1000, 3000):
        torch.cuda.synchronize(); t = time.perf_counter(); _, tr = fn(k); torch.cuda.synchronize(); dt = time.perf_counter() - t
        dev = tr.cumulative_seconds[-1]
        print(f"{name} {k:5d} it: wall {1e3*dt:8.2f} ms, device loop {1e3*dev:8.2f} ms ({1e6*dev/max(k,1):.2f} us/it), outside {1e3*(dt-dev):.2f} ms")
