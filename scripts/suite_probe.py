"""Per-kernel device times of the paper-shape workloads (C1 NNMF, C2 PET, C3 MDS)
through the per-iteration path with the launch profiler, plus the fused-engine
time per iteration."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib, datasets as D
be = M.Backend(dtype="fp32", fused=False)
bef = M.Backend(dtype="fp32")
x = np.random.default_rng(0).random((2429, 361)).astype(np.float32).astype(np.float64)
g = np.random.default_rng(1)
s0 = M.FactorPair(g.random((2429, 10)), g.random((10, 361)))
e = D.build_system_matrix(D.PetGeometry(64, 64))
y = D.simulate_counts(D.default_phantom(64), e, 20260811)
pp = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=D.build_neighborhoods(64))
diss = D.votes_to_dissimilarity(D.synthetic_votes(401, 671, 0))
mp_ = M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=3)
th0 = np.random.default_rng(1).uniform(-1, 1, size=(3, 401))
runs = {
  "nnmf-c1": lambda b, k: M.nnmf_run(M.NnmfProblem(x=x, rank=10), M.MmConfig(max_iters=k, epsilon=1e-300, monotone_tol=1e-6), b, state0=s0),
  "pet-c2": lambda b, k: M.pet_run(pp, M.MmConfig(max_iters=k, epsilon=1e-300, monotone_tol=1e-6), b),
  "mds-c3": lambda b, k: M.mds_run(mp_, M.MmConfig(max_iters=k, epsilon=1e-300, monotone_tol=1e-6), b, theta0=th0),
}
lib = _lib.load()
for name, fn in runs.items():
    fn(be, 5)
    lib.mmk_prof_enable(1); fn(be, 50); torch.cuda.synchronize(); lib.mmk_prof_enable(0)
    prof = _lib.prof_report()
    fn(bef, 1000); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(bef, 1000); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name}: fused {1e6*dt/1000:.1f} us/iter; kernels (per-iteration path):")
    for k, (c, ms) in prof.items(): print(f"   {k:22s} {c/51:5.1f}/it {1000*ms/c:8.2f} us")
