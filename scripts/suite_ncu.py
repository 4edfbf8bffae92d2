import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import datasets as D
bef = M.Backend(dtype="fp32", fused=False)
x = np.random.default_rng(0).random((2429, 361)).astype(np.float32).astype(np.float64)
g = np.random.default_rng(1)
s0 = M.FactorPair(g.random((2429, 10)), g.random((10, 361)))
e = D.build_system_matrix(D.PetGeometry(64, 64))
y = D.simulate_counts(D.default_phantom(64), e, 20260811)
pp = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=D.build_neighborhoods(64))
diss = D.votes_to_dissimilarity(D.synthetic_votes(401, 671, 0))
mp_ = M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=3)
th0 = np.random.default_rng(1).uniform(-1, 1, size=(3, 401))
cfg = M.MmConfig(max_iters=20, epsilon=1e-300, monotone_tol=1e-6)
M.nnmf_run(M.NnmfProblem(x=x, rank=10), cfg, bef, state0=s0)
M.pet_run(pp, cfg, bef)
M.mds_run(mp_, cfg, bef, theta0=th0)
torch.cuda.synchronize()
