import sys, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import datasets as D
e = D.build_system_matrix(D.PetGeometry(64, 64))
y = D.simulate_counts(D.default_phantom(64), e, 20260811)
pp = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=D.build_neighborhoods(64))
be = M.Backend(dtype="fp32")
cfg = M.MmConfig(max_iters=10, epsilon=1e-300, monotone_tol=1e-6)
M.pet_run(pp, cfg, be); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(5): M.pet_run(pp, cfg, be)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
