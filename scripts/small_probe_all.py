"""Run each persistent engine once (C1 NNMF, C1 Poisson, C2 PET, C3 MDS) for ncu."""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import datasets as D
import golden_io as G
be = M.Backend(dtype="fp32")
cfg = M.MmConfig(max_iters=200, epsilon=1e-300, monotone_tol=1e-6)
x, v0, w0 = G.c1_inputs()
M.nnmf_run(M.NnmfProblem(x=x, rank=10), cfg, be, state0=M.FactorPair(v0, w0))
xc, c0, d0 = G.poisson_c1_inputs()
M.nnmf_poisson_run(M.NnmfProblem(x=xc, rank=10), cfg, be, state0=M.FactorPair(c0, d0))
e, y, nbrs = G.c2_inputs()
M.pet_run(M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=nbrs), cfg, be)
diss, th0 = G.c3_inputs(3)
M.mds_run(M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=3), cfg, be, theta0=th0)
