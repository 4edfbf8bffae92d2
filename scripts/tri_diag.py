import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np
import golden_io as G
import paper_1003_3272_b200 as M
from oracle import oracle as O
from test_mds_tri_gpu import sym_diss
TRI = M.Backend(dtype="fp32", mds_kernel="tri"); ROWS = M.Backend(dtype="fp32", mds_kernel="rows")
for n, dim in [(300, 1), (300, 2)]:
    y = sym_diss(n, n + dim, dim)
    theta0 = G.f32(np.random.default_rng(7).uniform(-1, 1, size=(dim, n)))
    prob = M.MdsProblem(weights=1.0 - np.eye(n), dissimilarities=y, p=dim)
    md = O.MdsData(1.0 - np.eye(n), y, dim)
    for it in [0, 10, 30, 59]:
        th, _ = M.mds_run(prob, M.MmConfig(max_iters=max(it, 1), epsilon=1e-300), M.Backend(dtype="fp64"), theta0=theta0) if it else (theta0, None)
        th = G.f32(th)
        want = O.mds_update(th, md); fs = O.mds_stress(th, md)
        a = M.mds_update(th, prob, TRI); b = M.mds_update(th, prob, ROWS)
        sa = M.stress(th, prob, TRI); sb = M.stress(th, prob, ROWS)
        ea = np.abs(a - want).ravel(); eb = np.abs(b - want).ravel()
        k = int(np.argmax(ea))
        print(n, dim, it, "tri", G.rel(a, want), abs(sa - fs) / fs, "rows", G.rel(b, want), abs(sb - fs) / fs, "worst pt", k, ea[k], eb[k])
