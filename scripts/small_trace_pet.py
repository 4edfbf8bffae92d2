"""Phase stamps (clock64, CTA 0) of the persistent PET kernel at C2."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
dbg = torch.zeros(64 * 12, dtype=torch.int64, device="cuda")
os.environ["MMK_SMALL_TRACE"] = str(dbg.data_ptr())
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import datasets as D
e = D.build_system_matrix(D.PetGeometry(64, 64))
y = D.simulate_counts(D.default_phantom(64), e, 20260811)
pp = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=D.build_neighborhoods(64))
M.pet_run(pp, M.MmConfig(max_iters=40, epsilon=1e-300, monotone_tol=1e-6), M.Backend(dtype="fp32"))
torch.cuda.synchronize()
d = dbg.cpu().numpy().reshape(64, 12)[5:35, :8]
names = ["stage lam", "rays", "B1", "stage ratio", "pixels", "B2", "f + rule"]
med = np.median(np.diff(d, axis=1), axis=0)
print("median cycles:", dict(zip(names, med.astype(int))), "total", int(np.median(d[1:, 0] - d[:-1, 0])))
