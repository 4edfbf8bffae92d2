"""Is the last-CTA arrival counter the cost of pet_sback_pixel at pet-large?
Time the fused phase-B kernel with and without the objective (the arrival)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib
from paper_1003_3272_b200.pet import _GpuPet
side = 256
geo = M.PetGeometry(side, 256)
be = M.Backend(dtype="fp32")
sa = M.system_matrix_device(geo, be)
nb = M.build_neighborhoods(side)
lam_true = torch.ones(side * side, device="cuda")
means = M.SparsePetProblem(sa, np.zeros(geo.n_rays), 0.0, nb).forward(lam_true)
y = torch.poisson(means * 50.0, generator=torch.Generator(device="cuda").manual_seed(1))
mm = _GpuPet(M.SparsePetProblem(sa, y, 1e-6, nb), be)
lam = [torch.ones(side * side, device="cuda"), torch.empty(side * side, device="cuda")]
lib = _lib.load()
for flags, tag in [(_lib.MMK_PET_UPDATE | _lib.MMK_PET_OBJECTIVE, "update+objective"), (_lib.MMK_PET_UPDATE, "update only")]:
    for k in range(20):
        mm._iterate(lam[k & 1], lam[1 - (k & 1)], mm.status.f_ptr, mm.status.err_ptr, flags)
    torch.cuda.synchronize(); _lib.prof_report(); lib.mmk_prof_enable(1)
    for k in range(200):
        mm._iterate(lam[k & 1], lam[1 - (k & 1)], mm.status.f_ptr, mm.status.err_ptr, flags)
    torch.cuda.synchronize(); lib.mmk_prof_enable(0)
    prof = _lib.prof_report()
    print(tag, {k: round(1000 * ms / c, 1) for k, (c, ms) in prof.items()}, "us")
