"""Does a Morton (Z-order) pixel numbering speed up the sparse projectors at
the pet-large shape?  Same matrix, pixel indices permuted, kernel times compared."""
import sys, time
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

def morton(side):
    idx = np.arange(side * side)
    r, c = idx // side, idx % side
    def spread(v):
        v = v.astype(np.int64)
        out = np.zeros_like(v)
        for b in range(16):
            out |= ((v >> b) & 1) << (2 * b)
        return out
    key = spread(r) << 1 | spread(c)
    order = np.argsort(key, kind="stable")      # new index -> old pixel
    pi = np.empty_like(order); pi[order] = np.arange(len(order))   # old -> new
    return pi, order

def permuted(sa, nb, pi, order):
    dev = sa["ridx"].device
    pit = torch.from_numpy(pi).to(dev).to(torch.int32)
    ridx = pit[sa["ridx"].long()]
    # keep CSR rows sorted by (new) pixel index
    rptr = sa["rptr"].long()
    d = sa["n_rays"]
    rowid = torch.repeat_interleave(torch.arange(d, device=dev), rptr[1:] - rptr[:-1])
    key = rowid * (side * side) + ridx.long()
    o = torch.argsort(key)
    ridx, rval = ridx[o], sa["rval"][o]
    # CSC from the permuted CSR
    key2 = ridx.long() * d + rowid[o]
    o2 = torch.argsort(key2)
    cidx = rowid[o][o2].to(torch.int32)
    cval = rval[o2]
    counts = torch.bincount(ridx.long(), minlength=side * side)
    cptr = torch.zeros(side * side + 1, dtype=torch.int64, device=dev); cptr[1:] = torch.cumsum(counts, 0)
    out = dict(sa)
    out.update(ridx=ridx.to(torch.int32).contiguous(), rval=rval.contiguous(), cidx=cidx.contiguous(),
               cval=cval.contiguous(), cptr=cptr.to(torch.int32))
    nb2 = [None] * (side * side)
    for old, lst in enumerate(nb):
        nb2[pi[old]] = sorted(int(pi[k]) for k in lst)
    return out, nb2

def time_it(sa_, nb_, tag):
    lam_true = torch.ones(side * side, device="cuda")
    means = M.SparsePetProblem(sa_, np.zeros(geo.n_rays), 0.0, nb_).forward(lam_true)
    y = torch.poisson(means * 50.0, generator=torch.Generator(device="cuda").manual_seed(1))
    mm = _GpuPet(M.SparsePetProblem(sa_, y, 1e-6, nb_), be)
    lam = [torch.ones(side * side, device="cuda"), torch.empty(side * side, device="cuda")]
    for k in range(20):
        mm._iterate(lam[k & 1], lam[1 - (k & 1)], mm.status.f_ptr, mm.status.err_ptr)
    torch.cuda.synchronize()
    lib = _lib.load(); lib.mmk_prof_enable(1)
    for k in range(200):
        mm._iterate(lam[k & 1], lam[1 - (k & 1)], mm.status.f_ptr, mm.status.err_ptr)
    torch.cuda.synchronize(); lib.mmk_prof_enable(0)
    prof = _lib.prof_report()
    print(tag, {k: round(1000 * ms / c, 1) for k, (c, ms) in prof.items()}, "us")

time_it(sa, nb, "natural")
pi, order = morton(side)
sa2, nb2 = permuted(sa, nb, pi, order)
time_it(sa2, nb2, "morton ")
