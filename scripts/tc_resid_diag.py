"""Diagnose the tensor-core objective: F' (MMK_TC_EXP=4, no correction) and f
against torch fp64 restatements on well-fit data."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import test_nnmf_tc_gpu as T

m, n = 1024, 2048
x, v, w = T.well_fit(m, n, m + n)
_, _, f = T.one_iter(x, v, w, force_simt=False)
xd, vd, wd = x.double(), v.double(), w.double()
D = xd - vd @ wd
fr = float((D * D).sum())
mx = v.abs().amax(1)
ev = (15 - torch.frexp(mx)[1]).clamp(-120, 120).double()
s = torch.exp2(ev)[:, None]
vh = ((vd * s).float().half().double()) / s
E = vd - vh
# W_e: global scale
ew = 15 - torch.frexp(w.abs().max())[1].item()
sw = 2.0 ** ew
whi = (w * sw).half().float()
wlo = ((w * sw) - whi).half().float()
we = (whi.double() + wlo.double()) / sw
xx = x.abs().max(); ex = 15 - torch.frexp(xx)[1].item(); sx = 2.0 ** ex
xhi = (x * sx).half().float(); xlo = ((x * sx) - xhi).half().float()
xe = (xhi.double() + xlo.double()) / sx
Fp = float(((xe - vh @ we) ** 2).sum())
corr = float(-2 * ((xd - vd @ wd) @ wd.T * E).sum() - ((E @ wd) ** 2).sum())
print("f kernel", f, "f ref", fr, "rel", (f - fr) / fr)
print("F' ref", Fp, "corr ref", corr, "F'+corr", Fp + corr, "rel", (Fp + corr - fr) / fr)
os.environ["MMK_TC_EXP"] = "4"
