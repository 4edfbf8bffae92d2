import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_1003_3272_b200 import _lib
from paper_1003_3272_b200.parallel import ShardedNnmf
import paper_1003_3272_b200 as M
_lib.torch_mod()
m, n, r = 131072, 16384, 64
g = torch.Generator(device='cuda'); g.manual_seed(1)
x = torch.rand(m, n, device='cuda', generator=g)
v = torch.rand(m, r, device='cuda', generator=g); w = torch.rand(r, n, device='cuda', generator=g)
sh = ShardedNnmf(x, v, w, r, M.Backend(dtype='fp32'))
tv = torch.zeros(6 * 256, dtype=torch.int64, device='cuda'); tw = torch.zeros_like(tv)
sh.iterate(1); torch.cuda.synchronize()
_lib.load().mmk_tc_set_trace(_lib.ptr(tv), _lib.ptr(tw))
sh.iterate(1); torch.cuda.synchronize()
_lib.load().mmk_tc_set_trace(None, None)
for name, t in (("vstep", tv), ("wstep", tw)):
    a = t.cpu().numpy().reshape(6, 256).astype(np.int64)
    t0 = a[0, 0]
    a = a - t0
    print(name, "cols: tma_issue split_start split_done mma_start mma_done  (cycles rel. to first TMA issue)")
    for i in list(range(0, 24)) + list(range(100, 112)) + list(range(240, 256)):
        print(f"{i:4d} " + " ".join(f"{a[k, i]:9d}" for k in range(5)))
    d = np.diff(a[4, 20:250])
    print(name, "steady MMA-done spacing (cycles/stage): mean %.0f" % d.mean(),
          " split latency (start->done) mean %.0f" % (a[2, 20:250] - a[1, 20:250]).mean(),
          " TMA issue->split start mean %.0f" % (a[1, 20:250] - a[0, 20:250]).mean(),
          " split done->mma start %.0f" % (a[3, 20:250] - a[2, 20:250]).mean(),
          " mma issue time %.0f" % (a[4, 20:250] - a[3, 20:250]).mean(),
          " operand ready->A ready (afull wait) %.0f" % (a[3, 20:250] - a[5, 20:250]).mean(),
          " prev MMA issued->operand ready %.0f" % (a[5, 21:251] - a[4, 20:250]).mean())
