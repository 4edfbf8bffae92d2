import sys, time
sys.path.insert(0, '.')
import torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib
from paper_1003_3272_b200.parallel import ShardedNnmf
_lib.torch_mod()
m, n, r = 131072, 16384, 64
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(m, n, device="cuda", generator=g)
v = torch.rand(m, r, device="cuda", generator=g)
w = torch.rand(r, n, device="cuda", generator=g)
be = M.Backend(dtype="fp32")
sh = ShardedNnmf(x, v.clone(), w.clone(), r, be)
for _ in range(5): sh.iterate(1)
torch.cuda.synchronize()
for rep in range(2):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); [sh.iterate(1) for _ in range(100)]; e.record(); torch.cuda.synchronize()
    print("eager  %.3f ms/it" % (s.elapsed_time(e) / 100))
    prob = M.NnmfProblem(x=x, rank=r)
    cfg = M.MmConfig(max_iters=100, epsilon=1e-300, monotone_tol=1e-5)
    M.nnmf_run(prob, M.MmConfig(max_iters=4, epsilon=1e-300, monotone_tol=1e-5), be, state0=M.FactorPair(v, w))
    torch.cuda.synchronize()
    s.record(); st, tr = M.nnmf_run(prob, cfg, be, state0=M.FactorPair(v, w)); e.record(); torch.cuda.synchronize()
    print("engine %.3f ms/it (%d it, incl. graph build)" % (s.elapsed_time(e) / tr.iters, tr.iters))
