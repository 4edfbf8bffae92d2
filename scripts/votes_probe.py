import sys, time
sys.path.insert(0, '.')
import torch
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib
from paper_1003_3272_b200.mds import PackedMdsProblem
q, m = 65536, 671
g = torch.Generator(device="cuda").manual_seed(0)
votes = (torch.randint(-1, 2, (q, m), generator=g, device="cuda").float())
votes[:, 0] = 1.0     # every pair shares roll call 0
be = M.Backend(dtype="fp32", mds_kernel="tri")
PackedMdsProblem.from_votes(votes[:4096], 3, be)
lib = _lib.load(); lib.mmk_prof_enable(1)
torch.cuda.synchronize(); t0 = time.perf_counter()
pk = PackedMdsProblem.from_votes(votes, 3, be)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
lib.mmk_prof_enable(0)
print("q=65536 m=671 votes -> packed tiles: %.1f ms wall" % (1e3 * dt), _lib.prof_report())
flops = 2 * (q / 128) * (q / 128 + 1) / 2 * 128 * 256 * 2 * 704
print("MMA flop %.3g" % flops)
