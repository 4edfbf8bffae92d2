"""Pipeline trace of the tensor-core V step (CTA 0), from a -DMMK_TC_TRACE
build of nnmf_tc.cu (scripts/tc_variants.sh build trace "-DMMK_TC_TRACE"):
per-stage clock64 stamps -> medians of the pipeline intervals."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import test_nnmf_tc_gpu as T
from paper_1003_3272_b200 import _lib

m, n = 131072, 16384
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(m, n, device="cuda", generator=g)
v = torch.rand(m, 64, device="cuda", generator=g)
w = torch.rand(64, n, device="cuda", generator=g)
for _ in range(3):
    v, w, f = T.one_iter(x, v, w, False)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8 * 4096))()
lib = _lib.load()
lib.mmk_tc_trace_read.restype = ctypes.c_int
assert lib.mmk_tc_trace_read(buf) == 0
tr = np.frombuffer(buf, dtype=np.uint64).reshape(8, 4096).astype(np.int64)
nst = int(np.count_nonzero(tr[0]))
tr = tr[:, :nst]
t0 = tr[0, 0]
names = ["tma_issue", "mma_landed", "q_issued", "rempty_ok", "r_issued", "res_xfull", "res_rfull", "res_done"]
st = slice(20, nst - 5)
def med(a): return float(np.median(a[st]))
print("stages", nst, "total cycles", tr[0, -1] - t0)
print("period (tma issue)", med(np.diff(tr[0])))
print("period (mma landed)", med(np.diff(tr[1])))
print("issue->landed", med(tr[1] - tr[0]))
print("landed->Q issued", med(tr[2] - tr[1]))
print("Q issued->rempty ok", med(tr[3] - tr[2]))
print("rempty ok->R issued", med(tr[4] - tr[3]))
res = tr[5] > 0
print("residual: xfull seen - landed(mma)", med(tr[5] - tr[1]))
print("residual: rfull seen - R issued", med(tr[6] - tr[4]))
print("residual: work (rfull->done)", med(tr[7] - tr[6]))
print("MMA next landed wait: landed(k+1) - r_issued(k)", med(tr[1][1:] - tr[4][:-1]))
print("slot turnaround: tma issue(k+4) - tma issue(k)", med(tr[0][4:] - tr[0][:-4]))
