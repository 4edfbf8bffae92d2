"""Cross-CTA hand-off latencies inside a CTA pair (mmk_tc_pingpong)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1003_3272_b200 import _lib
_lib.torch_mod()
out = torch.zeros(4, dtype=torch.int64, device="cuda")
st = _lib.stream_handle(torch, torch.device("cuda", 0))
for iters in (64, 1024):
    out.zero_()
    _lib.call_diag("mmk_tc_pingpong", iters, _lib.ptr(out), st)
    torch.cuda.synchronize()
o = out.cpu().tolist()
print(f"remote arrive round trip: {o[0]} cycles; commit-multicast + remote arrive round trip: {o[1]} cycles; timeouts {o[2]},{o[3]}")
