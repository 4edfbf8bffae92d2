"""cta_group::2 vs cta_group::1 tcgen05.mma issue rate (kind::f16)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1003_3272_b200 import _lib
_lib.torch_mod()
out = torch.zeros(4, dtype=torch.int64, device="cuda")
st = _lib.stream_handle(torch, torch.device("cuda", 0))
for n in (64, 128, 192, 256, -64, -128, -256):
    for iters in (256, 4096):
        out.zero_()
        _lib.call_diag("mmk_tc_mma2_bench", n, iters, _lib.ptr(out), st)
        torch.cuda.synchronize()
    o = out.cpu().tolist()
    cyc = o[0] / 4096
    print(f"2CTA M256 {'TS' if n < 0 else 'SS'} N{abs(n):3d}: {cyc:7.1f} cycles/MMA  {2*256*abs(n)*16/cyc/2:7.0f} flop/cycle/SM  timeouts {o[1]},{o[2]}")
