import sys
sys.path.insert(0, '.')
import torch
from paper_1003_3272_b200 import _lib
_lib.torch_mod()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
st = _lib.stream_handle(torch, torch.device("cuda", 0))
names = ["SS tf32 N128 K8", "TS tf32 N128 K8", "TS tf32 N64 K8", "SS tf32 N256 K8", "SS f16 N128 K16", "SS tf32 N64 K8", "TS f16 N256 K16", "SS f16 N256 K16",
         "SS tf32 N128 rot4", "TS tf32 N64 rot4", "SS tf32 N128 rot2", "TS tf32 N128 rot2", "SS f16 N256 rot2"]
flops = [2*128*128*8, 2*128*128*8, 2*128*64*8, 2*128*256*8, 2*128*128*16, 2*128*64*8, 2*128*256*16, 2*128*256*16,
         2*128*128*8, 2*128*64*8, 2*128*128*8, 2*128*128*8, 2*128*256*16]
for mode in range(13):
    for iters in (256, 4096):
        _lib.call_diag("mmk_tc_mma_bench", mode, iters, _lib.ptr(out), st)
        torch.cuda.synchronize()
    cyc = out.item() / 4096
    print(f"{names[mode]:18s} {cyc:7.1f} cycles/MMA  {flops[mode]/cyc:7.0f} flop/cycle")
