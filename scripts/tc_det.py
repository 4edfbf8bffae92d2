"""Run-to-run determinism of one tensor-core NNMF iteration at several shapes."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import test_nnmf_tc_gpu as T

for m, n in [(3000, 640), (40960, 1024), (131072, 2048), (131072, 16384)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(m, n, device="cuda", generator=g)
    v = torch.rand(m, 64, device="cuda", generator=g)
    w = torch.rand(64, n, device="cuda", generator=g)
    outs = [T.one_iter(x, v, w, False) for _ in range(3)]
    a = outs[0]
    for b in outs[1:]:
        print(m, n, "V eq", torch.equal(a[0], b[0]), "W eq", torch.equal(a[1], b[1]), "f eq", a[2] == b[2],
              "dV", float((a[0] - b[0]).abs().max()), "dW", float((a[1] - b[1]).abs().max()), "df", a[2] - b[2])
    del x, v, w, outs
    torch.cuda.empty_cache()
