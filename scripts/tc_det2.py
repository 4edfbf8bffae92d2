"""Repeat one tensor-core NNMF iteration at C4 and count distinct objectives."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import collections, torch
import test_nnmf_tc_gpu as T
m, n = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(m, n, device="cuda", generator=g)
v = torch.rand(m, 64, device="cuda", generator=g)
w = torch.rand(64, n, device="cuda", generator=g)
for _ in range(3):
    v, w, _ = T.one_iter(x, v, w, False)
fs = collections.Counter()
v0 = None
for i in range(int(sys.argv[3])):
    a = T.one_iter(x, v, w, False)
    fs[a[2]] += 1
    if v0 is None:
        v0, w0 = a[0], a[1]
    elif not (torch.equal(a[0], v0) and torch.equal(a[1], w0)):
        print("V/W differ at repeat", i)
print(m, n, dict(fs))
