import sys
import torch
sys.path.insert(0, '.')
from paper_1003_3272_b200 import _lib
_lib.torch_mod()
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(128, 64, device="cuda", generator=g)
B = torch.rand(64, 64, device="cuda", generator=g)
X = torch.rand(32, 128, device="cuda", generator=g)
V = torch.rand(32, 64, device="cuda", generator=g)
d = torch.float64
st = _lib.stream_handle(torch, torch.device("cuda", 0))
for mode in (1, 2, 4, 8, 14):
    D1 = torch.full((128, 64), -7.0, device="cuda")
    D2 = torch.full((128, 32), -7.0, device="cuda")
    D3 = torch.full((128, 64), -7.0, device="cuda")
    diag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call_diag("mmk_selftest_tc", *(_lib.ptr(t) for t in (A, B, X, V, D1, D2, D3)), mode, _lib.ptr(diag), st)
    torch.cuda.synchronize()
    print("mode", mode, "diag", diag.item(), flush=True)
    if mode == 1:
        raw = D1.reshape(-1).cpu()
        Ah = A.cpu()
        ok = 0; bad = 0
        for b in range(2):
            for i in range(128):
                for c in range(8):
                    cs = c ^ (i % 8)
                    off = b * 4096 + i * 32 + cs * 4
                    if torch.equal(raw[off:off + 4], Ah[i, b * 32 + 4 * c: b * 32 + 4 * c + 4]):
                        ok += 1
                    else:
                        bad += 1
        print(" swizzle model ok", ok, "bad", bad, " raw[0:8]", raw[:8].tolist(), " A[0,:8]", Ah[0, :8].tolist(), flush=True)
        continue
    for name, got, want in (("D1", D1, A.to(d) @ B.to(d).T), ("D2", D2, A.to(d) @ B.to(d)[:, :32]), ("D3", D3, X.to(d).T @ V.to(d))):
        err = ((got.to(d) - want).abs() / want.abs())
        print(" ", name, "maxerr %.3e med %.3e" % (err.max().item(), err.median().item()), "got", [round(x, 3) for x in got[0, :4].tolist()], "want", [round(x, 3) for x in want[0, :4].tolist()], flush=True)
# 32B-atom swizzle model check on the dumps from mode 1
D1 = torch.zeros(128, 64, device="cuda"); D2 = torch.zeros(128, 32, device="cuda"); D3 = torch.zeros(128, 64, device="cuda")
diag = torch.zeros(1, dtype=torch.int32, device="cuda")
_lib.call_diag("mmk_selftest_tc", *(_lib.ptr(t) for t in (A, B, X, V, D1, D2, D3)), 1, _lib.ptr(diag), st)
torch.cuda.synchronize()
raw = D3.reshape(-1).cpu()
Xh, Bh = X.cpu(), B.cpu()
def check(rawbuf, src, rows, boxes, fn):
    ok = bad = 0
    for b in range(boxes):
        for i in range(rows):
            for c in range(4):
                cs = fn(c, i)
                off = b * rows * 32 + i * 32 + cs * 8
                if torch.equal(rawbuf[off:off + 8], src[i, b * 32 + 8 * c: b * 32 + 8 * c + 8]):
                    ok += 1
                else:
                    bad += 1
    return ok, bad
for nm, fn in (("i%4", lambda c, i: c ^ (i % 4)), ("(i/2)%4", lambda c, i: c ^ ((i // 2) % 4)), ("none", lambda c, i: c)):
    print("X atom32 model", nm, check(raw[:128 * 32], Xh, 32, 4, fn), "B atom32", check(raw[128 * 32:128 * 32 + 64 * 32], Bh, 64, 1, fn), flush=True)
