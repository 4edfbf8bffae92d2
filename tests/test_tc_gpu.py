"""Known-answer test of the tcgen05 building blocks (csrc/diag/tc_selftest.cu, libmmk_diag.so)."""

import pytest
import torch

from paper_1003_3272_b200 import _lib

pytestmark = pytest.mark.gpu


def test_tcgen05_tf32_descriptors():
    _lib.torch_mod()
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.rand(128, 64, device="cuda", generator=g)
    B = torch.rand(64, 64, device="cuda", generator=g)
    X = torch.rand(32, 128, device="cuda", generator=g)
    V = torch.rand(32, 64, device="cuda", generator=g)
    D1 = torch.zeros(128, 64, device="cuda")
    D2 = torch.zeros(128, 32, device="cuda")
    D3 = torch.zeros(128, 64, device="cuda")
    diag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call_diag("mmk_selftest_tc", *(_lib.ptr(t) for t in (A, B, X, V, D1, D2, D3)), 14,
              _lib.ptr(diag), _lib.stream_handle(torch, torch.device("cuda", 0)))
    torch.cuda.synchronize()
    assert diag.item() == 0
    d = torch.float64
    for got, want in ((D1, A.to(d) @ B.to(d).T), (D2, A.to(d) @ B.to(d)[:, :32]),
                      (D3, X.to(d).T @ V.to(d))):
        err = ((got.to(d) - want).abs() / want.abs()).max().item()
        assert err < 3e-3, err
