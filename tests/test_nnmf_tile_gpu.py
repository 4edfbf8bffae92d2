"""Register-blocked CUDA-core NNMF kernels for ranks 17..128
(csrc/nnmf_tile.cu): fp64 at a large shape and fp32 shapes the tensor-core
path does not take, against the same iterations in torch fp64 (cuBLAS DGEMM,
not our kernels); the grouping of the reference (nnmf.py:84-110) up to
rounding."""

import numpy as np
import pytest
import torch

import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib

pytestmark = pytest.mark.gpu


def torch_trace(x, v, w, iters):
    xd, v, w = x.double(), v.double(), w.double()
    trace = []
    for _ in range(iters):
        trace.append(float(((xd - v @ w) ** 2).sum()))
        v = v * ((xd @ w.T) / (v @ (w @ w.T) + 1e-300))
        w = w * ((v.T @ xd) / ((v.T @ v) @ w + 1e-300))
    trace.append(float(((xd - v @ w) ** 2).sum()))
    return np.array(trace), v @ w


def run_profiled(x, r, dtype, iters, v0, w0, fused=True):
    lib = _lib.load()
    lib.mmk_prof_enable(1)
    try:
        st, tr = M.nnmf_run(M.NnmfProblem(x=x, rank=r),
                            M.MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6),
                            M.Backend(dtype=dtype, fused=fused), state0=M.FactorPair(v0, w0))
        torch.cuda.synchronize()
    finally:
        lib.mmk_prof_enable(0)
    return st, tr, _lib.prof_report()


def test_fp64_large_shape_matches_torch_fp64():
    """fp64, 32768 x 8192, r = 64 -- the shape class of BASELINE config 4 in
    the reference's precision -- 4 iterations per-iteration (the launch
    profiler sees every kernel): trace and V W to 1e-10."""
    m, n, r, iters = 32768, 8192, 64, 4
    g = torch.Generator(device="cuda").manual_seed(64)
    x = torch.rand(m, n, device="cuda", generator=g, dtype=torch.float64)
    v0 = torch.rand(m, r, device="cuda", generator=g, dtype=torch.float64)
    w0 = torch.rand(r, n, device="cuda", generator=g, dtype=torch.float64)
    st, tr, prof = run_profiled(x, r, "fp64", iters, v0, w0, fused=False)
    assert "nnmf_vstep_tile" in prof and "nnmf_wpart_tile" in prof, sorted(prof)
    want, vw = torch_trace(x, v0, w0, iters)
    assert np.max(np.abs(tr.objective_values - want) / want) < 1e-10
    got = st.v.double() @ st.w.double()
    assert float((got - vw).norm() / vw.norm()) < 1e-10


@pytest.mark.parametrize("m,n,r", [(1001, 777, 40), (2050, 3001, 17), (515, 4099, 64),
                                   (1001, 777, 100), (2050, 3001, 128)])
def test_fp32_shapes_off_the_tensor_cores(m, n, r):
    """fp32 with m or n not a multiple of 8 (no TMA-aligned pre-split copy):
    the tile kernels, 8 fused iterations, to 1e-4."""
    iters = 8
    g = torch.Generator(device="cuda").manual_seed(m + n + r)
    x = torch.rand(m, n, device="cuda", generator=g)
    v0 = torch.rand(m, r, device="cuda", generator=g)
    w0 = torch.rand(r, n, device="cuda", generator=g)
    st, tr, prof = run_profiled(x, r, "fp32", iters, v0, w0, fused=False)
    assert "nnmf_vstep_tile" in prof and "nnmf_vstep_tc" not in prof, sorted(prof)
    want, vw = torch_trace(x, v0, w0, iters)
    assert np.max(np.abs(tr.objective_values - want) / want) < 1e-4
    got = st.v.double() @ st.w.double()
    assert float((got - vw).norm() / vw.norm()) < 1e-4
    # and the fused device loop gives the same trace bitwise
    _, tr2, _ = run_profiled(x, r, "fp32", iters, v0, w0, fused=True)
    assert np.array_equal(tr.objective_values, tr2.objective_values)


def test_rank128_large_shape_fp32_tiles():
    """r = 128 at 65536 x 16384 in fp32 on the 128-rank CUDA-core tiles
    (MMK_NNMF_TC=0; the default path for this shape is the rank-128
    tensor-core kernels, tests/test_nnmf_tc_gpu.py), 5 iterations against torch
    fp64, trace and V W to 1e-4."""
    import os
    m, n, r, iters = 65536, 16384, 128, 5
    g = torch.Generator(device="cuda").manual_seed(128)
    x = torch.rand(m, n, device="cuda", generator=g)
    v0 = torch.rand(m, r, device="cuda", generator=g)
    w0 = torch.rand(r, n, device="cuda", generator=g)
    old = os.environ.get("MMK_NNMF_TC")
    os.environ["MMK_NNMF_TC"] = "0"
    try:
        st, tr, prof = run_profiled(x, r, "fp32", iters, v0, w0, fused=False)
    finally:
        if old is None:
            os.environ.pop("MMK_NNMF_TC")
        else:
            os.environ["MMK_NNMF_TC"] = old
    assert "nnmf_vstep_tile" in prof and "nnmf_wpart_tile" in prof, sorted(prof)
    want, vw = torch_trace(x, v0, w0, iters)
    assert np.max(np.abs(tr.objective_values - want) / want) < 1e-4
    got = st.v.double() @ st.w.double()
    assert float((got - vw).norm() / vw.norm()) < 1e-4


@pytest.mark.parametrize("r", [40, 64, 100, 128])
def test_fp64_dmma_deterministic_and_fused_equal(r):
    """fp64 on the DMMA tiles: two runs bitwise equal, and the fused device
    loop equals the per-iteration path bit for bit (same kernels, fixed
    split-K order)."""
    m, n, iters = 2050, 1001, 5
    g = torch.Generator(device="cuda").manual_seed(r + 7)
    x = torch.rand(m, n, device="cuda", generator=g, dtype=torch.float64)
    v0 = torch.rand(m, r, device="cuda", generator=g, dtype=torch.float64)
    w0 = torch.rand(r, n, device="cuda", generator=g, dtype=torch.float64)
    a, ta, prof = run_profiled(x, r, "fp64", iters, v0, w0, fused=False)
    b, tb, _ = run_profiled(x, r, "fp64", iters, v0, w0, fused=False)
    c, tc_, _ = run_profiled(x, r, "fp64", iters, v0, w0, fused=True)
    assert "nnmf_vstep_tile" in prof, sorted(prof)
    assert np.array_equal(ta.objective_values, tb.objective_values)
    assert np.array_equal(ta.objective_values, tc_.objective_values)
    assert torch.equal(a.v, b.v) and torch.equal(a.w, b.w)
    assert torch.equal(a.v, c.v) and torch.equal(a.w, c.w)


@pytest.mark.parametrize("r", [65, 100, 128])
def test_fp64_ranks_above_64(r):
    """fp64, ranks 65..128 (the 128-rank tiles, zero-padded ranks), 6
    iterations against torch fp64 to 1e-10."""
    m, n, iters = 3000, 2100, 6
    g = torch.Generator(device="cuda").manual_seed(r)
    x = torch.rand(m, n, device="cuda", generator=g, dtype=torch.float64)
    v0 = torch.rand(m, r, device="cuda", generator=g, dtype=torch.float64)
    w0 = torch.rand(r, n, device="cuda", generator=g, dtype=torch.float64)
    st, tr, prof = run_profiled(x, r, "fp64", iters, v0, w0, fused=False)
    assert "nnmf_vstep_tile" in prof, sorted(prof)
    want, vw = torch_trace(x, v0, w0, iters)
    assert np.max(np.abs(tr.objective_values - want) / want) < 1e-10
    got = st.v.double() @ st.w.double()
    assert float((got - vw).norm() / vw.norm()) < 1e-10


def torch_poisson(x, v, w, iters):
    """nnmf_poisson_objective / nnmf_poisson_update (nnmf.py:194-242) in torch fp64."""
    xd, v, w = x.double(), v.double(), w.double()
    pos = xd > 0
    trace = []

    def fit(v, w):
        b = v @ w
        return float(torch.where(pos, xd * torch.log(torch.where(pos, b, 1.0)), 0.0).sum()
                     - b.sum())

    for _ in range(iters):
        trace.append(fit(v, w))
        ratio = torch.where(pos, xd / (v @ w), 0.0)
        v = v * torch.sqrt((ratio @ w.T) / (w.sum(1)[None, :] + 1e-300))
        ratio = torch.where(pos, xd / (v @ w), 0.0)
        w = w * torch.sqrt((v.T @ ratio) / (v.sum(0)[:, None] + 1e-300))
    trace.append(fit(v, w))
    return np.array(trace), v @ w


@pytest.mark.parametrize("dtype,tol,m,n,r", [("fp64", 1e-10, 2050, 3001, 40),
                                             ("fp64", 1e-10, 1000, 777, 64),
                                             ("fp32", 1e-4, 16384, 8192, 64),
                                             ("fp64", 1e-10, 1000, 777, 100),
                                             ("fp64", 1e-10, 2050, 1001, 128),
                                             ("fp32", 1e-4, 8192, 4096, 128)])
def test_poisson_tiles_match_torch(dtype, tol, m, n, r):
    """Poisson NNMF on the tile kernels (ranks 17..128, rank tiles of 64 and
    128; the warp-per-row kernels spilled at r = 64: 58.6 ms per V step at
    32768 x 8192), count-like data with zeros, 5 iterations against torch
    fp64."""
    iters = 5
    tdt = torch.float64 if dtype == "fp64" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(m + r)
    x = torch.floor(4.0 * torch.rand(m, n, device="cuda", generator=g, dtype=tdt))   # 0..3
    v0 = torch.rand(m, r, device="cuda", generator=g, dtype=tdt) + 0.1
    w0 = torch.rand(r, n, device="cuda", generator=g, dtype=tdt) + 0.1
    lib = _lib.load()
    lib.mmk_prof_enable(1)
    try:
        st, tr = M.nnmf_poisson_run(M.NnmfProblem(x=x, rank=r),
                                    M.MmConfig(max_iters=iters, epsilon=1e-300,
                                               monotone_tol=1e-6),
                                    M.Backend(dtype=dtype, fused=False),
                                    state0=M.FactorPair(v0, w0))
        torch.cuda.synchronize()
    finally:
        lib.mmk_prof_enable(0)
    prof = _lib.prof_report()
    assert "pois_vstep_tile" in prof and "pois_wpart_tile" in prof, sorted(prof)
    want, vw = torch_poisson(x, v0, w0, iters)
    assert np.max(np.abs(tr.objective_values - want) / np.abs(want)) < tol
    got = st.v.double() @ st.w.double()
    assert float((got - vw).norm() / vw.norm()) < tol
