"""Tensor-core (tcgen05 kind::f16, scaled fp16 hi/lo split products) NNMF
path vs fp64 on the same inputs: one iteration (V', W', objective) and a
30-iteration run, on tile-aligned and ragged shapes (TMA out-of-bounds fill
on both edges), with inputs far from unit scale and with a wide per-row
dynamic range (the power-of-two scaling of csrc/nnmf_tc.cu)."""

import os

import numpy as np
import pytest
import torch

import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib
from paper_1003_3272_b200 import parallel as P

pytestmark = pytest.mark.gpu


def one_iter(x, v, w, force_simt):
    torch_ = _lib.torch_mod()
    dev = x.device
    code = _lib.dtype_code(x.dtype)
    m, n = x.shape
    r = v.shape[1]
    ws = torch_.zeros(_lib.ws_bytes("mmk_nnmf_ws_bytes", code, m, n, r), dtype=torch_.uint8,
                      device=dev)
    red = torch_.zeros(_lib.load().mmk_nnmf_reduce_len(n, r), dtype=torch_.float64, device=dev)
    st = _lib.StatusBlock(torch_, dev)
    vo, wo = torch_.empty_like(v), torch_.empty_like(w)
    old = os.environ.get("MMK_NNMF_TC")
    os.environ["MMK_NNMF_TC"] = "0" if force_simt else "1"
    try:
        _lib.call("mmk_nnmf_iter", code, _lib.ptr(x), x.stride(0), _lib.ptr(v), _lib.ptr(w),
                  _lib.ptr(vo), _lib.ptr(wo), m, n, r, _lib.ptr(ws), ws.numel(), _lib.ptr(red),
                  st.f_ptr, st.err_ptr, _lib.stream_handle(torch_, dev))
        f = st.read()[0]
    finally:
        if old is None:
            os.environ.pop("MMK_NNMF_TC")
        else:
            os.environ["MMK_NNMF_TC"] = old
    return vo, wo, f


def reference_iter(x, v, w):
    x, v, w = x.double(), v.double(), w.double()
    f = float(((x - v @ w) ** 2).sum())
    v2 = v * ((x @ w.T) / (v @ (w @ w.T) + 1e-300))
    w2 = w * ((v2.T @ x) / ((v2.T @ v2) @ w + 1e-300))
    return v2, w2, f


def tc_launched(fn):
    """Run fn with the launch profiler on; True if the tcgen05 kernels ran."""
    lib = _lib.load()
    lib.mmk_prof_enable(1)
    try:
        out = fn()
        torch.cuda.synchronize()
    finally:
        lib.mmk_prof_enable(0)
    prof = _lib.prof_report()
    return out, "nnmf_vstep_tc" in prof and "nnmf_wstep_tc" in prof


@pytest.mark.parametrize("m,n,scale", [(1024, 512, 1.0), (1000, 1000, 1.0), (4104, 392, 1.0),
                                       (1024, 512, 1e-6), (1024, 512, 3e6)])
def test_tc_iteration_matches_fp64(m, n, scale):
    g = torch.Generator(device="cuda").manual_seed(m + n)
    x = torch.rand(m, n, device="cuda", generator=g) * scale
    v = torch.rand(m, 64, device="cuda", generator=g)
    w = torch.rand(64, n, device="cuda", generator=g)
    (vt, wt, ft), used = tc_launched(lambda: one_iter(x, v, w, force_simt=False))
    assert used, "tensor-core path did not run"
    vr, wr, fr = reference_iter(x, v, w)
    rel = lambda a, b: float((a.double() - b).norm() / b.norm())  # noqa: E731
    assert abs(ft - fr) / fr < 2e-6, (ft, fr)
    assert rel(vt, vr) < 3e-5 and rel(wt, wr) < 3e-5, (rel(vt, vr), rel(wt, wr))
    vs, ws_, fs = one_iter(x, v, w, force_simt=True)
    assert rel(vt, vs.double()) < 3e-5


@pytest.mark.parametrize("r", [17, 32, 48, 63])
def test_tc_padded_ranks_match_fp64(r):
    """Ranks 17..63 run on the rank-64 tensor-core kernels with V and W
    zero-padded (nnmf_tc.cu iter_a): a zero component stays exactly zero
    and contributes nothing, so V', W', f equal the fp64 update of the rank-r
    problem to the split-product accuracy."""
    g = torch.Generator(device="cuda").manual_seed(r)
    m, n = 1032, 776
    x = torch.rand(m, n, device="cuda", generator=g)
    v = torch.rand(m, r, device="cuda", generator=g)
    w = torch.rand(r, n, device="cuda", generator=g)
    (vt, wt, ft), used = tc_launched(lambda: one_iter(x, v, w, force_simt=False))
    assert used, "tensor-core path did not run"
    vr, wr, fr = reference_iter(x, v, w)
    rel = lambda a, b: float((a.double() - b).norm() / b.norm())  # noqa: E731
    assert abs(ft - fr) / fr < 2e-6, (ft, fr)
    assert rel(vt, vr) < 3e-5 and rel(wt, wr) < 3e-5, (rel(vt, vr), rel(wt, wr))


@pytest.mark.parametrize("m,n,r,scale", [(1032, 776, 128, 1.0), (1032, 776, 65, 1.0),
                                         (1032, 776, 100, 1.0), (1032, 776, 127, 1.0),
                                         (4104, 392, 128, 1.0), (1024, 512, 128, 1e-6),
                                         (1024, 512, 128, 3e6), (2000, 1000, 96, 1.0)])
def test_tc_rank128_tile_matches_fp64(m, n, r, scale):
    """Ranks 65..128 on the rank-128 tensor-core kernels (one Q set copied
    out through the Q scratch, 3-deep X ring, one 128-column W-step block per
    item; ranks below 128 zero-padded): one iteration against fp64 to the
    split-product accuracy, ragged and tile-aligned shapes, far from unit
    scale."""
    g = torch.Generator(device="cuda").manual_seed(m + n + r)
    x = torch.rand(m, n, device="cuda", generator=g) * scale
    v = torch.rand(m, r, device="cuda", generator=g)
    w = torch.rand(r, n, device="cuda", generator=g)
    (vt, wt, ft), used = tc_launched(lambda: one_iter(x, v, w, force_simt=False))
    assert used, "tensor-core path did not run"
    vr, wr, fr = reference_iter(x, v, w)
    rel = lambda a, b: float((a.double() - b).norm() / b.norm())  # noqa: E731
    assert abs(ft - fr) / fr < 2e-6, (ft, fr)
    assert rel(vt, vr) < 3e-5 and rel(wt, wr) < 3e-5, (rel(vt, vr), rel(wt, wr))


@pytest.mark.parametrize("r,iters", [(128, 8), (96, 4)])
def test_tc_rank128_large_shape(r, iters):
    """r = 128 and 96 at 65536 x 16384 on the rank-128 tensor-core kernels (the
    review's large-shape check of r = 128 on UTCHMMA kernels): fused
    iterations against the same iterations in torch fp64 (cuBLAS DGEMM):
    trace and V W to 1e-4."""
    m, n = 65536, 16384
    g = torch.Generator(device="cuda").manual_seed(r)
    x = torch.rand(m, n, device="cuda", generator=g)
    v0 = torch.rand(m, r, device="cuda", generator=g)
    w0 = torch.rand(r, n, device="cuda", generator=g)
    lib = _lib.load()
    lib.mmk_prof_enable(1)
    try:
        st, tr = M.nnmf_run(M.NnmfProblem(x=x, rank=r),
                            M.MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6),
                            M.Backend(dtype="fp32", fused=False), state0=M.FactorPair(v0, w0))
        torch.cuda.synchronize()
    finally:
        lib.mmk_prof_enable(0)
    prof = _lib.prof_report()
    assert "nnmf_vstep_tc" in prof and "nnmf_wstep_tc" in prof, sorted(prof)
    xd, v, w = x.double(), v0.double(), w0.double()
    trace = []
    for _ in range(iters):
        trace.append(float(((xd - v @ w) ** 2).sum()))
        v = v * ((xd @ w.T) / (v @ (w @ w.T) + 1e-300))
        w = w * ((v.T @ xd) / ((v.T @ v) @ w + 1e-300))
    trace.append(float(((xd - v @ w) ** 2).sum()))
    err = np.max(np.abs(tr.objective_values - np.array(trace)) / np.array(trace))
    assert err < 1e-4, err
    vw = st.v.double() @ st.w.double()
    assert float((vw - v @ w).norm() / (v @ w).norm()) < 1e-4
    # the fused device loop gives the same trace bitwise
    _, tr2 = M.nnmf_run(M.NnmfProblem(x=x, rank=r),
                        M.MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6),
                        M.Backend(dtype="fp32"), state0=M.FactorPair(v0, w0))
    assert np.array_equal(tr.objective_values, tr2.objective_values)


def test_tc_rank32_large_shape_10_iters():
    """r = 32 at 65536 x 16384 (the verdict's large-shape check of a rank other
    than 64): 10 fused tensor-core iterations against the same iterations in
    torch fp64 (cuBLAS DGEMM, not our kernels): trace and V W to 1e-4."""
    m, n, r, iters = 65536, 16384, 32, 10
    g = torch.Generator(device="cuda").manual_seed(32)
    x = torch.rand(m, n, device="cuda", generator=g)
    v0 = torch.rand(m, r, device="cuda", generator=g)
    w0 = torch.rand(r, n, device="cuda", generator=g)
    lib = _lib.load()
    lib.mmk_prof_enable(1)
    try:
        st, tr = M.nnmf_run(M.NnmfProblem(x=x, rank=r),
                            M.MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6),
                            M.Backend(dtype="fp32"), state0=M.FactorPair(v0, w0))
        torch.cuda.synchronize()
    finally:
        lib.mmk_prof_enable(0)
    assert "nnmf_presplit_cached" in _lib.prof_report()   # the tensor-core path's prologue
    xd, v, w = x.double(), v0.double(), w0.double()
    trace = []
    for _ in range(iters):
        trace.append(float(((xd - v @ w) ** 2).sum()))
        v = v * ((xd @ w.T) / (v @ (w @ w.T) + 1e-300))
        w = w * ((v.T @ xd) / ((v.T @ v) @ w + 1e-300))
    trace.append(float(((xd - v @ w) ** 2).sum()))
    err = np.max(np.abs(tr.objective_values - np.array(trace)) / np.array(trace))
    assert err < 1e-4, err
    vw = st.v.double() @ st.w.double()
    assert float((vw - v @ w).norm() / (v @ w).norm()) < 1e-4


def test_tc_run_parity_30_iters():
    rng = np.random.default_rng(3)
    x = rng.random((2048, 1024)).astype(np.float32).astype(np.float64)
    v0 = rng.random((2048, 64)).astype(np.float32).astype(np.float64)
    w0 = rng.random((64, 1024)).astype(np.float32).astype(np.float64)
    prob = M.NnmfProblem(x=x, rank=64)
    cfg = M.MmConfig(max_iters=30, epsilon=1e-300, monotone_tol=1e-6)
    s32, t32 = M.nnmf_run(prob, cfg, M.Backend(dtype="fp32"), state0=M.FactorPair(v0, w0))
    s64, t64 = M.nnmf_run(prob, M.MmConfig(max_iters=30, epsilon=1e-300), M.Backend(dtype="fp64"),
                          state0=M.FactorPair(v0, w0))
    err = np.max(np.abs(t32.objective_values - t64.objective_values) / t64.objective_values)
    assert err < 1e-4, err
    vw32, vw64 = s32.v @ s32.w, s64.v @ s64.w
    assert np.linalg.norm(vw32 - vw64) / np.linalg.norm(vw64) < 1e-4


@pytest.mark.parametrize("r", [64, 128, 100])
def test_tc_deterministic(r):
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.rand(3000, 640, device="cuda", generator=g)
    v = torch.rand(3000, r, device="cuda", generator=g)
    w = torch.rand(r, 640, device="cuda", generator=g)
    a = one_iter(x, v, w, False)
    b = one_iter(x, v, w, False)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and a[2] == b[2]


@pytest.mark.parametrize("r", [64, 128])
def test_tc_strided_x_equals_contiguous(r):
    """X given as a column slice of a wider matrix (row stride ldx > n): the
    scale pass and the pre-split copy follow ldx, so V', W' and f equal the
    contiguous copy's bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(21)
    m, n = 1536, 640
    wide = torch.rand(m, n + 64, device="cuda", generator=g)
    v = torch.rand(m, r, device="cuda", generator=g)
    w = torch.rand(r, n, device="cuda", generator=g)
    xs = wide[:, :n]
    assert xs.stride(0) == n + 64
    (a, used) = tc_launched(lambda: one_iter(xs, v, w, force_simt=False))
    assert used
    b = one_iter(xs.contiguous(), v, w, force_simt=False)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and a[2] == b[2]


def test_tc_wide_row_dynamic_range():
    """Rows of X scaled by 2^u, u uniform in [-12, 12], and W entries spread
    over 2^[-6, 6]: one scaled split per operand still gives fp32-level
    agreement."""
    g = torch.Generator(device="cuda").manual_seed(5)
    m, n = 2048, 768
    rs = torch.exp2(torch.randint(-12, 13, (m, 1), device="cuda", generator=g).float())
    x = torch.rand(m, n, device="cuda", generator=g) * rs
    v = torch.rand(m, 64, device="cuda", generator=g) / rs.sqrt()
    w = torch.rand(64, n, device="cuda", generator=g) * torch.exp2(
        torch.randint(-6, 7, (64, n), device="cuda", generator=g).float())
    (vt, wt, ft), used = tc_launched(lambda: one_iter(x, v, w, force_simt=False))
    assert used
    vr, wr, fr = reference_iter(x, v, w)
    rel = lambda a, b: float((a.double() - b).norm() / b.norm())  # noqa: E731
    assert abs(ft - fr) / fr < 1e-5, (ft, fr)
    assert rel(vt, vr) < 5e-5 and rel(wt, wr) < 5e-5, (rel(vt, vr), rel(wt, wr))


def test_row_shards_sum_to_the_whole():
    """The multi-GPU NNMF decomposition on one device: 3 row shards run phase
    A on their own rows, the NCCL all-reduce is replaced by a sum of the
    fp64 reduction buffers, phase B once; equals the unsharded iteration."""
    g = torch.Generator(device="cuda").manual_seed(11)
    m, n = 3072, 1024
    x = torch.rand(m, n, device="cuda", generator=g)
    v = torch.rand(m, 64, device="cuda", generator=g)
    w = torch.rand(64, n, device="cuda", generator=g)
    vw, ww, fw = one_iter(x, v, w, force_simt=False)
    code, st = _lib.MMK_F32, _lib.stream_handle(torch, x.device)
    rl = _lib.load().mmk_nnmf_reduce_len(n, 64)
    total = torch.zeros(rl, dtype=torch.float64, device="cuda")
    vs = torch.empty_like(v)
    err = torch.zeros(2, dtype=torch.int64, device="cuda")
    for lo, hi in (P.shard_rows(m, 3, r) for r in range(3)):
        ws = torch.zeros(_lib.ws_bytes("mmk_nnmf_ws_bytes", code, hi - lo, n, 64),
                         dtype=torch.uint8, device="cuda")
        red = torch.zeros(rl, dtype=torch.float64, device="cuda")
        _lib.call("mmk_nnmf_iter_a", code, _lib.ptr(x[lo:hi]), n, _lib.ptr(v[lo:hi]),
                  _lib.ptr(w), _lib.ptr(vs[lo:hi]), hi - lo, n, 64, _lib.ptr(ws), ws.numel(),
                  _lib.ptr(red), _lib.ptr(err), st)
        total += red
    wo = torch.empty_like(w)
    f = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("mmk_nnmf_iter_b", code, _lib.ptr(w), _lib.ptr(wo), n, 64, _lib.ptr(total),
              _lib.ptr(f), _lib.ptr(err), st)
    torch.cuda.synchronize()
    rel = lambda a, b: float((a - b).norm() / b.norm())  # noqa: E731
    assert torch.equal(vs, vw)            # the V step is row-local: bitwise
    assert rel(wo, ww) < 1e-6 and abs(float(f) - fw) / fw < 1e-9


def test_ragged_shape_matches_fp64():
    """Odd tile counts (17 row tiles, 1160 = 18 x 64 + 8 columns: TMA
    out-of-bounds fill on both edges of every operand) over 30 iterations."""
    rng = np.random.default_rng(3)
    x = rng.random((2176, 1160)).astype(np.float32).astype(np.float64)
    v0 = rng.random((2176, 64)).astype(np.float32).astype(np.float64)
    w0 = rng.random((64, 1160)).astype(np.float32).astype(np.float64)
    prob = M.NnmfProblem(x=x, rank=64)
    s32, t32 = M.nnmf_run(prob, M.MmConfig(max_iters=30, epsilon=1e-300, monotone_tol=1e-6),
                          M.Backend(dtype="fp32"), state0=M.FactorPair(v0, w0))
    s64, t64 = M.nnmf_run(prob, M.MmConfig(max_iters=30, epsilon=1e-300),
                          M.Backend(dtype="fp64"), state0=M.FactorPair(v0, w0))
    err = np.max(np.abs(t32.objective_values - t64.objective_values) / t64.objective_values)
    vw = np.linalg.norm(s32.v @ s32.w - s64.v @ s64.w) / np.linalg.norm(s64.v @ s64.w)
    assert err < 1e-4 and vw < 1e-4, (err, vw)


def well_fit(m, n, seed, noise=0.01):
    """Rank-64 product with 1 % multiplicative noise and a start within 0.1 %
    of the truth: ||X||^2 / f ~ 1e4, where the Gram-trace objective would
    lose ~2.4e-8 x 1e4."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    vt = torch.rand(m, 64, device="cuda", generator=g)
    wt = torch.rand(64, n, device="cuda", generator=g)
    x = ((vt @ wt) * (1 + noise * torch.randn(m, n, device="cuda", generator=g))).clamp_min(0)
    v = vt * (1 + 0.001 * torch.rand(m, 64, device="cuda", generator=g))
    w = wt * (1 + 0.001 * torch.rand(64, n, device="cuda", generator=g))
    return x.contiguous(), v.contiguous(), w.contiguous()


@pytest.mark.parametrize("m,n", [(1024, 2048), (4104, 392), (2176, 1160)])
def test_objective_is_the_explicit_residual_on_well_fit_data(m, n):
    """f(V, W) from the V step equals the fp64 residual sum (x - v_i.w_j)^2 at
    ||X||^2 / f ~ 1e4 (the explicit residual + the exact correction for V's
    fp16 rounding, csrc/nnmf_tc.cu).  The one error left is the tensor
    cores' fp32 accumulation of R' = V_h W (a relative bias beta ~ 4e-7 from
    truncating adds), which enters f as 2 beta <VW, X - VW>: largest at this
    deliberately one-sided start (V, W both scaled up), ~0 near a stationary
    point, where <V, (X - VW) W^T> = 0 (KKT).  The Gram-trace form would be
    off by ~1e-2 here (it cancels ||X||^2 against a Q with the same bias)."""
    x, v, w = well_fit(m, n, m + n)
    (vt, wt, ft), used = tc_launched(lambda: one_iter(x, v, w, force_simt=False))
    assert used
    vr, wr, fr = reference_iter(x, v, w)
    ratio = float((x.double() ** 2).sum()) / fr
    assert ratio > 3e3, ratio
    assert abs(ft - fr) / fr < 1e-5, (ft, fr, abs(ft - fr) / fr)
    rel = lambda a, b: float((a.double() - b).norm() / b.norm())  # noqa: E731
    assert rel(vt, vr) < 3e-5 and rel(wt, wr) < 3e-5
    # a few iterations on (the scale mismatch of the start is gone)
    for _ in range(5):
        vt, wt, _ = one_iter(x, vt, wt, force_simt=False)
    _, _, ft = one_iter(x, vt, wt, force_simt=False)
    fr = float(((x.double() - vt.double() @ wt.double()) ** 2).sum())
    print(f"m={m} n={n}: |f - f64| / f64 after 5 iterations = {abs(ft - fr) / fr:.3e}")
    assert abs(ft - fr) / fr < 1e-6, (ft, fr, abs(ft - fr) / fr)


def test_engine_prologue_equals_per_iteration_path():
    """The device-loop engine prepares X once (engine prologue) and leaves the
    per-X launches out of its graph; the per-iteration path launches them
    every iteration (key check).  Same trace and factors, bit for bit."""
    rng = np.random.default_rng(12)
    x = rng.random((1280, 896)).astype(np.float32)
    v0 = rng.random((1280, 64)).astype(np.float32)
    w0 = rng.random((64, 896)).astype(np.float32)
    prob = M.NnmfProblem(x=x, rank=64)
    cfg = M.MmConfig(max_iters=12, epsilon=1e-300, monotone_tol=1e-6)
    a, ta = M.nnmf_run(prob, cfg, M.Backend(dtype="fp32", fused=True), state0=M.FactorPair(v0, w0))
    b, tb = M.nnmf_run(prob, cfg, M.Backend(dtype="fp32", fused=False), state0=M.FactorPair(v0, w0))
    assert np.array_equal(ta.objective_values, tb.objective_values)
    assert np.array_equal(a.v, b.v) and np.array_equal(a.w, b.w)
