"""The headline path -- fp32 rank-64 NNMF on the tensor cores (csrc/nnmf_tc.cu)
-- pinned against the REFERENCE and at BASELINE config 4 itself.

* tests/golden/nnmf_r64_{uniform,wellfit}.npz: the reference's own run_mm
  (_FrobeniusNnmf, nnmf.py:143-159, fp64) on a tensor-core-eligible shape
  (1024 x 2048, rank 64: 8 row tiles, 16 column blocks, 32 K-blocks), made
  by tests/golden/make_golden.py; uniform data for 500 iterations and
  well-fit data (rank-64 product + 1 % noise, ||X||^2 / f ~ 1e4, the regime
  where a Gram-trace objective cancels) for 1000.  The fp32 GPU run from the
  same fp32-exact start matches the trace and V W to 1e-4 with descent
  checked at monotone_tol = 1e-6 (the fp32 tolerance of DESIGN.md); fp64 to
  1e-9.
* C4 (131072 x 16384, r = 64, fp32) at full size: size-independent
  properties -- monotone descent over 20 fused iterations, the fused
  objective at iterations 0 and 20 equal to an independent fp64 residual
  (computed here in row blocks with torch) to 1e-6, and bitwise run-to-run
  determinism of trace and factors.
"""

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib

pytestmark = pytest.mark.gpu


def tc_ran(fn):
    lib = _lib.load()
    lib.mmk_prof_enable(1)
    try:
        out = fn()
        torch.cuda.synchronize()
    finally:
        lib.mmk_prof_enable(0)
    prof = _lib.prof_report()
    # a fused run's iterations are graph replays (not profiled); its per-X
    # prologue (the pre-split copy) is a tensor-core-path launch
    return out, "nnmf_vstep_tc" in prof or "nnmf_presplit_cached" in prof


@pytest.mark.parametrize("kind,iters", [("uniform", 500), ("wellfit", 1000)])
def test_r64_fp32_matches_reference_golden(kind, iters):
    gold = G.load(f"nnmf_r64_{kind}")
    x, v0, w0 = G.r64_inputs(kind)
    assert G.digest(x) == str(gold["x_digest"]) and G.digest(v0) == str(gold["v0_digest"])
    assert G.digest(w0) == str(gold["w0_digest"])
    prob = M.NnmfProblem(x=x, rank=64)
    cfg = M.MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6)
    (st, tr), used = tc_ran(lambda: M.nnmf_run(prob, cfg, M.Backend(dtype="fp32", fused=False),
                                               state0=M.FactorPair(v0, w0)))
    assert used, "the tensor-core path did not run"
    ref = gold["trace"]
    assert tr.objective_values.shape == ref.shape
    err = np.max(np.abs(tr.objective_values - ref) / ref)
    assert err < 1e-4, err
    vw, rvw = st.v @ st.w, gold["v"] @ gold["w"]
    assert G.rel(vw, rvw) < 1e-4, G.rel(vw, rvw)
    # the fused device loop (the default) gives the same run bit for bit
    st2, tr2 = M.nnmf_run(prob, cfg, M.Backend(dtype="fp32"), state0=M.FactorPair(v0, w0))
    assert np.array_equal(tr2.objective_values, tr.objective_values)
    assert np.array_equal(st2.v, st.v) and np.array_equal(st2.w, st.w)


@pytest.mark.parametrize("kind", ["uniform", "wellfit"])
def test_r64_fp64_matches_reference_golden(kind):
    gold = G.load(f"nnmf_r64_{kind}")
    x, v0, w0 = G.r64_inputs(kind)
    iters = len(gold["trace"]) - 1
    st, tr = M.nnmf_run(M.NnmfProblem(x=x, rank=64), M.MmConfig(max_iters=iters, epsilon=1e-300),
                        M.Backend(dtype="fp64"), state0=M.FactorPair(v0, w0))
    assert np.max(np.abs(tr.objective_values - gold["trace"]) / gold["trace"]) < 1e-9
    assert G.rel(st.v @ st.w, gold["v"] @ gold["w"]) < 1e-9


def residual64(x, v, w, block=8192):
    """sum (x - v w)^2 in fp64, row blocks (independent of the kernels)."""
    f = 0.0
    wd = w.double()
    for i in range(0, x.shape[0], block):
        d = x[i:i + block].double() - v[i:i + block].double() @ wd
        f += float((d * d).sum())
    return f


def test_c4_full_shape_properties():
    m, n, r, iters = 131072, 16384, 64, 20
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(m, n, device="cuda", generator=g)
    v0 = torch.rand(m, r, device="cuda", generator=g)
    w0 = torch.rand(r, n, device="cuda", generator=g)
    prob = M.NnmfProblem(x=x, rank=r)
    cfg = M.MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6)
    be = M.Backend(dtype="fp32", device=0)
    (a, ta), used = tc_ran(lambda: M.nnmf_run(prob, cfg, be, state0=M.FactorPair(v0, w0)))
    assert used
    fv = ta.objective_values
    assert len(fv) == iters + 1 and np.all(np.diff(fv) <= 1e-6 * (1 + np.abs(fv[:-1])))
    # the objective is the explicit residual; its one systematic error is the
    # fp32 tensor accumulation of V_h W (relative bias beta ~ 2e-7), which
    # enters as 2 beta <VW, X - VW> / f -- largest at this far-off start,
    # where X - VW ~ -VW
    f0 = residual64(x, v0, w0)
    assert abs(fv[0] - f0) / f0 < 1e-6, (fv[0], f0)
    vt = torch.as_tensor(a.v, device="cuda").float()
    wt = torch.as_tensor(a.w, device="cuda").float()
    fn = residual64(x, vt, wt)
    # the trace's last entry is f at the returned state
    assert abs(fv[-1] - fn) / fn < 1e-6, (fv[-1], fn)
    # bitwise run to run (this caught a missing generic -> async proxy fence
    # between the residual warps' reads of an X slot and its next TMA fill)
    b, tb = M.nnmf_run(prob, cfg, be, state0=M.FactorPair(v0, w0))
    assert np.array_equal(ta.objective_values, tb.objective_values)
    assert torch.equal(torch.as_tensor(a.v), torch.as_tensor(b.v))
    assert torch.equal(torch.as_tensor(a.w), torch.as_tensor(b.w))
