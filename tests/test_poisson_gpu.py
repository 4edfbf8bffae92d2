"""Poisson-loss NNMF (reference nnmf.py:178-265) on the
GPU against golden vectors the reference produced (tests/golden) and the
CPU oracle, plus the reference's own known answers (test_nnmf.py:145-175,
test_acceptance.py criteria 1 and 3c).  Tolerances: 1e-9 relative in fp64,
1e-4 in fp32 (trace max-relative; final iterate relative Frobenius, V W for
the gauge-free product)."""

import numpy as np
import pytest

import golden_io as G
import paper_1003_3272_b200 as M
from oracle import oracle as O
from paper_1003_3272_b200 import Backend, MmConfig

pytestmark = pytest.mark.gpu

FP64 = Backend(dtype="fp64")
FP32 = Backend(dtype="fp32")


def trace_err(got, want):
    return float(np.max(np.abs(np.asarray(got) - want) / np.abs(want)))


def test_poisson_small_seeded_run():
    g = G.load("poisson_small")
    prob = M.NnmfProblem(x=g["x"], rank=3)
    st, tr = M.nnmf_poisson_run(prob, MmConfig(max_iters=40, seed=4), FP64)
    assert trace_err(tr.objective_values, g["trace"]) <= 1e-12
    assert G.rel(st.v, g["v"]) <= 1e-11 and G.rel(st.w, g["w"]) <= 1e-11


@pytest.mark.parametrize("dtype,fused", [("fp64", True), ("fp64", False), ("fp32", True)])
def test_poisson_c1_100_iters(dtype, fused):
    g = G.load("poisson_c1")
    x, v0, w0 = G.poisson_c1_inputs()
    prob = M.NnmfProblem(x=x, rank=10)
    tol = 1e-9 if dtype == "fp64" else 1e-4
    cfg = MmConfig(max_iters=100, epsilon=1e-300,
                   monotone_tol=1e-12 if dtype == "fp64" else 1e-6)
    st, tr = M.nnmf_poisson_run(prob, cfg, Backend(dtype=dtype, fused=fused),
                                state0=M.FactorPair(v0, w0))
    assert tr.iters == 100
    assert trace_err(tr.objective_values, g["trace"]) <= tol
    assert G.rel(st.v @ st.w, g["v"] @ g["w"]) <= tol
    if dtype == "fp64":
        assert G.rel(st.v, g["v"]) <= tol and G.rel(st.w, g["w"]) <= tol


def test_poisson_kats():
    rng = np.random.default_rng(8)
    v = rng.random((5, 2)) + 0.1
    w = rng.random((2, 6)) + 0.1
    x = O.matmul(v, w)
    v2, w2 = M.nnmf_poisson_update(x, v, w, FP64)
    np.testing.assert_allclose(v2, v, rtol=4e-16 * 8)
    np.testing.assert_allclose(w2, w, rtol=4e-16 * 8)
    v2, w2 = M.nnmf_poisson_update(np.array([[4.0]]), np.array([[1.0]]), np.array([[1.0]]), FP64)
    assert v2[0, 0] == 2.0
    f = M.nnmf_poisson_objective(np.array([[2.0, 0.0]]), np.array([[1.0]]),
                                 np.array([[2.0, 3.0]]), FP64)
    assert abs(f - (2.0 * np.log(2.0) - 2.0 - 3.0)) <= 1e-15


def test_poisson_ascent_and_oracle_updates():
    rng = np.random.default_rng(9)
    for _ in range(20):
        p, q = (int(a) for a in rng.integers(2, 9, size=2))
        r = int(rng.integers(1, min(p, q) + 1))
        x = np.floor(rng.random((p, q)) * 3.0)
        v, w = rng.random((p, r)) + 0.05, rng.random((r, q)) + 0.05
        before = M.nnmf_poisson_objective(x, v, w, FP64)
        assert abs(before - O.nnmf_poisson_objective(x, v, w)) <= 1e-12 * (1 + abs(before))
        v2, w2 = M.nnmf_poisson_update(x, v, w, FP64)
        ov, ow = O.nnmf_poisson_update(x, v, w)
        np.testing.assert_allclose(v2, ov, rtol=1e-12)
        np.testing.assert_allclose(w2, ow, rtol=1e-12)
        after = M.nnmf_poisson_objective(x, v2, w2, FP64)
        assert after >= before - 1e-12 * (1.0 + abs(before))


def test_poisson_zero_mean_errors():
    x = np.array([[1.0, 2.0], [0.0, 3.0]])
    v = np.array([[0.0], [1.0]])
    w = np.array([[1.0, 1.0]])
    with pytest.raises(M.NumericsError, match="zero reconstruction mean at a positive"):
        M.nnmf_poisson_objective(x, v, w, FP64)
    with pytest.raises(M.DomainError):
        M.nnmf_poisson_update(-x, v + 1.0, w, FP64)


def test_poisson_run_monotone_random():
    rng = np.random.default_rng(10)
    for seed in range(10):
        p, q = (int(a) for a in rng.integers(2, 7, size=2))
        r = int(rng.integers(1, min(p, q) + 1))
        prob = M.NnmfProblem(x=np.floor(rng.random((p, q)) * 6.0), rank=r)
        _, tr = M.nnmf_poisson_run(prob, MmConfig(max_iters=25, seed=seed), FP64)
        d = np.diff(tr.objective_values)
        assert np.all(d >= -1e-12 * (1.0 + np.abs(tr.objective_values[:-1])))
