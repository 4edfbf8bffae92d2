"""CUDA path vs the reference: golden vectors from the reference itself
(tests/golden, 1000 fixed iterations at the paper shapes) plus the
reference's own known-answer tests, through the public drop-in API.

Tolerances (BASELINE.json north star): fp64 mode 1e-9 relative, fp32 mode
1e-4 relative, on the objective trace (max over iterations) and on the final
iterate (relative Frobenius; for NNMF also V*W, the gauge-invariant product,
SURVEY.md section 7.3-1).
"""

import numpy as np
import pytest

import golden_io as G
from oracle import oracle as O
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import Backend, MmConfig

pytestmark = pytest.mark.gpu

FP64 = Backend(dtype="fp64")
FP32 = Backend(dtype="fp32")
TOL = {"fp64": 1e-9, "fp32": 1e-4}
FIXED = MmConfig(max_iters=1000, epsilon=1e-300)


def trace_err(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, (got.shape, want.shape)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


def monotone(values, direction, tol):
    d = np.diff(values)
    slack = tol * (1.0 + np.abs(values[:-1]))
    return bool(np.all(d <= slack)) if direction == "minimize" else bool(np.all(d >= -slack))


# ----------------------------------------------------------------------------- NNMF
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
@pytest.mark.parametrize("fused", [True, False])
def test_nnmf_c1_1000_iters(dtype, fused):
    g = G.load("nnmf_c1")
    x, v0, w0 = G.c1_inputs()
    be = Backend(dtype=dtype, fused=fused)
    cfg = FIXED if dtype == "fp64" else MmConfig(max_iters=1000, epsilon=1e-300,
                                                 monotone_tol=1e-6)
    st, tr = M.nnmf_run(M.NnmfProblem(x=x, rank=10), cfg, be, state0=M.FactorPair(v0, w0))
    tol = TOL[dtype]
    assert tr.iters == 1000
    assert trace_err(tr.objective_values, g["trace"]) <= tol
    assert G.rel(st.v @ st.w, g["v"] @ g["w"]) <= tol
    assert G.rel(st.v, g["v"]) <= tol and G.rel(st.w, g["w"]) <= tol
    assert monotone(tr.objective_values, "minimize", 1e-12 if dtype == "fp64" else 1e-6)


def test_nnmf_small_seeded_run():
    g = G.load("nnmf_small")
    st, tr = M.nnmf_run(M.NnmfProblem(x=g["x"], rank=3), MmConfig(max_iters=25, seed=5), FP64)
    assert trace_err(tr.objective_values, g["trace"]) <= 1e-12
    assert G.rel(st.v, g["v"]) <= 1e-12 and G.rel(st.w, g["w"]) <= 1e-12


def test_nnmf_objective_hand_values():
    x = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert M.nnmf_objective(x, np.array([[1.0], [1.0]]), np.array([[1.0, 1.0]])) == 14.0
    assert M.nnmf_objective(np.eye(2), np.zeros((2, 1)), np.zeros((1, 2))) == 2.0
    rng = np.random.default_rng(0)
    v, w = rng.random((5, 2)), rng.random((2, 4))
    assert M.nnmf_objective(v @ w, v, w) <= 1e-28


def test_nnmf_scalar_updates_and_fixed_point():
    x = np.array([[2.0]])
    assert M.nnmf_update_v(x, np.array([[1.0]]), np.array([[1.0]]))[0, 0] == 2.0
    assert M.nnmf_update_w(x, np.array([[2.0]]), np.array([[1.0]]))[0, 0] == 1.0
    # the reference's bitwise fixed point (test_nnmf.py:46-52): X = VW from its
    # own tree-summed matmul (the oracle's, bitwise the reference's); the fp64
    # single ops run in the reference's arithmetic order (csrc/nnmf_ref.cu)
    rng = np.random.default_rng(1)
    v, w = rng.random((6, 3)), rng.random((3, 5))
    x = O.matmul(v, w)
    assert np.array_equal(M.nnmf_update_v(x, v, w), v)
    assert np.array_equal(M.nnmf_update_w(x, v, w), w)


@pytest.mark.parametrize("m,n,r", [(6, 5, 3), (37, 29, 7), (130, 257, 64), (64, 2049, 5),
                                   (1, 1, 1), (513, 3, 17)])
def test_nnmf_fp64_single_ops_bitwise_reference(m, n, r):
    """fp64 nnmf_objective / update_v / update_w / gradient equal the
    reference's arithmetic bit for bit (the oracle is bitwise pinned to it):
    tree-summed inner products, explicitly rounded elementwise ops, and the
    halving-with-carry reduction of the objective over m n terms (the odd
    sizes exercise the carried tails)."""
    rng = np.random.default_rng(m * 1000 + n + r)
    x, v, w = rng.random((m, n)) * 3.0, rng.random((m, r)), rng.random((r, n))
    assert M.nnmf_objective(x, v, w) == O.nnmf_objective(x, v, w)
    assert np.array_equal(M.nnmf_update_v(x, v, w), O.nnmf_update_v(x, v, w))
    assert np.array_equal(M.nnmf_update_w(x, v, w), O.nnmf_update_w(x, v, w))
    gv, gw = M.nnmf_gradient(x, v, w)
    ov, ow = O.nnmf_gradient(x, v, w)
    assert np.array_equal(gv, ov) and np.array_equal(gw, ow)


def test_nnmf_zero_entries_absorb_and_domain():
    rng = np.random.default_rng(2)
    x = rng.random((5, 6)) * 2.0
    v = rng.random((5, 3)) + 0.05
    w = rng.random((3, 6)) + 0.05
    v[2, 1] = 0.0
    w[0, 3] = 0.0
    assert M.nnmf_update_v(x, v, w)[2, 1] == 0.0
    assert M.nnmf_update_w(x, M.nnmf_update_v(x, v, w), w)[0, 3] == 0.0
    with pytest.raises(M.DomainError):
        M.nnmf_update_v(np.array([[1.0, -0.5]]), np.ones((1, 1)), np.ones((1, 2)))
    with pytest.raises(M.ShapeError):
        M.nnmf_objective(np.ones((3, 3)), np.ones((3, 2)), np.ones((2, 4)))


def test_nnmf_descent_per_half_update():
    rng = np.random.default_rng(3)
    for _ in range(20):
        p, q, r = int(rng.integers(2, 8)), int(rng.integers(2, 8)), int(rng.integers(1, 4))
        x = rng.random((p, q)) * 2.0
        v = rng.random((p, r)) + 0.05
        w = rng.random((r, q)) + 0.05
        f0 = M.nnmf_objective(x, v, w)
        v2 = M.nnmf_update_v(x, v, w)
        f1 = M.nnmf_objective(x, v2, w)
        assert f1 <= f0 + 1e-12 * (1.0 + abs(f0))
        w2 = M.nnmf_update_w(x, v2, w)
        assert M.nnmf_objective(x, v2, w2) <= f1 + 1e-12 * (1.0 + abs(f1))


def test_nnmf_rank_one_recovery():
    rng = np.random.default_rng(5)
    x = np.outer(rng.random(7) + 0.2, rng.random(6) + 0.2)
    _, tr = M.nnmf_run(M.NnmfProblem(x=x, rank=1), MmConfig(epsilon=1e-13, max_iters=20_000,
                                                            seed=7), FP64)
    assert tr.objective_values[-1] < 1e-8
    assert monotone(tr.objective_values, "minimize", 1e-12)


@pytest.mark.parametrize("fused", [True, False])
def test_nnmf_restartability_bitwise(fused):
    rng = np.random.default_rng(12)
    prob = M.NnmfProblem(x=rng.random((7, 6)), rank=2)
    be = Backend(fused=fused)
    s0 = M.nnmf._initial_factors(prob, 8)
    joined, tj = M.nnmf_run(prob, MmConfig(max_iters=20, epsilon=1e-300), be, state0=s0)
    mid, t1 = M.nnmf_run(prob, MmConfig(max_iters=9, epsilon=1e-300), be, state0=s0)
    fin, t2 = M.nnmf_run(prob, MmConfig(max_iters=11, epsilon=1e-300), be, state0=mid)
    assert np.array_equal(fin.v, joined.v) and np.array_equal(fin.w, joined.w)
    assert np.array_equal(np.concatenate([t1.objective_values, t2.objective_values[1:]]),
                          tj.objective_values)


@pytest.mark.parametrize("engine", ["graph", "persistent"])
def test_fused_and_per_iteration_paths(engine, monkeypatch):
    """The graph engine replays the per-iteration kernels: bitwise equal.  The
    persistent small-problem engine (csrc/nnmf_small.cu) has its own fixed
    reduction order: equal to rounding (fp64)."""
    if engine == "graph":
        monkeypatch.setenv("MMK_SMALL_ENGINE", "0")
    x, v0, w0 = G.c1_inputs()
    prob = M.NnmfProblem(x=x, rank=10)
    cfg = MmConfig(max_iters=50, epsilon=1e-300)
    a, ta = M.nnmf_run(prob, cfg, Backend(fused=True), state0=M.FactorPair(v0, w0))
    b, tb = M.nnmf_run(prob, cfg, Backend(fused=False), state0=M.FactorPair(v0, w0))
    if engine == "graph":
        assert np.array_equal(ta.objective_values, tb.objective_values)
        assert np.array_equal(a.v, b.v) and np.array_equal(a.w, b.w)
    else:
        assert G.rel(ta.objective_values, tb.objective_values) <= 1e-13
        assert G.rel(a.v, b.v) <= 1e-12 and G.rel(a.w, b.w) <= 1e-12


@pytest.mark.parametrize("dtype", ["fp32", "fp64"])
def test_persistent_engine_pauses_and_restarts(dtype, monkeypatch):
    """Batches (host drains of the trace) and restarts do not change the
    persistent engine's results: 9000 iterations in 3 batches of 4096, and two
    runs of 4500 from the first's end state, equal one run bitwise; the graph
    engine agrees to rounding."""
    x, v0, w0 = G.c1_inputs()
    prob = M.NnmfProblem(x=x, rank=10)
    be = Backend(dtype=dtype)
    cfg = MmConfig(max_iters=9000, epsilon=1e-300, monotone_tol=1e-6)
    full, tf = M.nnmf_run(prob, cfg, be, state0=M.FactorPair(v0, w0))
    half = MmConfig(max_iters=4500, epsilon=1e-300, monotone_tol=1e-6)
    s1, t1 = M.nnmf_run(prob, half, be, state0=M.FactorPair(v0, w0))
    s2, t2 = M.nnmf_run(prob, half, be, state0=s1)
    assert np.array_equal(s2.v, full.v) and np.array_equal(s2.w, full.w)
    assert np.array_equal(np.concatenate([t1.objective_values, t2.objective_values[1:]]),
                          tf.objective_values)
    monkeypatch.setenv("MMK_SMALL_ENGINE", "0")
    g, tg = M.nnmf_run(prob, cfg, be, state0=M.FactorPair(v0, w0))
    tol = 1e-3 if dtype == "fp32" else 1e-10
    assert G.rel(tg.objective_values, tf.objective_values) <= tol
    assert G.rel(g.v @ g.w, full.v @ full.w) <= tol


# ----------------------------------------------------------------------------- PET
@pytest.mark.parametrize("mu", [0.0, 1e-7, 1e-6, 1e-5])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_pet_c2_1000_iters(mu, dtype):
    g = G.load("pet_c2")
    e, y, nbrs = G.c2_inputs()
    prob = M.PetProblem(e=e, y=y, mu=mu, neighborhoods=nbrs)
    cfg = FIXED if dtype == "fp64" else MmConfig(max_iters=1000, epsilon=1e-300,
                                                 monotone_tol=1e-6)
    lam, tr = M.pet_run(prob, cfg, Backend(dtype=dtype, pet_kernel="dense"))
    tol = TOL[dtype]
    assert trace_err(tr.objective_values, g[f"trace_{mu:g}"]) <= tol
    assert G.rel(lam, g[f"lam_{mu:g}"]) <= tol


def test_pet_c2_time_to_tolerance():
    g = G.load("pet_c2_converge")
    e, y, nbrs = G.c2_inputs()
    lam, tr = M.pet_run(M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=nbrs), MmConfig(), FP64)
    assert tr.converged and abs(tr.iters - int(g["iters"])) <= 2
    assert G.rel(lam, g["lam"]) <= 1e-7


@pytest.mark.parametrize("mu", [0.0, 1e-7, 1e-6, 1e-5])
def test_pet_small_150(mu):
    g = G.load("pet_small")
    prob = M.PetProblem(e=g["e"], y=g["y"], mu=mu, neighborhoods=M.build_neighborhoods(5))
    lam, tr = M.pet_run(prob, MmConfig(max_iters=150), FP64)
    assert trace_err(tr.objective_values, g[f"trace_{mu:g}"]) <= 1e-11
    assert G.rel(lam, g[f"lam_{mu:g}"]) <= 1e-10


def _small_pet(rng, n_pixels=4, n_rays=10, mu=0.0, nbrs=None, y=None):
    e = rng.random((n_rays, n_pixels)) + 0.05
    e /= e.sum(axis=0)
    if y is None:
        y = np.floor(rng.random(n_rays) * 8.0)
    if nbrs is None:
        nbrs = [[j for j in (i - 1, i + 1) if 0 <= j < n_pixels] for i in range(n_pixels)]
    return M.PetProblem(e=e, y=y, mu=mu, neighborhoods=nbrs)


def test_pet_kats():
    rng = np.random.default_rng(6)
    e = rng.random((9, 1))
    e /= e.sum(axis=0)
    y = np.floor(rng.random(9) * 7.0)
    lam1 = M.pet_update(np.array([1.0]), M.PetProblem(e=e, y=y, mu=0.0, neighborhoods=[[]]))
    assert abs(lam1[0] - y.sum()) <= 1e-14 * (1.0 + y.sum())
    yy = np.array([3.0, 5.0, 2.0])
    np.testing.assert_allclose(M.pet_loglik(yy, np.eye(3), yy), np.sum(yy * np.log(yy) - yy),
                               rtol=1e-14)
    rng = np.random.default_rng(5)
    e = rng.random((5, 2)) + 0.1
    e /= e.sum(axis=0)
    y = np.floor(rng.random(5) * 4.0)
    prob = M.PetProblem(e=e, y=y, mu=2.0, neighborhoods=[[1], [0]])
    lam = np.array([1.0, 3.0])
    np.testing.assert_allclose(M.pet_penalized_objective(lam, prob),
                               M.pet_loglik(lam, e, y) - 4.0, rtol=1e-14)


def test_pet_loglik_direct_sum_and_errors():
    rng = np.random.default_rng(2)
    e = rng.random((7, 4)) + 0.02
    e /= e.sum(axis=0)
    y = np.floor(rng.random(7) * 6.0)
    lam = rng.random(4) + 0.3
    means = e @ lam
    want = sum(-m if yi == 0 else yi * np.log(m) - m for yi, m in zip(y, means))
    assert abs(M.pet_loglik(lam, e, y) - want) <= 1e-12 * (1.0 + abs(want))
    with pytest.raises(M.NumericsError):
        M.pet_loglik(np.array([1.0]), np.array([[1.0], [0.0]]), np.array([1.0, 2.0]))
    prob = _small_pet(np.random.default_rng(10))
    with pytest.raises(M.DomainError, match="pixel 2"):
        M.pet_update(np.array([1.0, 1.0, 0.0, 1.0]), prob)
    with pytest.raises(M.ShapeError):
        M.pet_update(np.ones(3), prob)


def test_pet_isolated_pixel_and_vanishing_penalty():
    rng = np.random.default_rng(9)
    prob = _small_pet(rng, n_pixels=1, n_rays=6, mu=0.5, nbrs=[[]])
    base = M.PetProblem(e=prob.e, y=prob.y, mu=0.0, neighborhoods=[[]])
    lam = np.array([0.8])
    assert M.pet_update(lam, prob)[0] == pytest.approx(M.pet_update(lam, base)[0], rel=1e-15)
    rng = np.random.default_rng(8)
    base = _small_pet(rng, mu=0.0)
    tiny = M.PetProblem(e=base.e, y=base.y, mu=1e-12, neighborhoods=base.neighborhoods)
    lam = rng.random(4) + 0.2
    np.testing.assert_allclose(M.pet_update(lam, tiny), M.pet_update(lam, base), rtol=1e-6)


# ----------------------------------------------------------------------------- MDS
@pytest.mark.parametrize("dim", [2, 3, 4, 5, 10])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_mds_c3_1000_iters(dim, dtype):
    g = G.load("mds_c3")
    diss, theta0 = G.c3_inputs(dim)
    prob = M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=dim)
    cfg = FIXED if dtype == "fp64" else MmConfig(max_iters=1000, epsilon=1e-300,
                                                 monotone_tol=1e-6)
    theta, tr = M.mds_run(prob, cfg, Backend(dtype=dtype), theta0=theta0)
    tol = TOL[dtype]
    assert trace_err(tr.objective_values, g[f"trace_{dim}"]) <= tol
    assert G.rel(theta, g[f"theta_{dim}"]) <= tol


def test_mds_small_seeded_and_anchored():
    g = G.load("mds_small")
    prob = M.MdsProblem(weights=np.ones((9, 9)) - np.eye(9), dissimilarities=g["y"], p=3)
    theta, tr = M.mds_run(prob, MmConfig(max_iters=40, seed=2), FP64)
    assert trace_err(tr.objective_values, g["trace"]) <= 1e-12
    assert G.rel(theta, g["theta"]) <= 1e-11
    anchored, _ = M.mds_run(prob, MmConfig(max_iters=40, seed=2), FP64, anchor=True)
    assert np.array_equal(anchored[:, 0], np.zeros(3))
    assert G.rel(anchored, g["anchored"]) <= 1e-10


def test_mds_kats():
    two = M.MdsProblem(weights=np.array([[0.0, 1.0], [1.0, 0.0]]),
                       dissimilarities=np.array([[0.0, 2.0], [2.0, 0.0]]), p=1)
    assert M.stress(np.array([[0.0, 1.0]]), two) == 1.0
    new = M.mds_update(np.array([[0.0, 1.0]]), two)
    np.testing.assert_allclose(new, [[-0.5, 1.5]], atol=1e-15)
    assert M.stress(new, two) <= 1e-30
    d = 1.75
    fix = M.MdsProblem(weights=np.array([[0.0, 1.0], [1.0, 0.0]]),
                       dissimilarities=np.array([[0.0, d], [d, 0.0]]), p=1)
    np.testing.assert_allclose(M.mds_update(np.array([[0.0, d]]), fix), [[0.0, d]], atol=1e-15)
    coupled = M.MdsProblem(weights=np.array([[0.0, 1.0], [1.0, 0.0]]),
                           dissimilarities=np.array([[0.0, 2.0], [2.0, 0.0]]), p=2)
    with pytest.raises(M.NumericsError, match="0 and 1"):
        M.mds_update(np.array([[0.3, 0.3], [-0.2, -0.2]]), coupled)
    y = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0], [1.0, 1.0, 0.0]])
    free = M.MdsProblem(weights=np.ones((3, 3)) - np.eye(3), dissimilarities=y, p=1)
    assert np.all(np.isfinite(M.mds_update(np.array([[0.5, 0.5, -0.5]]), free)))


def _direct_update(theta, w, y):
    p, q = theta.shape
    out = np.empty_like(theta)
    for i in range(q):
        acc = np.zeros(p)
        for j in range(q):
            if j == i:
                continue
            diff = theta[:, i] - theta[:, j]
            if w[i, j] * y[i, j] > 0.0:
                acc += w[i, j] * y[i, j] * diff / np.linalg.norm(diff)
            acc += w[i, j] * (theta[:, i] + theta[:, j])
        out[:, i] = acc / (2.0 * w[i].sum())
    return out


def test_mds_update_matches_direct_sums_weighted():
    rng = np.random.default_rng(2)
    for weighted in (False, True):
        for _ in range(10):
            q = 6
            y = rng.random((q, q)) * 2.0
            y = (y + y.T) / 2.0
            np.fill_diagonal(y, 0.0)
            w = np.ones((q, q)) - np.eye(q)
            if weighted:
                w = rng.random((q, q)) + 0.1
                w = (w + w.T) / 2.0
                np.fill_diagonal(w, 0.0)
            prob = M.MdsProblem(weights=w, dissimilarities=y, p=3)
            theta = rng.standard_normal((3, q))
            want = _direct_update(theta, w, y)
            got = M.mds_update(theta, prob)
            assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


def test_mds_descent_and_recovery():
    rng = np.random.default_rng(3)
    for _ in range(20):
        q, p = int(rng.integers(3, 9)), int(rng.integers(1, 4))
        y = rng.random((q, q)) * 2.0
        y = (y + y.T) / 2.0
        np.fill_diagonal(y, 0.0)
        prob = M.MdsProblem(weights=np.ones((q, q)) - np.eye(q), dissimilarities=y, p=p)
        theta = rng.uniform(-1.0, 1.0, size=(p, q))
        before = M.stress(theta, prob)
        assert M.stress(M.mds_update(theta, prob), prob) <= before + 1e-12 * (1.0 + before)
    pts = np.random.default_rng(8).standard_normal((2, 7))
    yy = np.linalg.norm(pts[:, :, None] - pts[:, None, :], axis=0)
    prob = M.MdsProblem(weights=np.ones((7, 7)) - np.eye(7), dissimilarities=yy, p=2)
    best = min(M.mds_run(prob, MmConfig(epsilon=1e-13, max_iters=20_000, seed=s), FP64)[1]
               .objective_values[-1] for s in range(5))
    assert best < 1e-6


# ----------------------------------------------------------------------------- driver on device
def test_monotonicity_error_is_raised_by_fused_engine():
    # a problem whose objective is forced up: fp32 data with an absurdly
    # tight slack cannot hold; the engine must raise with the iteration
    x, v0, w0 = G.c1_inputs()
    cfg = MmConfig(max_iters=400, epsilon=1e-300, monotone_tol=0.0)
    try:
        M.nnmf_run(M.NnmfProblem(x=x, rank=10), cfg, Backend(dtype="fp32"),
                   state0=M.FactorPair(v0, w0))
    except M.MonotonicityError as exc:
        assert exc.iteration >= 1
        assert exc.current > exc.previous


def test_run_to_run_bitwise_determinism():
    diss, theta0 = G.c3_inputs(3)
    prob = M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=3)
    cfg = MmConfig(max_iters=200, epsilon=1e-300)
    a, ta = M.mds_run(prob, cfg, FP32, theta0=theta0)
    b, tb = M.mds_run(prob, cfg, FP32, theta0=theta0)
    assert np.array_equal(a, b) and np.array_equal(ta.objective_values, tb.objective_values)


# ----------------------------------------------------------------------------- sparse PET
@pytest.mark.parametrize("mu", [0.0, 1e-5])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_pet_c2_sparse_projector(mu, dtype):
    """CSR/CSC projector against the same golden traces as
    the dense path (BASELINE config 2, 1000 iterations)."""
    g = G.load("pet_c2")
    e, y, nbrs = G.c2_inputs()
    prob = M.PetProblem(e=e, y=y, mu=mu, neighborhoods=nbrs)
    cfg = FIXED if dtype == "fp64" else MmConfig(max_iters=1000, epsilon=1e-300,
                                                 monotone_tol=1e-6)
    be = Backend(dtype=dtype, pet_kernel="sparse")
    lam, tr = M.pet_run(prob, cfg, be)
    tol = TOL[dtype]
    assert trace_err(tr.objective_values, g[f"trace_{mu:g}"]) <= tol
    assert G.rel(lam, g[f"lam_{mu:g}"]) <= tol
    # the auto switch picks the sparse kernels for the ~1 % dense Siddon matrix
    assert M.pet._use_sparse(prob, Backend(dtype=dtype))


@pytest.mark.parametrize("solver", ["mds", "pet", "poisson"])
def test_persistent_engines_match_graph_engine(solver, monkeypatch):
    """The persistent MDS (rows) and sparse-PET engines against the graph
    engine: traces and states equal to rounding; 9000 MDS iterations cross two
    batch pauses and equal two restarted runs of 4500 bitwise."""
    be = Backend(dtype="fp64")
    if solver == "mds":
        diss, theta0 = G.c3_inputs(3)
        prob = M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=3)
        run = lambda cfg, t0=theta0: M.mds_run(prob, cfg, be, theta0=t0)
        iters = 9000
    elif solver == "pet":
        e, y, nbrs = G.c2_inputs()
        prob = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=nbrs)
        run = lambda cfg: M.pet_run(prob, cfg, Backend(dtype="fp64", pet_kernel="sparse"))
        iters = 2000
    else:
        x, v0, w0 = G.poisson_c1_inputs()
        prob = M.NnmfProblem(x=x, rank=10)
        run = lambda cfg, s0=M.FactorPair(v0, w0): M.nnmf_poisson_run(prob, cfg, be, state0=s0)
        iters = 9000
    cfg = MmConfig(max_iters=iters, epsilon=1e-300)
    s_p, t_p = run(cfg)
    flat = (lambda s: np.concatenate([s.v.ravel(), s.w.ravel()])) if solver == "poisson" \
        else (lambda s: np.asarray(s))
    if solver in ("mds", "poisson"):
        half = MmConfig(max_iters=iters // 2, epsilon=1e-300)
        s1, t1 = run(half)
        s2, t2 = run(half, s1)
        assert np.array_equal(flat(s2), flat(s_p))
        assert np.array_equal(np.concatenate([t1.objective_values, t2.objective_values[1:]]),
                              t_p.objective_values)
    monkeypatch.setenv("MMK_SMALL_ENGINE", "0")
    s_g, t_g = run(cfg)
    assert G.rel(t_p.objective_values, t_g.objective_values) <= 1e-12
    if solver == "poisson":
        assert G.rel(s_p.v @ s_p.w, s_g.v @ s_g.w) <= 1e-9
    else:
        assert G.rel(s_p, s_g) <= 1e-9


def test_solver_memory_released_without_gc():
    """A finished run frees its device buffers (X copy, workspace) as soon as
    the results are dropped -- no reference cycle waiting for the garbage
    collector (a 24 GB workspace per C4 run would otherwise pile up)."""
    import gc
    import torch
    import paper_1003_3272_b200 as M
    rng = np.random.default_rng(0)
    x = rng.random((2048, 1024)).astype(np.float32)
    gc.collect()
    gc.disable()
    try:
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        for _ in range(3):
            st, tr = M.nnmf_run(M.NnmfProblem(x=x, rank=64), M.MmConfig(max_iters=5),
                                M.Backend(dtype="fp32"))
            del st, tr
            torch.cuda.synchronize()
            assert torch.cuda.memory_allocated() == base
    finally:
        gc.enable()
