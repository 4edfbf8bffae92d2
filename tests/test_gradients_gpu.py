"""Analytic gradients on the device: nnmf_gradient,
pet_penalized_gradient, stress_gradient against the reference's values
(tests/golden/gradients.npz, which also pin the oracle bitwise), and the
reference's own gradient KATs (stationarity at convergence, central
differences, the coincidence error)."""

import numpy as np
import pytest

import golden_io as G
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import Backend, MmConfig

pytestmark = pytest.mark.gpu


def fro_err(got, want, scale=None):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    return np.linalg.norm(got - want) / (scale if scale is not None else np.linalg.norm(want))


# The gradient is a difference of two products (2 (V G_W - X W^T), b - colsum,
# theta_i row_i - sum_j coef_ij theta_j): near a stationary point it is small
# next to them, so the error bound is relative to the product magnitude
# (fp64: 1e-12 of it; fp32: 1e-5), and relative to the gradient itself
# (1e-9 / 1e-4, the north-star tolerances) away from stationarity.
@pytest.mark.parametrize("dtype,tol,ptol", [("fp64", 1e-9, 1e-12), ("fp32", 1e-4, 1e-5)])
def test_nnmf_gradient_goldens(dtype, tol, ptol):
    g = G.load("gradients")
    x, v0, w0 = G.c1_inputs()
    c1 = G.load("nnmf_c1")
    for tag, (v, w) in (("start", (v0, w0)), ("it1000", (c1["v"], c1["w"]))):
        gv, gw = M.nnmf_gradient(x, v, w, backend=Backend(dtype=dtype))
        pv = 2.0 * np.linalg.norm(x @ w.T)
        pw = 2.0 * np.linalg.norm(v.T @ x)
        for got, want, prod in ((gv, g[f"nnmf_gv_{tag}"], pv), (gw, g[f"nnmf_gw_{tag}"], pw)):
            assert fro_err(got, want) <= tol or fro_err(got, want, prod) <= ptol, tag


@pytest.mark.parametrize("dtype,tol,ptol", [("fp64", 1e-9, 1e-12), ("fp32", 1e-4, 1e-5)])
@pytest.mark.parametrize("mu", [0.0, 1e-5])
def test_pet_gradient_goldens(dtype, tol, ptol, mu):
    g = G.load("gradients")
    e, y, nbrs = G.c2_inputs()
    c2 = G.load("pet_c2")
    for kernel in ("dense", "sparse"):
        be = Backend(dtype=dtype, pet_kernel=kernel)
        prob = M.PetProblem(e=e, y=y, mu=mu, neighborhoods=nbrs)
        for tag, lam in (("start", np.ones(4096)), ("it1000", c2[f"lam_{mu:g}"])):
            got = M.pet_penalized_gradient(lam, prob, backend=be)
            want = g[f"pet_g_{mu:g}_{tag}"]
            prod = np.linalg.norm(prob.col_sums)
            assert fro_err(got, want) <= tol or fro_err(got, want, prod) <= ptol, (kernel, tag)


def test_pet_gradient_device_built_matrix():
    g = G.load("gradients")
    _, y, nbrs = G.c2_inputs()
    sa = M.system_matrix_device(M.PetGeometry(64, 64))
    prob = M.SparsePetProblem(sa, y, 1e-5, nbrs)
    got = M.pet_penalized_gradient(G.load("pet_c2")["lam_1e-05"], prob, backend=Backend())
    want = g["pet_g_1e-05_it1000"]
    assert fro_err(got, want) <= 1e-9 or fro_err(got, want, np.sqrt(4096.0)) <= 1e-12


@pytest.mark.parametrize("dtype,tol,ptol", [("fp64", 1e-9, 1e-12), ("fp32", 1e-4, 1e-5)])
def test_stress_gradient_goldens(dtype, tol, ptol):
    g = G.load("gradients")
    diss, theta0 = G.c3_inputs(3)
    prob = M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=3)
    c3 = G.load("mds_c3")
    for tag, th in (("start", theta0), ("it1000", c3["theta_3"])):
        got = M.stress_gradient(th, prob, backend=Backend(dtype=dtype))
        want = g[f"mds_g_{tag}"]
        prod = 2.0 * 400 * np.linalg.norm(th)
        assert fro_err(got, want) <= tol or fro_err(got, want, prod) <= ptol, tag


def test_nnmf_interior_stationarity_at_convergence():
    """test_nnmf.py:121-132 on the device."""
    rng = np.random.default_rng(7)
    v_true = rng.random((6, 2)) + 0.5
    w_true = rng.random((2, 5)) + 0.5
    problem = M.NnmfProblem(x=v_true @ w_true, rank=2)
    state, trace = M.nnmf_run(problem, MmConfig(epsilon=1e-15, max_iters=50_000, seed=3),
                              Backend())
    assert np.min(state.v) > 1e-8 and np.min(state.w) > 1e-8
    scale = 1.0 + abs(trace.objective_values[-1])
    gv, gw = M.nnmf_gradient(problem.x, state.v, state.w)
    assert np.max(np.abs(gv)) <= 1e-4 * scale
    assert np.max(np.abs(gw)) <= 1e-4 * scale


def test_pet_stationarity_at_convergence():
    """test_pet.py:294-311 on the device."""
    rng = np.random.default_rng(15)
    p = 4
    e = np.vstack([np.eye(p) * 3.0 + rng.random((p, p)) * 0.3, rng.random((6, p)) + 0.1])
    e /= e.sum(axis=0)
    lam_true = rng.random(p) * 3.0 + 1.0
    y = np.round((e @ lam_true) * 40.0)
    nbrs = [[j for j in (i - 1, i + 1) if 0 <= j < p] for i in range(p)]
    problem = M.PetProblem(e=e, y=y, mu=1e-3, neighborhoods=nbrs)
    lam, trace = M.pet_run(problem, MmConfig(epsilon=1e-14, max_iters=60_000))
    assert trace.converged and np.min(lam) > 1e-8
    grad = M.pet_penalized_gradient(lam, problem)
    f = trace.objective_values[-1]
    assert np.max(np.abs(grad)) <= 1e-4 * (1.0 + abs(f) / problem.n_pixels)


def _random_mds(rng, q, p):
    w = rng.random((q, q)) + 0.1
    w = (w + w.T) / 2.0
    np.fill_diagonal(w, 0.0)
    y = rng.random((q, q)) * 2.0
    y = (y + y.T) / 2.0
    np.fill_diagonal(y, 0.0)
    return M.MdsProblem(weights=w, dissimilarities=y, p=p)


def test_stress_gradient_central_differences():
    """test_mds.py:156-172 on the device (random weights)."""
    rng = np.random.default_rng(5)
    step = 1e-5
    for _ in range(20):
        problem = _random_mds(rng, 5, 2)
        theta = rng.uniform(-1.0, 1.0, size=(2, 5))
        grad = M.stress_gradient(theta, problem)
        fd = np.empty_like(theta)
        for k in range(2):
            for i in range(5):
                hi, lo = theta.copy(), theta.copy()
                hi[k, i] += step
                lo[k, i] -= step
                fd[k, i] = (M.stress(hi, problem) - M.stress(lo, problem)) / (2 * step)
        assert np.linalg.norm(grad - fd) <= 1e-5 * np.linalg.norm(fd)


def test_stress_gradient_coincidence_error():
    """stress_gradient needs d > 0 wherever w > 0, even where y = 0 (unlike
    mds_update, which allows uncoupled coincidence)."""
    y = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0], [1.0, 1.0, 0.0]])
    problem = M.MdsProblem(weights=1.0 - np.eye(3), dissimilarities=y, p=2)
    theta = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0]])
    M.mds_update(theta, problem)        # allowed: objects 0 and 1 are not coupled
    with pytest.raises(M.NumericsError) as e:
        M.stress_gradient(theta, problem)
    assert str(e.value).startswith("objects 0 and 1 coincide")
