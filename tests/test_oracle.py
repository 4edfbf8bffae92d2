"""The CPU oracle is pinned to the reference: bitwise against golden vectors
the reference produced (tests/golden/make_golden.py), and -- when the
reference is mounted, i.e. in the build container -- against the live
reference on fresh random inputs."""

import numpy as np
import pytest

import golden_io as G
import refload
from oracle import oracle as O


def test_nnmf_small_run_bitwise():
    g = G.load("nnmf_small")
    x = g["x"]
    rng = np.random.default_rng(5)          # nnmf_run's init, nnmf.py:162-167
    v0, w0 = rng.random((12, 3)), rng.random((3, 9))
    (v, w), trace, _ = O.nnmf_run(x, v0, w0, 25, threads=3, epsilon=1e-9)
    assert np.array_equal(trace, g["trace"])
    assert np.array_equal(v, g["v"]) and np.array_equal(w, g["w"])


def test_nnmf_c1_prefix_bitwise():
    g = G.load("nnmf_c1")
    x, v0, w0 = G.c1_inputs()
    assert G.digest(x) == str(g["x_digest"])
    _, trace, _ = O.nnmf_run(x, v0, w0, 2, threads=8)
    assert np.array_equal(trace, g["trace"][:3])


def test_poisson_small_run_bitwise():
    g = G.load("poisson_small")
    x = g["x"]
    rng = np.random.default_rng(4)          # nnmf_poisson_run's init, nnmf.py:262-265
    v0, w0 = rng.random((12, 3)), rng.random((3, 9))
    (v, w), trace, _ = O.nnmf_poisson_run(x, v0, w0, 40, threads=3, epsilon=1e-9)
    assert np.array_equal(trace, g["trace"])
    assert np.array_equal(v, g["v"]) and np.array_equal(w, g["w"])


def test_poisson_c1_prefix_bitwise():
    g = G.load("poisson_c1")
    x, v0, w0 = G.poisson_c1_inputs()
    assert G.digest(x) == str(g["x_digest"]) and G.digest(v0) == str(g["v0_digest"])
    _, trace, _ = O.nnmf_poisson_run(x, v0, w0, 2, threads=8)
    assert np.array_equal(trace, g["trace"][:3])


def test_poisson_kats():
    """test_nnmf.py:146-158: X = VW is a fixed point; 1x1 square-root update."""
    rng = np.random.default_rng(8)
    v = rng.random((5, 2)) + 0.1
    w = rng.random((2, 6)) + 0.1
    x = O.matmul(v, w)
    v2, w2 = O.nnmf_poisson_update(x, v, w)
    assert np.array_equal(v2, v) and np.array_equal(w2, w)
    v2, _ = O.nnmf_poisson_update(np.array([[4.0]]), np.array([[1.0]]), np.array([[1.0]]))
    assert v2[0, 0] == 2.0


@pytest.mark.parametrize("mu", [0.0, 1e-7, 1e-6, 1e-5])
def test_pet_small_run_bitwise(mu):
    g = G.load("pet_small")
    from paper_1003_3272_b200 import datasets as D
    pd = O.PetData(g["e"], g["y"], mu, D.build_neighborhoods(5))
    lam, trace, _ = O.pet_run(pd, 150, threads=2, epsilon=1e-9)
    assert np.array_equal(trace, g[f"trace_{mu:g}"])
    assert np.array_equal(lam, g[f"lam_{mu:g}"])


def test_pet_c2_prefix_bitwise():
    g = G.load("pet_c2")
    e, y, nbrs = G.c2_inputs()
    assert G.digest(e) == str(g["e_digest"])
    assert np.array_equal(y, g["y"])
    for mu in (0.0, 1e-5):
        pd = O.PetData(e, y, mu, nbrs)
        _, trace, _ = O.pet_run(pd, 3, threads=8)
        assert np.array_equal(trace, g[f"trace_{mu:g}"][:4])


def test_mds_small_run_bitwise():
    g = G.load("mds_small")
    y = g["y"]
    md = O.MdsData(np.ones((9, 9)) - np.eye(9), y, 3)
    theta0 = np.random.default_rng(2).uniform(-1.0, 1.0, size=(3, 9))
    theta, trace, _ = O.mds_run(md, theta0, 40, epsilon=1e-9)
    assert np.array_equal(trace, g["trace"])
    assert np.array_equal(theta, g["theta"])


@pytest.mark.parametrize("dim", [2, 3, 10])
def test_mds_c3_prefix_bitwise(dim):
    g = G.load("mds_c3")
    diss, theta0 = G.c3_inputs(dim)
    assert G.digest(diss) == str(g["diss_digest"])
    md = O.MdsData(1.0 - np.eye(401), diss, dim)
    _, trace, _ = O.mds_run(md, theta0, 3, threads=8)
    assert np.array_equal(trace, g[f"trace_{dim}"][:4])


def test_kernels_hand_values():
    # kernels.py association KATs (test_kernels.py:87-97 style)
    assert O.tree_sum(np.array([1e16, 1.0, -1e16, 1.0])) == ((1e16 + 1.0) + (-1e16 + 1.0))
    assert O.tree_sum(np.array([1.0, 2.0, 3.0])) == (1.0 + 2.0) + 3.0
    assert O.tree_sum(np.zeros(0)) == 0.0
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert np.array_equal(O.matmul(a, a), a @ a)


@pytest.mark.skipif(not refload.available(), reason="reference not mounted")
def test_oracle_matches_live_reference_random():
    R = refload.load()
    rng = np.random.default_rng(123)
    for _ in range(10):
        p, q, r = (int(v) for v in rng.integers(1, 9, size=3))
        x = rng.random((p, q)) * 2.0
        v = rng.random((p, r)) + 0.05
        w = rng.random((r, q)) + 0.05
        assert np.array_equal(O.nnmf_update_v(x, v, w, 3), R.nnmf_update_v(x, v, w))
        assert np.array_equal(O.nnmf_update_w(x, v, w, 2), R.nnmf_update_w(x, v, w))
        assert O.nnmf_objective(x, v, w) == R.nnmf_objective(x, v, w)
        xc = np.floor(x * 3.0)
        v2o, w2o = O.nnmf_poisson_update(xc, v, w, 2)
        v2r, w2r = R.nnmf_poisson_update(xc, v, w)
        assert np.array_equal(v2o, v2r) and np.array_equal(w2o, w2r)
        assert O.nnmf_poisson_objective(xc, v, w) == R.nnmf_poisson_objective(xc, v, w)
        y = rng.random((q + 2, q + 2))
        y = (y + y.T) / 2.0
        np.fill_diagonal(y, 0.0)
        n = q + 2
        theta = rng.uniform(-1, 1, size=(r, n))
        md = O.MdsData(1.0 - np.eye(n), y, r)
        prob = R.MdsProblem(weights=1.0 - np.eye(n), dissimilarities=y, p=r)
        assert np.array_equal(O.mds_update(theta, md), R.mds_update(theta, prob))
        assert O.mds_stress(theta, md) == R.stress(theta, prob)


def test_gradients_bitwise():
    """The oracle's gradient restatements equal the reference's analytic
    gradients (nnmf.py:113-119, pet.py:349-360, mds.py:147-167) bitwise at the
    config starts and the 1000-iteration goldens."""
    g = G.load("gradients")
    x, v0, w0 = G.c1_inputs()
    c1 = G.load("nnmf_c1")
    for tag, (v, w) in (("start", (v0, w0)), ("it1000", (c1["v"], c1["w"]))):
        gv, gw = O.nnmf_gradient(x, v, w, threads=8)
        assert np.array_equal(gv, g[f"nnmf_gv_{tag}"]) and np.array_equal(gw, g[f"nnmf_gw_{tag}"])
    e, y, nbrs = G.c2_inputs()
    c2 = G.load("pet_c2")
    for mu in (0.0, 1e-5):
        pd = O.PetData(e, y, mu, nbrs)
        for tag, lam in (("start", np.ones(4096)), ("it1000", c2[f"lam_{mu:g}"])):
            assert np.array_equal(O.pet_gradient(lam, pd, threads=8), g[f"pet_g_{mu:g}_{tag}"])
    diss, theta0 = G.c3_inputs(3)
    md = O.MdsData(1.0 - np.eye(401), diss, 3)
    c3 = G.load("mds_c3")
    for tag, th in (("start", theta0), ("it1000", c3["theta_3"])):
        assert np.array_equal(O.mds_stress_gradient(th, md, threads=8), g[f"mds_g_{tag}"])
