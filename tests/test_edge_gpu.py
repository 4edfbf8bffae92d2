"""Edge shapes against the oracle: every rank bucket of the NNMF kernels
(r = 1 .. 128, tensor-core eligible and not), degenerate and ragged shapes,
every MDS dimension specialisation (1..10 and the generic kernel above),
tiny and ragged PET problems with explicit weights; 8 MM iterations each
through the public API (fp64 1e-9 / fp32 1e-4, relative Frobenius)."""

import warnings

import numpy as np
import pytest

import golden_io as G
import paper_1003_3272_b200 as M
from oracle import oracle as O
from paper_1003_3272_b200 import Backend, MmConfig

pytestmark = pytest.mark.gpu

ITERS = 8
CFG = MmConfig(max_iters=ITERS, epsilon=1e-300, monotone_tol=1e-6)


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


@pytest.mark.parametrize("m,n,r", [(1, 1, 1), (2, 9, 1), (7, 3, 5), (33, 65, 17), (64, 40, 33),
                                   (130, 257, 64), (256, 264, 64), (50, 20, 100), (41, 19, 128),
                                   (256, 264, 32), (136, 392, 48), (264, 136, 17)])
@pytest.mark.parametrize("dtype,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_nnmf_rank_buckets_and_shapes(m, n, r, dtype, tol):
    rng = np.random.default_rng(m * 1000 + n * 10 + r)
    x = f32(rng.random((m, n)))
    v0, w0 = f32(rng.random((m, r)) + 0.1), f32(rng.random((r, n)) + 0.1)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")       # rank > min(m, n) warns, as the reference
        prob = M.NnmfProblem(x=x, rank=r)
    st, tr = M.nnmf_run(prob, CFG, Backend(dtype=dtype), state0=M.FactorPair(v0, w0))
    (v, w), trace, _ = O.nnmf_run(x, v0, w0, ITERS, threads=4, monotone_tol=1e-6)
    assert G.rel(tr.objective_values, trace) <= tol
    assert G.rel(st.v @ st.w, v @ w) <= tol


@pytest.mark.parametrize("n,dim", [(4, 1), (3, 2), (37, 3), (37, 7), (19, 10), (23, 11),
                                   (17, 16)])
@pytest.mark.parametrize("dtype,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_mds_dims_with_explicit_weights(n, dim, dtype, tol):
    rng = np.random.default_rng(n * 100 + dim)
    w = f32(rng.random((n, n)) + 0.2)
    w = np.triu(w, 1) + np.triu(w, 1).T
    y = f32(rng.random((n, n)) * 2.0)
    y = np.triu(y, 1) + np.triu(y, 1).T
    theta0 = f32(rng.uniform(-1.0, 1.0, size=(dim, n)))
    prob = M.MdsProblem(weights=w, dissimilarities=y, p=dim)
    th, tr = M.mds_run(prob, CFG, Backend(dtype=dtype), theta0=theta0)
    theta, trace, _ = O.mds_run(O.MdsData(w, y, dim), theta0, ITERS, monotone_tol=1e-6)
    assert G.rel(tr.objective_values, trace) <= tol
    if dim > 1:    # 1-D stress majorization is too ill-conditioned for state parity
        assert G.rel(th, theta) <= 10 * tol


@pytest.mark.parametrize("side,det", [(2, 4), (3, 7), (9, 10)])
@pytest.mark.parametrize("mu", [0.0, 1e-3])
@pytest.mark.parametrize("kernel", ["dense", "sparse"])
def test_pet_small_geometries(side, det, mu, kernel):
    geo = M.PetGeometry(side, det)
    e = M.build_system_matrix(geo)
    y = M.simulate_counts(M.default_phantom(side) + 0.5, e, 7)
    nb = M.build_neighborhoods(side)
    prob = M.PetProblem(e=e, y=y, mu=mu, neighborhoods=nb)
    lam, tr = M.pet_run(prob, CFG, Backend(dtype="fp64", pet_kernel=kernel))
    ref, trace, _ = O.pet_run(O.PetData(e, y, mu, nb), ITERS, monotone_tol=1e-6)
    assert G.rel(tr.objective_values, trace) <= 1e-9
    assert G.rel(lam, ref) <= 1e-9
