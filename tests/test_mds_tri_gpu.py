"""Packed-triangle MDS kernel (csrc/mds_tri.cu, BASELINE config 5 path)
against the CPU oracle (oracle/, pinned bitwise to the reference), the
reference's MDS known-answer tests, the full-row kernel, and size-independent
properties at the full n = 65536 shape.

Tolerance: fp32 mode, 1e-4 relative (BASELINE.json north star) on the
objective trace and the configuration (relative Frobenius)."""

import numpy as np
import pytest

import golden_io as G
import paper_1003_3272_b200 as M
from oracle import oracle as O
from paper_1003_3272_b200 import Backend, MmConfig
from paper_1003_3272_b200 import _lib
from paper_1003_3272_b200.mds import PackedMdsProblem, tile_count
from paper_1003_3272_b200.parallel import tile_range

pytestmark = pytest.mark.gpu

TRI = Backend(dtype="fp32", mds_kernel="tri")
ROWS = Backend(dtype="fp32", mds_kernel="rows")
TOL = 1e-4


def sym_diss(n, seed, dim=3):
    """Noisy Euclidean dissimilarities of a latent configuration, rounded to
    fp32 (so the fp64 oracle and the fp32 kernel see identical values)."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((n, dim + 2))
    sq = (z * z).sum(1)
    d = np.sqrt(np.maximum(sq[:, None] + sq[None, :] - 2.0 * (z @ z.T), 0.0))
    e = rng.uniform(-1.0, 1.0, size=(n, n))
    y = d * (1.0 + 0.05 * (e + e.T) / 2.0)
    np.fill_diagonal(y, 0.0)
    return G.f32(y)


def trace_err(got, want):
    return float(np.max(np.abs(np.asarray(got) - want) / np.abs(want)))


@pytest.mark.parametrize("n,dim", [(300, 2), (517, 3), (1024, 3), (1000, 2)])
def test_tri_matches_oracle(n, dim):
    y = sym_diss(n, n + dim, dim)
    theta0 = G.f32(np.random.default_rng(7).uniform(-1, 1, size=(dim, n)))
    iters = 60
    prob = M.MdsProblem(weights=1.0 - np.eye(n), dissimilarities=y, p=dim)
    cfg = MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6)
    th, tr = M.mds_run(prob, cfg, TRI, theta0=theta0)
    oth, otr, _ = O.mds_run(O.MdsData(1.0 - np.eye(n), y, dim), theta0, iters,
                            threads=O.default_threads())
    assert tr.iters == iters
    assert trace_err(tr.objective_values, otr) <= TOL
    assert G.rel(th, oth) <= TOL


@pytest.mark.parametrize("n,dim", [(300, 1), (517, 2), (777, 3)])
def test_tri_single_step_matches_oracle(n, dim):
    """One update + stress from several states of a run.  (1-D stress
    majorization is chaotic over long runs -- fp32 kernels that agree to
    1e-6 per step drift apart by 1e-3 after 60 steps -- so dim 1 is pinned
    per step.)"""
    y = sym_diss(n, n + dim, dim)
    md = O.MdsData(1.0 - np.eye(n), y, dim)
    prob = M.MdsProblem(weights=1.0 - np.eye(n), dissimilarities=y, p=dim)
    th = G.f32(np.random.default_rng(7).uniform(-1, 1, size=(dim, n)))
    for _ in range(3):
        want = O.mds_update(th, md, threads=O.default_threads())
        got = M.mds_update(th, prob, TRI)
        assert G.rel(got, want) <= 2e-5
        fs = O.mds_stress(th, md, threads=O.default_threads())
        assert abs(M.stress(th, prob, TRI) - fs) / fs <= 1e-5
        th = G.f32(want)


@pytest.mark.parametrize("dim", [2, 3])
def test_tri_c3_golden(dim):
    """BASELINE config 3 (n = 401, roll-call shape) through the packed kernel
    against the reference's own 1000-iteration golden trace."""
    g = G.load("mds_c3")
    diss, theta0 = G.c3_inputs(dim)
    prob = M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=dim)
    cfg = MmConfig(max_iters=1000, epsilon=1e-300, monotone_tol=1e-6)
    theta, tr = M.mds_run(prob, cfg, TRI, theta0=theta0)
    assert trace_err(tr.objective_values, g[f"trace_{dim}"]) <= TOL
    assert G.rel(theta, g[f"theta_{dim}"]) <= TOL


def test_tri_kats():
    """mds.py known answers (test_mds.py:49-80, 119-136) on the packed path."""
    two = M.MdsProblem(weights=np.array([[0.0, 1.0], [1.0, 0.0]]),
                       dissimilarities=np.array([[0.0, 2.0], [2.0, 0.0]]), p=1)
    assert abs(M.stress(np.array([[0.0, 1.0]]), two, TRI) - 1.0) <= 1e-6
    new = M.mds_update(np.array([[0.0, 1.0]]), two, TRI)
    np.testing.assert_allclose(new, [[-0.5, 1.5]], atol=1e-6)
    coupled = M.MdsProblem(weights=np.array([[0.0, 1.0], [1.0, 0.0]]),
                           dissimilarities=np.array([[0.0, 2.0], [2.0, 0.0]]), p=2)
    with pytest.raises(M.NumericsError, match="objects 0 and 1"):
        M.mds_update(np.array([[0.3, 0.3], [-0.2, -0.2]]), coupled, TRI)
    y = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0], [1.0, 1.0, 0.0]])
    free = M.MdsProblem(weights=np.ones((3, 3)) - np.eye(3), dissimilarities=y, p=1)
    got = M.mds_update(np.array([[0.5, 0.5, -0.5]]), free, TRI)
    want = O.mds_update(np.array([[0.5, 0.5, -0.5]]), O.MdsData(np.ones((3, 3)) - np.eye(3), y, 1))
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-7)


def test_tri_coincidence_far_from_origin_tile():
    """A coupled coincident pair deep inside an off-diagonal tile (points 130
    and 600) is reported with the reference's message and indices."""
    n = 700
    y = sym_diss(n, 3)
    theta = G.f32(np.random.default_rng(4).uniform(-1, 1, size=(3, n)))
    theta[:, 600] = theta[:, 130]
    prob = M.MdsProblem(weights=1.0 - np.eye(n), dissimilarities=y, p=3)
    with pytest.raises(M.NumericsError, match="objects 130 and 600"):
        M.mds_update(theta, prob, TRI)
    y0 = y.copy()
    y0[130, 600] = y0[600, 130] = 0.0        # uncoupled: allowed, finite
    prob0 = M.MdsProblem(weights=1.0 - np.eye(n), dissimilarities=y0, p=3)
    got = M.mds_update(theta, prob0, TRI)
    want = O.mds_update(theta, O.MdsData(1.0 - np.eye(n), y0, 3), threads=O.default_threads())
    assert G.rel(got, want) <= 1e-5


def test_tri_from_dense_validates_on_device():
    y = sym_diss(260, 1)
    ok = PackedMdsProblem.from_dense(y, 2, TRI)
    assert ok.t1 - ok.t0 == tile_count(260) == 6
    bad = y.copy()
    bad[3, 200] += 0.5
    with pytest.raises(M.DomainError, match="symmetric"):
        PackedMdsProblem.from_dense(bad, 2, TRI)
    bad = y.copy()
    bad[129, 129] = 1.0
    with pytest.raises(M.DomainError, match="diagonal"):
        PackedMdsProblem.from_dense(bad, 2, TRI)
    bad = y.copy()
    bad[5, 7] = bad[7, 5] = -1.0
    with pytest.raises(M.DomainError, match="nonnegative"):
        PackedMdsProblem.from_dense(bad, 2, TRI)


def test_tri_agrees_with_rows_kernel_and_is_deterministic():
    n, dim = 5000, 3
    y = sym_diss(n, 11)
    theta0 = G.f32(np.random.default_rng(2).uniform(-1, 1, size=(dim, n)))
    prob = M.MdsProblem(weights=1.0 - np.eye(n), dissimilarities=y, p=dim)
    cfg = MmConfig(max_iters=20, epsilon=1e-300, monotone_tol=1e-6)
    a, ta = M.mds_run(prob, cfg, TRI, theta0=theta0)
    b, tb = M.mds_run(prob, cfg, TRI, theta0=theta0)
    assert np.array_equal(a, b) and np.array_equal(ta.objective_values, tb.objective_values)
    r, tr = M.mds_run(prob, cfg, ROWS, theta0=theta0)
    assert trace_err(ta.objective_values, tr.objective_values) <= 1e-5
    assert G.rel(a, r) <= 1e-5


def test_tri_sharded_slices_sum_to_the_whole():
    """The multi-GPU decomposition on one device: G tile slices, phase A per
    slice, the all-reduce replaced by a sum, phase B once."""
    import torch
    n, dim = 3000, 3
    y = sym_diss(n, 5)
    theta = torch.tensor(G.f32(np.random.default_rng(3).uniform(-1, 1, size=(dim, n))),
                         dtype=torch.float32, device="cuda")
    whole = PackedMdsProblem.from_dense(y, dim, TRI)
    mm = M.mds._GpuMdsTri(whole, TRI)
    ref_out = torch.empty_like(theta)
    mm._iterate(theta, ref_out, mm.status.f_ptr, mm.status.err_ptr)
    f_ref = mm._check_error()
    total = None
    nt = tile_count(n)
    for rank in range(3):
        part = PackedMdsProblem.from_dense(y, dim, TRI, tiles=tile_range(nt, 3, rank))
        pm = M.mds._GpuMdsTri(part, TRI)
        _lib.call("mmk_mds_tri_iter_a", _lib.ptr(pm.pk), pm.t0, pm.t1, _lib.ptr(theta), dim, n,
                  _lib.ptr(pm.ws), pm.ws.numel(), _lib.ptr(pm.red), pm.status.err_ptr,
                  pm.stream())
        total = pm.red.clone() if total is None else total + pm.red
    out = torch.empty_like(theta)
    f = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("mmk_mds_tri_iter_b", _lib.ptr(theta), _lib.ptr(out), dim, n, _lib.ptr(total),
              _lib.ptr(f), mm.status.err_ptr, mm.stream())
    torch.cuda.synchronize()
    assert abs(float(f) - f_ref) / f_ref <= 1e-6
    assert float((out - ref_out).norm() / ref_out.norm()) <= 1e-6


def c5_rows(n, seed=0):
    return M.datasets.distance_rows(n, seed)


def test_c5_full_shape_properties():
    """n = 65536, dim 3 (BASELINE config 5): monotone stress over 8 fused
    iterations, bitwise-reproducible, stress of the start equal to an
    independent fp64 evaluation on a sample of tile rows."""
    import torch
    n, dim = 65536, 3
    prob = PackedMdsProblem.from_rows(c5_rows(n), n, dim, TRI)
    theta0 = torch.rand(dim, n, generator=torch.Generator(device="cuda").manual_seed(2),
                        device="cuda") * 2 - 1
    cfg = MmConfig(max_iters=8, epsilon=1e-300, monotone_tol=1e-6)
    th, tr = M.mds_run(prob, cfg, TRI, theta0=theta0)
    th2, tr2 = M.mds_run(prob, cfg, TRI, theta0=theta0)
    v = tr.objective_values
    assert tr.iters == 8 and np.all(np.diff(v) <= 1e-6 * (1 + np.abs(v[:-1])))
    assert np.array_equal(v, tr2.objective_values) and torch.equal(th, th2)
    # independent fp64 stress at theta0 from regenerated rows
    rows = c5_rows(n)
    t64 = theta0.double()
    s = 0.0
    for r0 in range(0, n, 4096):
        yb = rows(r0, r0 + 4096).double()
        d = torch.cdist(t64[:, r0:r0 + 4096].T, t64.T)
        mask = torch.arange(n, device="cuda")[None, :] > torch.arange(r0, r0 + 4096,
                                                                       device="cuda")[:, None]
        s += float((((yb - d) ** 2) * mask).sum())
    assert abs(v[0] - s) / s <= 1e-5


@pytest.mark.parametrize("q,m", [(401, 671), (300, 57), (1000, 130)])
def test_votes_to_packed_tiles_match_reference(q, m):
    """Roll calls -> packed dissimilarity tiles on the tensor cores equal the
    fp32 rounding of the reference's votes_to_dissimilarity bit for bit."""
    votes = M.datasets.synthetic_votes(q, m, q + m)
    want = PackedMdsProblem.from_dense(G.f32(M.votes_to_dissimilarity(votes)), 2, TRI,
                                       validate=False)
    got = PackedMdsProblem.from_votes(votes, 2, TRI)
    import torch
    assert torch.equal(got.packed, want.packed)
    half = PackedMdsProblem.from_votes(votes.astype(np.float32), 2, TRI,
                                       tiles=tile_range(tile_count(q), 2, 1))
    assert torch.equal(half.packed, want.packed[half.t0 * 16384:half.t1 * 16384])


def test_votes_errors():
    v = M.datasets.synthetic_votes(200, 40, 1)
    v[3, 5] = 2.0
    with pytest.raises(M.DomainError, match="votes must be 1"):
        PackedMdsProblem.from_votes(v, 2, TRI)
    v = M.datasets.synthetic_votes(200, 40, 1)
    v[7, :20] = 0.0
    v[150, 20:] = 0.0
    with pytest.raises(M.DomainError, match="voters 7 and 150 share no roll call"):
        PackedMdsProblem.from_votes(v, 2, TRI)
