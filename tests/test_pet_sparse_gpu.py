"""Device-built Siddon system matrix and the sparse PET projector (SURVEY.md
8f row 2) against the reference's dense construction (restated in
paper_1003_3272_b200.datasets, pinned by the config-2 golden traces) and the
golden PET runs."""

import numpy as np
import pytest

import golden_io as G
import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import Backend, MmConfig

pytestmark = pytest.mark.gpu


def dense_of(sa):
    out = np.zeros((sa["n_rays"], sa["n_pixels"]))
    rptr = sa["rptr"].cpu().numpy()
    ridx = sa["ridx"].cpu().numpy()
    rval = sa["rval"].cpu().numpy()
    for i in range(sa["n_rays"]):
        out[i, ridx[rptr[i]:rptr[i + 1]]] += rval[rptr[i]:rptr[i + 1]]
    return out


@pytest.mark.parametrize("side,det", [(8, 12), (16, 24), (64, 64)])
def test_device_siddon_matches_reference_build(side, det):
    geo = M.PetGeometry(side, det)
    want = M.build_system_matrix(geo)
    sa = M.system_matrix_device(geo)
    got = dense_of(sa)
    assert np.max(np.abs(got - want)) <= 1e-14
    assert sa["rval"].numel() == np.count_nonzero(want)
    # CSC holds the same entries by pixel
    cptr, cidx, cval = (sa[k].cpu().numpy() for k in ("cptr", "cidx", "cval"))
    j = side * side // 2 + side // 3
    col = np.zeros(geo.n_rays)
    col[cidx[cptr[j]:cptr[j + 1]]] = cval[cptr[j]:cptr[j + 1]]
    np.testing.assert_array_equal(col, got[:, j])


def test_device_siddon_uncovered_pixel():
    geo = M.PetGeometry(40, 3)
    with pytest.raises(M.DomainError) as ref:
        M.build_system_matrix(geo)
    with pytest.raises(M.DomainError) as dev:
        M.system_matrix_device(geo)
    assert str(dev.value) == str(ref.value)


@pytest.mark.parametrize("mu", [0.0, 1e-5])
def test_c2_on_device_built_matrix(mu):
    g = G.load("pet_c2")
    _, y, nbrs = G.c2_inputs()
    sa = M.system_matrix_device(M.PetGeometry(64, 64))
    prob = M.SparsePetProblem(sa, y, mu, nbrs)
    lam, tr = M.pet_run(prob, MmConfig(max_iters=1000, epsilon=1e-300), Backend(dtype="fp64"))
    err = np.max(np.abs(tr.objective_values - g[f"trace_{mu:g}"]) / np.abs(g[f"trace_{mu:g}"]))
    assert err <= 1e-9
    assert G.rel(lam, g[f"lam_{mu:g}"]) <= 1e-9


def test_large_geometry_runs_monotone():
    """256 x 256 image, 256 detectors (32,640 rays): 17 GB as a dense fp64
    matrix; built on the device, reconstructed from simulated counts."""
    import torch
    geo = M.PetGeometry(256, 256)
    sa = M.system_matrix_device(geo)
    col = torch.zeros(geo.n_pixels, dtype=torch.float64, device="cuda")
    col.index_add_(0, sa["ridx"].long(), sa["rval"])
    assert float((col - 1.0).abs().max()) <= 1e-12
    lam_true = torch.from_numpy(M.default_phantom(256)).cuda()
    means = M.SparsePetProblem(sa, np.zeros(geo.n_rays), 0.0, M.build_neighborhoods(256)).forward(lam_true)
    gen = torch.Generator(device="cuda").manual_seed(5)
    y = torch.poisson(means * 50.0, generator=gen)
    prob = M.SparsePetProblem(sa, y, 1e-6, M.build_neighborhoods(256))
    _, tr = M.pet_run(prob, MmConfig(max_iters=20, epsilon=1e-300, monotone_tol=1e-6),
                      Backend(dtype="fp32"))
    d = np.diff(tr.objective_values)
    assert tr.iters == 20 and np.all(d >= -1e-6 * (1 + np.abs(tr.objective_values[:-1])))


@pytest.mark.parametrize("dtype", ["fp32", "fp64"])
@pytest.mark.parametrize("side,det,mu", [(64, 64, 1e-5), (37, 40, 0.0), (256, 96, 1e-6)])
def test_fused_sparse_iteration_equals_split_phases(dtype, side, det, mu):
    """mmk_pet_sparse_iter (forward projection + fused back-projection/pixel
    kernel) gives bitwise the intensities of the split iter_a (b in memory) /
    iter_b pair that a sharded caller uses, and the same objective up to the
    grouping of the penalty partials; ragged pixel counts exercise a partial
    last CTA."""
    import ctypes
    import torch
    from paper_1003_3272_b200 import _lib
    from paper_1003_3272_b200.pet import _GpuPet
    geo = M.PetGeometry(side, det)
    be = Backend(dtype=dtype)
    sa = M.system_matrix_device(geo, be)
    nb = M.build_neighborhoods(side)
    rng = np.random.default_rng(side)
    lam_true = torch.from_numpy(rng.uniform(0.5, 2.0, geo.n_pixels)).cuda()
    means = M.SparsePetProblem(sa, np.zeros(geo.n_rays), 0.0, nb).forward(lam_true)
    y = torch.floor(means * 20.0).cpu().numpy()
    mm = _GpuPet(M.SparsePetProblem(sa, y, mu, nb), be)
    tdt = torch.float32 if dtype == "fp32" else torch.float64
    lam = torch.from_numpy(rng.uniform(0.2, 3.0, geo.n_pixels)).to("cuda", tdt)
    P = _lib.ptr
    flags = _lib.MMK_PET_UPDATE | _lib.MMK_PET_OBJECTIVE
    outs, fs = [], []
    for fused in (True, False):
        out = torch.empty_like(lam)
        f = torch.zeros(1, dtype=torch.float64, device="cuda")
        mm.ws.zero_()
        if fused:
            mm._iterate(lam, out, P(f), mm.status.err_ptr, flags)
        else:
            s, sd = mm.stream(), mm.sa    # arrays in the backend's dtype
            _lib.call("mmk_pet_sparse_iter_a", mm.code, P(sd["rptr"]), P(sd["ridx"]),
                      P(sd["rval"]), P(sd["cptr"]), P(sd["cidx"]), P(sd["cval"]), P(mm.y),
                      P(lam), mm.d, mm.p, P(mm.ws), mm.ws.numel(), P(mm.red),
                      mm.status.err_ptr, s)
            _lib.call("mmk_pet_iter_b", mm.code, P(lam), P(out), mm.p, P(mm.ptr), P(mm.idx),
                      mm.mu, flags, P(mm.red), P(mm.ws), mm.ws.numel(), P(f),
                      mm.status.err_ptr, s)
        torch.cuda.synchronize()
        mm._check_error()
        outs.append(out)
        fs.append(float(f.item()))
    assert torch.equal(outs[0], outs[1])
    assert abs(fs[0] - fs[1]) <= 1e-13 * abs(fs[1])


def test_device_sparse_ray_shards_sum_to_the_whole():
    """Ray shards of the device-built matrix (pet._shard_device_sparse): the
    phase-A buffers [b | loglik] of three shards sum to the unsharded one,
    and each shard's CSC holds exactly its rays' entries."""
    import torch
    from paper_1003_3272_b200 import _lib, parallel as P
    from paper_1003_3272_b200.pet import _GpuPet
    geo = M.PetGeometry(24, 32)
    sa = M.system_matrix_device(geo)
    y = M.simulate_counts(M.default_phantom(24) + 0.5, M.build_system_matrix(geo), 5)
    prob = M.SparsePetProblem(sa, y, 1e-4, M.build_neighborhoods(24))
    be = Backend(dtype="fp64", fused=False)
    lam = torch.rand(geo.n_pixels, dtype=torch.float64, device="cuda") + 0.5

    def phase_a(mm):
        s = mm.sa
        P_ = _lib.ptr
        _lib.call("mmk_pet_sparse_iter_a", mm.code, P_(s["rptr"]), P_(s["ridx"]), P_(s["rval"]),
                  P_(s["cptr"]), P_(s["cidx"]), P_(s["cval"]), P_(mm.y), P_(lam), mm.d, mm.p,
                  P_(mm.ws), mm.ws.numel(), P_(mm.red), mm.status.err_ptr, mm.stream())
        torch.cuda.synchronize()
        return mm.red.clone()
    whole = phase_a(_GpuPet(prob, be))
    total = torch.zeros_like(whole)
    nnz = 0
    for r in range(3):
        lo, hi = P.shard_rows(geo.n_rays, 3, r)
        mm = _GpuPet(prob, be, rows=(lo, hi))
        nnz += int(mm.sa["cptr"][-1])
        total += phase_a(mm)
    assert nnz == int(sa["cptr"][-1])
    assert float((total - whole).abs().max() / whole.abs().max()) <= 1e-13
