"""The sharded solvers with TWO ranks: two processes share the one GPU of the
pool and exchange the phase-A reduction buffer through a real
torch.distributed group (gloo, which all-reduces CUDA tensors through host
staging; NCCL refuses two ranks on one device).  Rank r holds rows
shard_rows(m, 2, r) of X (NNMF) or tiles tile_range(T, 2, r) of the packed
triangle (MDS); both ranks must return the same trace, equal to the unsharded
solver up to the order of the cross-rank sum."""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _nnmf_worker(rank, world, port, poisson, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import parallel as P
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        x, v0, w0 = _nnmf_inputs(poisson)
        lo, hi = P.shard_rows(x.shape[0], world, rank)
        xd = torch.tensor(x[lo:hi], dtype=torch.float32, device="cuda")
        cfg = M.MmConfig(max_iters=12, epsilon=1e-300, monotone_tol=1e-6)
        st, tr = P.nnmf_run_sharded(xd, 64, cfg, M.Backend(dtype="fp32", fused=False),
                                    state0=(v0[lo:hi], w0), poisson=poisson)
        q.put((rank, tr.objective_values, st.v.cpu().numpy(), st.w.cpu().numpy()))
        dist.destroy_process_group()
    except Exception as e:   # surface the failure in the parent
        q.put((rank, repr(e), None, None))


def _nnmf_inputs(poisson):
    rng = np.random.default_rng(8)
    x = np.floor(rng.random((1024, 256)) * 5.0) if poisson else rng.random((1024, 256))
    return x, rng.random((1024, 64)), rng.random((64, 256))


def _run_ranks(target, *args, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    for rank, res, *_ in out:
        assert not isinstance(res, str), f"rank {rank} failed: {res}"
    return out


@pytest.mark.parametrize("poisson", [False, True])
def test_nnmf_two_ranks(poisson):
    import torch
    import paper_1003_3272_b200 as M
    out = _run_ranks(_nnmf_worker, poisson)
    (_, t0, v0s, w0s), (_, t1, v1s, w1s) = out
    assert np.array_equal(t0, t1) and np.array_equal(w0s, w1s)
    x, v0, w0 = _nnmf_inputs(poisson)
    run = M.nnmf_poisson_run if poisson else M.nnmf_run
    xd = torch.tensor(x, dtype=torch.float32, device="cuda")
    ref, rtr = run(M.NnmfProblem(x=xd, rank=64), M.MmConfig(max_iters=12, epsilon=1e-300,
                                                            monotone_tol=1e-6),
                   M.Backend(dtype="fp32"), state0=M.FactorPair(v0, w0))
    assert G.rel(t0, rtr.objective_values) <= 1e-6
    v = np.concatenate([v0s, v1s])
    assert G.rel(v @ w0s, (ref.v @ ref.w).cpu().numpy()) <= 1e-5


def _mds_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import datasets as D
    from paper_1003_3272_b200 import parallel as P
    from paper_1003_3272_b200.mds import PackedMdsProblem, tile_count
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n = 1500
        be = M.Backend(dtype="fp32", mds_kernel="tri", fused=False)
        prob = PackedMdsProblem.from_rows(D.distance_rows(n, seed=3), n, 3, be,
                                          tiles=P.tile_range(tile_count(n), world, rank))
        th0 = np.random.default_rng(5).uniform(-1, 1, size=(3, n))
        cfg = M.MmConfig(max_iters=10, epsilon=1e-300, monotone_tol=1e-6)
        th, tr = P.mds_run_sharded(prob, cfg, be, theta0=th0)
        th = th.cpu().numpy() if hasattr(th, "cpu") else np.asarray(th)
        q.put((rank, tr.objective_values, th, None))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e), None, None))


def test_mds_tri_two_ranks():
    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import datasets as D
    from paper_1003_3272_b200.mds import PackedMdsProblem
    out = _run_ranks(_mds_worker)
    (_, t0, th0s, _), (_, t1, th1s, _) = out
    assert np.array_equal(t0, t1), (t0 - t1, len(t0), len(t1))
    assert np.array_equal(th0s, th1s)
    n = 1500
    be = M.Backend(dtype="fp32", mds_kernel="tri", fused=False)
    prob = PackedMdsProblem.from_rows(D.distance_rows(n, seed=3), n, 3, be)
    th0 = np.random.default_rng(5).uniform(-1, 1, size=(3, n))
    ref, rtr = M.mds_run(prob, M.MmConfig(max_iters=10, epsilon=1e-300, monotone_tol=1e-6), be,
                         theta0=th0)
    assert G.rel(t0, rtr.objective_values) <= 1e-6
    assert G.rel(th0s, np.asarray(ref)) <= 1e-5


def _pet_worker(rank, world, port, kernel, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import parallel as P
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        e, y, nbrs = G.c2_inputs()
        prob = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=nbrs)
        lam, tr = P.pet_run_sharded(prob, M.MmConfig(max_iters=50, epsilon=1e-300),
                                    M.Backend(dtype="fp64", pet_kernel=kernel))
        q.put((rank, tr.objective_values, np.asarray(lam), None))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e), None, None))


@pytest.mark.parametrize("kernel", ["dense", "sparse"])
def test_pet_two_ranks(kernel):
    """Ray shards (1008 rays each at C2) with the all-reduce of [b | loglik]."""
    import paper_1003_3272_b200 as M
    out = _run_ranks(_pet_worker, kernel)
    (_, t0, l0, _), (_, t1, l1, _) = out
    assert np.array_equal(t0, t1) and np.array_equal(l0, l1)
    e, y, nbrs = G.c2_inputs()
    prob = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=nbrs)
    ref, rtr = M.pet_run(prob, M.MmConfig(max_iters=50, epsilon=1e-300),
                         M.Backend(dtype="fp64", pet_kernel=kernel))
    assert G.rel(t0, rtr.objective_values) <= 1e-12
    assert G.rel(l0, ref) <= 1e-11


def _mds_rows_worker(rank, world, port, weighted, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import parallel as P
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        prob, th0 = _mds_rows_problem(weighted)
        th, tr = P.mds_run_sharded(prob, M.MmConfig(max_iters=40, epsilon=1e-300),
                                   M.Backend(dtype="fp64"), theta0=th0)
        th = th.cpu().numpy() if hasattr(th, "cpu") else np.asarray(th)
        q.put((rank, tr.objective_values, th, None))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e), None, None))


def _mds_rows_problem(weighted):
    import paper_1003_3272_b200 as M
    diss, th0 = G.c3_inputs(3)
    w = 1.0 - np.eye(401)
    if weighted:
        rng = np.random.default_rng(9)
        w = rng.random((401, 401)) + 0.5
        w = np.triu(w, 1) + np.triu(w, 1).T
    return M.MdsProblem(weights=w, dissimilarities=diss, p=3), th0


@pytest.mark.parametrize("weighted", [False, True])
def test_mds_rows_two_ranks(weighted):
    """Dense MDS, points split over the ranks: each rank updates its points from
    its rows of Y (and W), then all-gather of theta' and all-reduce of the
    stress partial."""
    import paper_1003_3272_b200 as M
    out = _run_ranks(_mds_rows_worker, weighted)
    (_, t0, th0s, _), (_, t1, th1s, _) = out
    assert np.array_equal(t0, t1) and np.array_equal(th0s, th1s)
    prob, th0 = _mds_rows_problem(weighted)
    ref, rtr = M.mds_run(prob, M.MmConfig(max_iters=40, epsilon=1e-300), M.Backend(dtype="fp64"),
                         theta0=th0)
    assert G.rel(t0, rtr.objective_values) <= 1e-12
    assert G.rel(th0s, np.asarray(ref)) <= 1e-10


def _pet_device_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import parallel as P
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        _, y, nbrs = G.c2_inputs()
        prob = M.SparsePetProblem(M.system_matrix_device(M.PetGeometry(64, 64)), y, 1e-5, nbrs)
        lam, tr = P.pet_run_sharded(prob, M.MmConfig(max_iters=50, epsilon=1e-300),
                                    M.Backend(dtype="fp64", fused=False))
        lam = lam.cpu().numpy() if hasattr(lam, "cpu") else np.asarray(lam)
        q.put((rank, tr.objective_values, lam, None))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e), None, None))


def test_pet_device_built_matrix_two_ranks():
    """Ray shards of a DEVICE-BUILT sparse system matrix (SparsePetProblem):
    each rank slices its CSR rows and the CSC restricted to its rays on the
    device (pet._shard_device_sparse); equal to the unsharded run."""
    import paper_1003_3272_b200 as M
    out = _run_ranks(_pet_device_worker)
    (_, t0, l0, _), (_, t1, l1, _) = out
    assert np.array_equal(t0, t1) and np.array_equal(l0, l1)
    _, y, nbrs = G.c2_inputs()
    prob = M.SparsePetProblem(M.system_matrix_device(M.PetGeometry(64, 64)), y, 1e-5, nbrs)
    ref, rtr = M.pet_run(prob, M.MmConfig(max_iters=50, epsilon=1e-300),
                         M.Backend(dtype="fp64", fused=False))
    ref = ref.cpu().numpy() if hasattr(ref, "cpu") else np.asarray(ref)
    assert G.rel(t0, rtr.objective_values) <= 1e-12
    assert G.rel(l0, ref) <= 1e-11
