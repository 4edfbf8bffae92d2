"""The public sharded solvers (parallel.nnmf_run_sharded / mds_run_sharded)
through a real NCCL process group.  The pool gives one GPU, so the group has
one rank: every collective of the multi-GPU path runs (on the compute
stream, NCCL), and the results must equal the unsharded solver bitwise.  The
decomposition itself is checked at world size 2-3 on CPU (gloo,
tests/test_sharding_cpu.py) and on one GPU with virtual shards
(test_nnmf_tc_gpu.py::test_row_shards_sum_to_the_whole,
test_mds_tri_gpu.py::test_tri_sharded_slices_sum_to_the_whole)."""

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_1003_3272_b200 as M
from paper_1003_3272_b200 import Backend, MmConfig
from paper_1003_3272_b200 import parallel as P
from paper_1003_3272_b200.mds import PackedMdsProblem, tile_count

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("poisson", [False, True])
def test_nnmf_sharded_equals_unsharded(group, poisson):
    rng = np.random.default_rng(4)
    x = np.floor(rng.random((1024, 256)) * 5.0) if poisson else rng.random((1024, 256))
    v0, w0 = rng.random((1024, 64)), rng.random((64, 256))
    be = Backend(dtype="fp32", fused=False)
    cfg = MmConfig(max_iters=15, epsilon=1e-300, monotone_tol=1e-6)
    xd = torch.tensor(x, dtype=torch.float32, device="cuda")
    st, tr = P.nnmf_run_sharded(xd, 64, cfg, be, group=group, state0=(v0, w0), poisson=poisson)
    run = M.nnmf_poisson_run if poisson else M.nnmf_run
    ref, rtr = run(M.NnmfProblem(x=xd, rank=64), cfg, be, state0=M.FactorPair(v0, w0))
    assert np.array_equal(tr.objective_values, rtr.objective_values)
    assert torch.equal(st.v, ref.v) and torch.equal(st.w, ref.w)


def test_mds_sharded_equals_unsharded(group):
    n = 1500
    rows = M.datasets.distance_rows(n, seed=3)
    be = Backend(dtype="fp32", mds_kernel="tri", fused=False)
    prob = PackedMdsProblem.from_rows(rows, n, 3, be, tiles=P.tile_range(tile_count(n), 1, 0))
    th0 = np.random.default_rng(5).uniform(-1, 1, size=(3, n))
    cfg = MmConfig(max_iters=10, epsilon=1e-300, monotone_tol=1e-6)
    th, tr = P.mds_run_sharded(prob, cfg, be, group=group, theta0=th0)
    ref, rtr = M.mds_run(prob, cfg, be, theta0=th0)
    assert np.array_equal(tr.objective_values, rtr.objective_values)
    assert np.array_equal(np.asarray(th.cpu() if hasattr(th, "cpu") else th), ref)


def test_in_graph_nccl_engine(group, monkeypatch):
    """The fused device engine with the all-reduce captured inside its CUDA
    graph (ncclAllReduce of torch's communicator, resolved with dlsym):
    equal to the graph engine without the collective (the persistent
    small-problem engine, which a single-GPU run of this size would pick,
    is switched off for the reference run)."""
    from paper_1003_3272_b200 import _lib
    monkeypatch.setenv("MMK_SMALL_ENGINE", "0")
    comm = P.nccl_comm_ptr()
    assert comm, "no NCCL communicator pointer"
    assert _lib.load().mmk_nccl_available() == 1
    rng = np.random.default_rng(6)
    x = rng.random((512, 192))
    v0, w0 = rng.random((512, 8)), rng.random((8, 192))
    be = Backend(dtype="fp64")
    cfg = MmConfig(max_iters=12, epsilon=1e-300)
    prob = M.NnmfProblem(x=x, rank=8)
    mm = M.nnmf._GpuNnmf(prob, be)
    mm.comm = comm
    st, tr = M.run_mm(mm, mm.device_state(M.FactorPair(v0, w0)), cfg)
    ref, rtr = M.nnmf_run(prob, cfg, be, state0=M.FactorPair(v0, w0))
    assert np.array_equal(tr.objective_values, rtr.objective_values)
    assert np.array_equal(st.v.cpu().numpy(), ref.v)
