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


@pytest.mark.parametrize("poisson,r", [(False, 64), (True, 64), (False, 128), (True, 100)])
def test_nnmf_sharded_fused_engine_equals_unsharded(group, poisson, r):
    """The public sharded solver on the device-loop engine (Backend(fused=True),
    NCCL group): the all-reduce of the phase-A buffer captured inside the CUDA
    graph, one collective per iteration; bitwise equal to nnmf_run (the graph
    engine there too: a tensor-core-size problem, so no persistent engine).
    r = 128: the rank-128 tensor-core tile; Poisson r = 100: its 128-rank
    CUDA-core tiles."""
    rng = np.random.default_rng(14)
    m, n = 2048, 1024
    x = np.floor(rng.random((m, n)) * 5.0) if poisson else rng.random((m, n))
    v0, w0 = rng.random((m, r)), rng.random((r, n))
    be = Backend(dtype="fp32", fused=True)
    cfg = MmConfig(max_iters=12, epsilon=1e-300, monotone_tol=1e-6)
    xd = torch.tensor(x, dtype=torch.float32, device="cuda")
    st, tr = P.nnmf_run_sharded(xd, r, cfg, be, group=group, state0=(v0, w0), poisson=poisson)
    run = M.nnmf_poisson_run if poisson else M.nnmf_run
    ref, rtr = run(M.NnmfProblem(x=xd, rank=r), cfg, be, state0=M.FactorPair(v0, w0))
    assert tr.iters == 12
    assert np.array_equal(tr.objective_values, rtr.objective_values)
    assert torch.equal(st.v, ref.v) and torch.equal(st.w, ref.w)


def test_mds_sharded_fused_engine_equals_unsharded(group):
    n = 1500
    rows = M.datasets.distance_rows(n, seed=3)
    be = Backend(dtype="fp32", mds_kernel="tri", fused=True)
    prob = PackedMdsProblem.from_rows(rows, n, 3, be, tiles=P.tile_range(tile_count(n), 1, 0))
    th0 = np.random.default_rng(5).uniform(-1, 1, size=(3, n))
    cfg = MmConfig(max_iters=10, epsilon=1e-300, monotone_tol=1e-6)
    th, tr = P.mds_run_sharded(prob, cfg, be, group=group, theta0=th0)
    ref, rtr = M.mds_run(prob, cfg, Backend(dtype="fp32", mds_kernel="tri", fused=False),
                         theta0=th0)
    assert np.allclose(tr.objective_values, rtr.objective_values, rtol=1e-6, atol=0)


def test_bench_self_launches_two_ranks():
    """`python bench.py --gpus 2` (no torchrun environment) re-launches itself
    under torch.distributed.run with two ranks; on a one-GPU box they share
    the device over a gloo group (a functional check of the sharded path):
    rank 0 prints one line with n_gpus 2."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "4",
                          "--warmup", "3", "--workload", "nnmf-mid", "--no-e2e",
                          "--cpu-seconds", "0"], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = lines[0]
    assert line["n_gpus"] == 2 and line["steps"] == 4
    assert line["config"]["parallelism"] == "rows-sharded x2"
    assert line["value"] > 0 and line["roofline"]["kernel"].startswith("nnmf_")
