"""Multi-GPU decomposition logic on CPU (gloo, world_size 2).

The sharded paths split NNMF by rows of X / V with one
all-reduce of the W-step partials, and the packed-triangle MDS by tiles with
one all-reduce of the per-point accumulators.  Here the host fp64 models of
the phase-A / phase-B kernels (paper_1003_3272_b200.parallel) run on two
gloo ranks and must reproduce the unsharded iteration of the CPU oracle
(oracle/, pinned to the reference)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1003_3272_b200 import parallel as P


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_row_partition_covers_and_balances():
    for n in (1, 7, 128, 1001, 131072):
        for world in (1, 2, 3, 8):
            spans = [P.shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_tile_partition_covers_and_balances():
    for n in (2, 300, 65536):
        nt = len(P.tri_tiles(n))
        for world in (1, 2, 4, 8):
            spans = [P.tile_range(nt, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nt
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _nnmf_worker(rank, world, port, x, v, w, out, bad_rank=-1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = P.shard_rows(x.shape[0], world, rank)
    v2, red = P.phase_a_model(x[lo:hi], v[lo:hi], w, error=rank == bad_rank)
    t = torch.from_numpy(red)
    P.allreduce_sum_(t)
    w2, f, err = P.phase_b_model(w, t.numpy(), x.shape[1], v.shape[1])
    out[rank] = (lo, hi, v2, w2, f, err)
    dist.destroy_process_group()


def test_nnmf_row_sharding_gloo():
    rng = np.random.default_rng(0)
    x, v, w = rng.random((37, 23)), rng.random((37, 4)), rng.random((4, 23))
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_nnmf_worker, args=(2, _free_port(), x, v, w, out), nprocs=2, join=True)
        res = dict(out)
    f_ref = O.nnmf_objective(x, v, w)
    v_ref, w_ref = O.nnmf_step(x, v, w)
    v_sh = np.concatenate([res[r][2] for r in range(2)])
    for r in range(2):
        assert abs(res[r][4] - f_ref) <= 1e-12 * f_ref
        np.testing.assert_allclose(res[r][3], w_ref, rtol=1e-12)
    np.testing.assert_allclose(v_sh, v_ref, rtol=1e-12)
    np.testing.assert_array_equal(res[0][3], res[1][3])   # W' replicated bitwise
    assert not res[0][5] and not res[1][5]


def test_device_error_flag_reaches_every_rank_gloo():
    """The device-error flag rides in the one all-reduce of the phase-A buffer
    (csrc: mmk_host::err_flag / peer_err): an error on rank 1 of 3 stops all
    three at the same iteration."""
    rng = np.random.default_rng(2)
    x, v, w = rng.random((30, 11)), rng.random((30, 3)), rng.random((3, 11))
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_nnmf_worker, args=(3, _free_port(), x, v, w, out, 1), nprocs=3, join=True)
        res = dict(out)
    assert all(res[r][5] for r in range(3))


def _mds_worker(rank, world, port, y, theta, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nt = len(P.tri_tiles(y.shape[0], 16))
    t0, t1 = P.tile_range(nt, world, rank)
    red = torch.from_numpy(P.tri_phase_a_model(y, theta, t0, t1, tile=16))
    P.allreduce_sum_(red)
    out[rank] = P.tri_phase_b_model(theta, red.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_mds_tile_sharding_gloo(world):
    rng = np.random.default_rng(1)
    n, dim = 45, 3
    a = rng.random((n, n))
    y = (a + a.T) / 2.0
    np.fill_diagonal(y, 0.0)
    theta = rng.uniform(-1, 1, size=(dim, n))
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_mds_worker, args=(world, _free_port(), y, theta, out), nprocs=world, join=True)
        res = dict(out)
    md = O.MdsData(1.0 - np.eye(n), y, dim)
    want = O.mds_update(theta, md)
    f_ref = O.mds_stress(theta, md)
    for r in range(world):
        got, f = res[r]
        np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-13)
        assert abs(f - f_ref) <= 1e-12 * f_ref


def test_update_only_error_sites():
    """Sites 16..31 of the device error record are update-only errors
    (csrc/mmk_common.cuh kUpdateSite); messages are keyed by the base site,
    and the reset / peer index (int64 max) is not update-only."""
    from paper_1003_3272_b200 import _lib
    idx = (17 << 48) | 12345
    assert _lib.update_only(idx) and _lib.split_site(idx) == (1, 12345)
    assert not _lib.update_only((1 << 48) | 5) and _lib.split_site((1 << 48) | 5) == (1, 5)
    assert not _lib.update_only(np.iinfo(np.int64).max)
