"""Multi-GPU sharding of the MM iterations (one process per GPU).

SURVEY.md section 8(e): the paths shard where the math does --

* NNMF: rows of X and V are split across ranks, W is replicated.  The V step
  is rank-local; the W step needs sum_rows V'^T X and V'^T V', so phase A of
  ``mmk_nnmf_iter_a`` leaves this rank's [P | G_V | f] partials in a fp64
  buffer, one NCCL all-reduce (sum) combines them, and phase B finishes W'
  redundantly on every rank (no broadcast).
* MDS (rows kernel): points (rows of Y) are split; each rank updates its own
  points from the full previous configuration, then the coordinates are
  all-gathered and the stress partials all-reduced.
* MDS (packed triangle, large unit-weight problems): the TILES of the packed
  upper triangle are split evenly (``tile_range``); phase A leaves per-point
  [zs_i, A_i] partials and the stress partial, one all-reduce combines them
  and every rank applies the (cheap, O(n dim)) update to all points.
* PET: rays are split; the back-projection vector and loglik partial (the
  phase-A buffer) are all-reduced before the pixel update.

``shard_rows`` is the row partition shared by all three.  The collectives
are issued on the compute stream through ``torch.distributed`` (NCCL over
NVLink/NVSwitch on the B200 box, gloo in the CPU tests).
"""

import numpy as np


def shard_rows(n, world, rank):
    """Contiguous near-equal row range [lo, hi) of rank ``rank``; the first
    ``n % world`` ranks get one extra row (the reference's partition rule,
    kernels.py:79-89)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def tile_range(ntiles, world, rank):
    """Contiguous balanced slice [t0, t1) of the packed-triangle MDS tiles
    (``csrc/mds_tri.cu``) held and processed by ``rank``: every rank gets
    the same number of 64 KB tiles (+-1), i.e. the same HBM traffic."""
    return ntiles * rank // world, ntiles * (rank + 1) // world


def padded_rows(n, world):
    """Equal-size padded shard length used for all-gathers."""
    return -(-n // world)


def allreduce_sum_(t, group=None):
    import torch.distributed as dist
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def nccl_comm_ptr(group=None):
    """ncclComm_t of torch's process group (for the in-graph collectives of
    the fused engine); None when the backend is not NCCL."""
    import torch
    import torch.distributed as dist
    try:
        pg = group or dist.distributed_c10d._get_default_group()
        backend = pg._get_backend(torch.device("cuda"))
        return int(backend._comm_ptr())
    except Exception:
        return None


class ShardedNnmf:
    """Row-sharded Frobenius NNMF on this rank's GPU: X_local (rows lo:hi),
    V_local, W replicated.  ``iterate`` = phase A, all-reduce, phase B."""

    def __init__(self, x_local, v_local, w, rank_of_r, backend, group=None):
        from . import _lib
        torch = _lib.torch_mod()
        self.torch, self.backend, self.group = torch, backend, group
        self.code = _lib.dtype_code(backend.torch_dtype())
        self.x = x_local
        self.m, self.n = x_local.shape
        self.r = rank_of_r
        dev = x_local.device
        self.ws = torch.zeros(_lib.ws_bytes("mmk_nnmf_ws_bytes", self.code, max(self.m, 1), self.n,
                                            self.r), dtype=torch.uint8, device=dev)
        self.red = torch.zeros(_lib.load().mmk_nnmf_reduce_len(self.n, self.r),
                               dtype=torch.float64, device=dev)
        self.status = _lib.StatusBlock(torch, dev)
        self.v = [v_local, torch.empty_like(v_local)]
        self.w = [w, torch.empty_like(w)]
        self.cur = 0
        self._lib = _lib

    def iterate(self, world):
        L = self._lib
        a, b = self.cur, 1 - self.cur
        st = L.stream_handle(self.torch, self.x.device)
        L.call("mmk_nnmf_iter_a", self.code, L.ptr(self.x), self.x.stride(0), L.ptr(self.v[a]),
               L.ptr(self.w[a]), L.ptr(self.v[b]), self.m, self.n, self.r, L.ptr(self.ws),
               self.ws.numel(), L.ptr(self.red), self.status.err_ptr, st)
        if world > 1:
            allreduce_sum_(self.red, self.group)
        L.call("mmk_nnmf_iter_b", self.code, L.ptr(self.w[a]), L.ptr(self.w[b]), self.n, self.r,
               L.ptr(self.red), self.status.f_ptr, self.status.err_ptr, st)
        self.cur = b

    def objective_ptr(self):
        return self.status.f_ptr


def phase_a_model(x, v, w, error=False):
    """Host fp64 model of phase A's buffer for one shard (tests only):
    [P | G_V' | f | device-error flag]."""
    q = x @ w.T
    g_w = w @ w.T
    v2 = v * (q / (v @ g_w + 1e-300))
    f = float(np.sum((x - v @ w) ** 2))
    return v2, np.concatenate([(v2.T @ x).ravel(), (v2.T @ v2).ravel(), [f, float(error)]])


def phase_b_model(w, red, n, r):
    """W', f, and whether any rank flagged a device error (all ranks agree)."""
    p = red[:r * n].reshape(r, n)
    g = red[r * n:r * n + r * r].reshape(r, r)
    return w * (p / (g @ w + 1e-300)), red[r * n + r * r], red[r * n + r * r + 1] > 0.5


def tri_tiles(n, tile=128):
    """(I, J) of every packed-triangle tile in linear order (csrc/mds_tri.cu)."""
    t = -(-n // tile)
    return [(i, j) for i in range(t) for j in range(i, t)]


def tri_phase_a_model(y, theta, t0, t1, tile=128):
    """Host fp64 model of ``mmk_mds_tri_iter_a`` for tiles [t0, t1) (tests
    only): red = [C (n x dim, row-major) | stress partial | S if t0 == 0 |
    device-error flag]."""
    dim, n = theta.shape
    c = np.zeros((n, dim))
    stress = 0.0
    for (bi, bj) in tri_tiles(n, tile)[t0:t1]:
        i = np.arange(bi * tile, min(n, (bi + 1) * tile))
        j = np.arange(bj * tile, min(n, (bj + 1) * tile))
        ii, jj = np.meshgrid(i, j, indexing="ij")
        keep = jj > ii
        ii, jj = ii[keep], jj[keep]
        g = theta[:, jj] - theta[:, ii]
        d = np.sqrt((g * g).sum(0))
        yy = y[ii, jj]
        z = np.where(yy > 0.0, yy / np.where(d > 0.0, d, 1.0), 0.0)
        stress += float(((yy - d) ** 2).sum())
        np.add.at(c, ii, (z * g).T)
        np.add.at(c, jj, -(z * g).T)
    s = theta.sum(1) if t0 == 0 else np.zeros(dim)
    return np.concatenate([c.ravel(), [stress], s, [0.0]])


def tri_phase_b_model(theta, red):
    """Host model of ``mmk_mds_tri_iter_b``: the unit-weight MM update."""
    dim, n = theta.shape
    c = red[:n * dim].reshape(n, dim).T
    s = red[n * dim + 1:n * dim + 1 + dim]
    w = n - 1.0
    return (theta * (w - 1.0) + s[:, None] - c) / (2.0 * w), red[n * dim]


# ---------------------------------------------------------------------------
# Public sharded solvers (one process per GPU, torch.distributed group).
# Each iteration: phase A on this rank's rows / tiles / rays, ONE all-reduce
# of the fp64 reduction buffer -- whose last slot carries the device-error
# flag (csrc: mmk_host::err_flag / peer_err), so every rank stops at the same
# iteration -- and phase B redundantly on every rank.
#
# With an NCCL group and Backend(fused=True) the whole run is the device
# engine: the per-iteration kernels and the ncclAllReduce captured in ONE CUDA
# graph with the stopping rule on the device (csrc/engine.cu).  Otherwise
# (gloo, fused=False) run_mm's per-iteration protocol drives it with the
# all-reduce issued through torch.distributed.  Either way the objective
# trace is the all-reduced value and identical on every rank.
MMK_E_PEER = 6   # include/mmk.h: error-record code "another rank flagged an error"


def _combine_error_records(status, group):
    """Slow path, only after a device error: every rank's record is nonzero
    (its own error, or MMK_E_PEER); reduce them to the first real offender
    (largest code, then smallest index) so all ranks raise the same error."""
    import torch
    import torch.distributed as dist
    rec = status.dev[1:3].clone()
    code = rec[0:1].clone()
    code[code == MMK_E_PEER] = 0
    dist.all_reduce(code, op=dist.ReduceOp.MAX, group=group)
    idx = rec[1:2].clone()
    idx[rec[0:1] != code] = torch.iinfo(torch.int64).max
    dist.all_reduce(idx, op=dist.ReduceOp.MIN, group=group)
    status.dev[1:2].copy_(code)
    status.dev[2:3].copy_(idx)


def _shard(mm, group, iter_fns=None):
    """Configure a DeviceMm for a sharded run (see the section comment)."""
    mm.group = group
    comm = nccl_comm_ptr(group) if group is not None else None
    mm.comm = comm
    mm._fused = bool(mm.backend.fused) and comm is not None
    def _status_read():
        f, code, idx = mm.status.read()
        if code == 0 or group is None:
            return f, code, idx
        _combine_error_records(mm.status, group)
        return mm.status.read()
    mm._status_read = _status_read
    return mm


def _default_group(group):
    if group is None:   # the default process group, as torch.distributed collectives use it
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            group = dist.group.WORLD
    return group


def _make_sharded_nnmf(base_cls, iter_a, iter_b):
    class _Sharded(base_cls):
        def _iterate(self, s, out, f_ptr, err_ptr):
            from . import _lib as L
            st = self.stream()
            L.call(iter_a, self.code, L.ptr(self.x), self.x.stride(0), L.ptr(s.v), L.ptr(s.w),
                   L.ptr(out.v), self.m, self.n, self.r, L.ptr(self.ws), self.ws.numel(),
                   L.ptr(self.red), err_ptr, st)
            if self.comm is not None:
                L.call("mmk_allreduce_f64", L.ptr(self.red), self.red.numel(),
                       L.ctypes.c_void_p(self.comm), st)
            elif self.group is not None:
                allreduce_sum_(self.red, self.group)
            L.call(iter_b, self.code, L.ptr(s.w), L.ptr(out.w), self.n, self.r, L.ptr(self.red),
                   f_ptr, err_ptr, st)
    return _Sharded


def nnmf_run_sharded(x_local, rank, config, backend, group=None, state0=None, poisson=False):
    """Row-sharded NNMF (Frobenius, or the Poisson fit with ``poisson=True``):
    this rank holds rows ``x_local`` of X (a CUDA tensor or array) and the
    matching rows of V; W is replicated.  ``state0`` = (V_local, W) (required:
    the ranks must agree on W and on the split of V).  Returns
    (FactorPair(V_local, W), MmTrace); every rank gets the same trace."""
    from . import nnmf as N
    from .driver import run_mm
    if state0 is None:
        raise ValueError("nnmf_run_sharded needs state0 = (V_local, W)")
    group = _default_group(group)
    prob = N.NnmfProblem(x=x_local, rank=rank)
    if poisson:
        cls = _make_sharded_nnmf(N._GpuPoissonNnmf, "mmk_nnmf_poisson_iter_a",
                                 "mmk_nnmf_poisson_iter_b")
    else:
        cls = _make_sharded_nnmf(N._GpuNnmf, "mmk_nnmf_iter_a", "mmk_nnmf_iter_b")
    mm = _shard(cls(prob, backend), group)
    state, trace = run_mm(mm, mm.device_state(N.FactorPair(state0[0], state0[1])), config)
    return state, trace


def mds_run_sharded(problem, config, backend, group=None, theta0=None):
    """Sharded MDS; every rank returns the same configuration and trace.

    * ``PackedMdsProblem`` (unit weights, packed triangle): ``problem`` is this
      rank's tile slice (``tile_range(ntiles, world, rank)``); one all-reduce
      of the per-point accumulators per iteration.
    * dense ``MdsProblem`` (any weights): rank r owns the points
      ``shard_rows(n, world, r)`` and uploads only their rows of Y (and W);
      per iteration it updates its points (``mmk_mds_iter`` on its row block),
      all-gathers the new coordinates and all-reduces the stress partial
      (SURVEY.md 8(e)).
    theta is replicated."""
    from . import mds as D
    from .driver import run_mm
    group = _default_group(group)
    if not isinstance(problem, D.PackedMdsProblem):
        return _mds_rows_sharded(problem, config, backend, group, theta0)
    if theta0 is None:
        theta0 = np.random.default_rng(config.seed).uniform(-1.0, 1.0,
                                                            size=(problem.p, problem.q))
    mm = _shard(D._GpuMdsTri(problem, backend, group=group), group)
    return run_mm(mm, mm.device_state(theta0), config)


def _mds_rows_sharded(problem, config, backend, group, theta0):
    import torch
    import torch.distributed as dist

    from . import _arrays as A
    from . import _lib as L
    from . import mds as D
    from ._engine import DeviceMm
    from .driver import run_mm
    world = dist.get_world_size(group) if group is not None else 1
    rank = dist.get_rank(group) if group is not None else 0
    n, dim = problem.q, problem.p
    bounds = [shard_rows(n, world, r) for r in range(world)]
    lo, hi = bounds[rank]
    pad = max(b - a for a, b in bounds)
    if theta0 is None:
        theta0 = np.random.default_rng(config.seed).uniform(-1.0, 1.0, size=(dim, n))

    class _RowsMm(DeviceMm):
        direction = "minimize"

        def __init__(self):
            super().__init__(backend)
            t = self.torch
            self.y = A.to_device(problem.dissimilarities[lo:hi], backend, t)
            self.w = None if problem.unit_weights else A.to_device(problem.weights[lo:hi],
                                                                   backend, t)
            self.wsum = t.from_numpy(np.ascontiguousarray(problem.weight_sums)).to(self.device)
            self.ws = t.zeros(L.ws_bytes("mmk_mds_ws_bytes", self.code, n, dim, max(hi - lo, 1)),
                              dtype=t.uint8, device=self.device)
            self.local = t.zeros((dim, pad), dtype=self.dtype, device=self.device)
            self.parts = [t.zeros((dim, pad), dtype=self.dtype, device=self.device)
                          for _ in range(world)]

        def device_state(self, theta):
            return A.to_device(theta, backend, self.torch)

        def _alloc_like(self, s):
            return self.torch.empty_like(s)

        def _copy_into(self, dst, src):
            dst.copy_(src)

        def _bytes_per_iter(self):
            return float((1 if self.w is None else 2) * (hi - lo) * n * self.y.element_size())

        def _messages(self):
            return {1: D._coincide_msg(n)}

        def _iterate(self, theta, out, f_ptr, err_ptr):
            P = L.ptr
            if hi > lo:
                L.call("mmk_mds_iter", self.code, P(self.y), P(self.w) if self.w is not None
                       else None, n, P(self.wsum), P(theta), P(self.local), pad, dim, n, lo,
                       hi - lo, L.MMK_MDS_UPDATE | L.MMK_MDS_OBJECTIVE, P(self.ws),
                       self.ws.numel(), f_ptr, err_ptr, self.stream())
            else:
                self.status.dev[0:1].zero_()
            if group is not None:
                dist.all_reduce(self.status.dev[0:1].view(self.torch.float64), group=group)
                dist.all_gather(self.parts, self.local, group=group)
                _combine_error_records(self.status, group)
            else:
                self.parts[0].copy_(self.local)
            for r, (a, b) in enumerate(bounds):
                out[:, a:b].copy_(self.parts[r][:, :b - a])

    mm = _RowsMm()
    mm._fused = False     # per-iteration protocol
    return run_mm(mm, mm.device_state(theta0), config)


def pet_run_sharded(problem, config, backend, group=None):
    """Ray-sharded penalized PET: rank r holds the rays
    shard_rows(n_rays, world, r) of a host-matrix ``PetProblem`` (dense or
    sparse projector); lam is replicated.  Per iteration: the projection phase
    on the local rays leaves [b | loglik] (p + 1 doubles), one all-reduce,
    then every rank applies the same pixel update and objective.  Returns
    (lam, MmTrace) on every rank, from the flat start lam = 1 as pet_run."""
    import torch.distributed as dist

    from . import _arrays as A
    from . import _lib as L
    from . import pet as PT
    from .driver import run_mm
    group = _default_group(group)
    world = dist.get_world_size(group) if group is not None else 1
    rank = dist.get_rank(group) if group is not None else 0
    lo, hi = shard_rows(problem.n_rays, world, rank)

    class _Sharded(PT._GpuPet):
        def _iterate(self, lam, out, f_ptr, err_ptr,
                     flags=L.MMK_PET_UPDATE | L.MMK_PET_OBJECTIVE):
            st, P = self.stream(), L.ptr
            if self.sparse:
                sa = self.sa
                L.call("mmk_pet_sparse_iter_a", self.code, P(sa["rptr"]), P(sa["ridx"]),
                       P(sa["rval"]), P(sa["cptr"]), P(sa["cidx"]), P(sa["cval"]), P(self.y),
                       P(lam), self.d, self.p, P(self.ws), self.ws.numel(), P(self.red),
                       err_ptr, st)
            else:
                L.call("mmk_pet_iter_a", self.code, P(self.e), self.e.stride(0), P(self.y),
                       P(lam), self.d, self.p, P(self.ws), self.ws.numel(), P(self.red), err_ptr,
                       st)
            if self.comm is not None:
                L.call("mmk_allreduce_f64", P(self.red), self.red.numel(),
                       L.ctypes.c_void_p(self.comm), st)
            elif group is not None:
                allreduce_sum_(self.red, group)
            L.call("mmk_pet_iter_b", self.code, P(lam), P(out), self.p, P(self.ptr), P(self.idx),
                   self.mu, flags, P(self.red), P(self.ws), self.ws.numel(), f_ptr, err_ptr, st)

    mm = _shard(_Sharded(problem, backend, rows=(lo, hi)), group)
    state, trace = run_mm(mm, mm.device_state(np.ones(problem.n_pixels)), config)
    return A.to_user(state, problem.e), trace
