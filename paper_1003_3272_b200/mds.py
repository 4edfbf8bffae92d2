"""Multidimensional scaling by stress majorization, on the GPU.

Drop-in for the reference's MDS path (``pkg/src/mmkit/mds.py``):

  MdsProblem            mds.py:23-67    same validation + weighted_diss / weight_sums
  stress                mds.py:92-102   sum_{i<j} w_ij (y_ij - d_ij)^2
  mds_update            mds.py:114-144  separated per-point MM update
  mds_run               mds.py:245-257  uniform[-1,1] start, optional anchoring
  anchor_configuration  mds.py:202-225  post-hoc rigid motion (host, dim x dim)

The configuration theta is dim x n ("p x q" in the reference): row k holds
coordinate k of every point, which is also the coalesced layout the pairwise
kernel wants.  Stress and update are computed by ``csrc/mds.cu`` directly
from coordinate differences; no n x n matrix is ever formed on the device.
Unit weights (W = 1 - I, what the CLI always builds) are detected once and
never uploaded.  Large unit-weight fp32 problems (and ``PackedMdsProblem``,
a device-resident problem built straight into the packed layout) run on
``csrc/mds_tri.cu``: Y stored once as the packed upper triangle of 128 x 128
tiles and every unordered pair visited once per iteration.  ``stress_gradient`` / ``mds_surrogate`` are host fp64
property-test helpers.
"""

import ctypes
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _arrays as A
from . import _lib
from ._engine import DeviceMm
from .backend import SERIAL
from .datasets import votes_to_dissimilarity  # noqa: F401  (re-export)
from .driver import run_mm
from .errors import DomainError, InputError, NumericsError, ShapeError

__all__ = ["MdsProblem", "PackedMdsProblem", "stress", "stress_gradient", "mds_update", "mds_run",
           "mds_surrogate", "anchor_configuration", "votes_to_dissimilarity"]


def _coincide_msg(n):
    def msg(idx):
        i, j = divmod(idx, n)
        return (f"objects {i} and {j} coincide but are coupled with positive "
                "weight * dissimilarity; the surrogate is undefined there")
    return msg


@dataclass(frozen=True)
class MdsProblem:
    """Symmetric nonnegative weights and dissimilarities over q objects and
    the embedding dimension p."""

    weights: Any
    dissimilarities: Any
    p: int

    weighted_diss: np.ndarray = field(init=False, repr=False)
    weight_sums: np.ndarray = field(init=False, repr=False)
    unit_weights: bool = field(init=False, repr=False)
    _dev: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        w = np.ascontiguousarray(np.asarray(self.weights, dtype=np.float64))
        y = np.ascontiguousarray(np.asarray(self.dissimilarities, dtype=np.float64))
        if w.ndim != 2 or w.shape[0] != w.shape[1]:
            raise ShapeError(f"weights must be square, got {w.shape}")
        if y.shape != w.shape:
            raise ShapeError(f"dissimilarities {y.shape} do not match weights {w.shape}")
        for name, mat in (("weights", w), ("dissimilarities", y)):
            if not np.all(np.isfinite(mat)):
                raise DomainError(f"{name} contain non-finite entries")
            if np.min(mat) < 0.0:
                raise DomainError(f"{name} must be nonnegative")
            if not np.array_equal(mat, mat.T):
                raise DomainError(f"{name} must be exactly symmetric")
            if np.any(np.diag(mat) != 0.0):
                raise DomainError(f"{name} must have a zero diagonal")
        if self.p < 1:
            raise InputError(f"embedding dimension must be >= 1, got {self.p}")
        sums = w.sum(axis=1)
        lonely = np.flatnonzero(sums == 0.0)
        if lonely.size:
            raise DomainError(f"object {lonely[0]} has zero total weight; its position "
                              "is undefined")
        unit = bool(np.array_equal(w, 1.0 - np.eye(w.shape[0])))
        s = object.__setattr__
        s(self, "weights", w)
        s(self, "dissimilarities", y)
        s(self, "weighted_diss", w * y)
        s(self, "weight_sums", sums)
        s(self, "unit_weights", unit)

    @property
    def q(self):
        return self.weights.shape[0]

    def device_arrays(self, backend, torch):
        key = (str(backend.torch_device()), backend.dtype)
        d = self._dev.get(key)
        if d is None:
            dev = backend.torch_device()
            d = {
                "y": A.to_device(self.dissimilarities, backend, torch),
                "w": None if self.unit_weights else A.to_device(self.weights, backend, torch),
                "wsum": torch.from_numpy(self.weight_sums).to(dev),
            }
            self._dev[key] = d
        return d


TRI_MIN_POINTS = 4096   # Backend(mds_kernel="auto") uses the packed kernel from here
TILE = 128

_DOMAIN_MSGS = {
    2: "dissimilarities contain non-finite entries",
    3: "dissimilarities must be nonnegative",
    4: "dissimilarities must be exactly symmetric",
    5: "dissimilarities must have a zero diagonal",
}


def tile_count(n):
    """Tiles of the packed upper triangle for n points."""
    t = -(-n // TILE)
    return t * (t + 1) // 2


class PackedMdsProblem:
    """Unit-weight MDS problem (W = 1 - I, ``cli.py:181``) whose
    dissimilarities live on one GPU as the packed upper triangle of 128 x 128
    fp32 tiles (``csrc/mds_tri.cu``) -- the form BASELINE config 5
    (n = 65536) takes: 8.6 GB instead of 17.2 GB for full rows (and 34 GB
    for the reference's fp64 n x n, ``mds.py:60-63``).

    ``tiles = (t0, t1)`` is the range of linear tile indices held here: all of
    them for one GPU, a balanced slice per rank when sharded
    (``parallel.tile_range``).  Build with ``from_rows`` (a generator of fp32
    row blocks on the device) or ``from_dense`` (a full matrix, validated on
    the device like ``MdsProblem``, ``mds.py:40-58``)."""

    unit_weights = True

    def __init__(self, packed, n, p, tiles, device):
        if p < 1:
            raise InputError(f"embedding dimension must be >= 1, got {p}")
        if n < 2:
            raise DomainError("object 0 has zero total weight; its position is undefined")
        self.packed, self.n, self.p = packed, int(n), int(p)
        self.t0, self.t1 = int(tiles[0]), int(tiles[1])
        self.device = device

    @property
    def q(self):
        return self.n

    @classmethod
    def from_rows(cls, rows_fn, n, p, backend=SERIAL, tiles=None, block=4096, validate=False):
        """``rows_fn(r0, r1)`` returns rows [r0, r1) of Y as an fp32 CUDA
        tensor (n columns); blocks are multiples of 128 rows."""
        torch = _lib.torch_mod()
        dev = backend.torch_device()
        t0, t1 = tiles if tiles is not None else (0, tile_count(n))
        packed = torch.empty((t1 - t0) * TILE * TILE, dtype=torch.float32, device=dev)
        status = _lib.StatusBlock(torch, dev)
        status.clear_error()
        block = max(TILE, -(-block // TILE) * TILE)
        st = _lib.stream_handle(torch, dev)
        for r0 in range(0, n, block):
            r1 = min(n, r0 + block)
            yb = rows_fn(r0, r1)
            if yb.dtype != torch.float32 or yb.device != dev or yb.shape != (r1 - r0, n):
                raise ShapeError(f"row block [{r0}, {r1}) must be fp32 ({r1 - r0}, {n}) on {dev}")
            if yb.stride(1) != 1:
                yb = yb.contiguous()
            _lib.call("mmk_mds_tri_pack", _lib.ptr(yb), yb.stride(0), n, r0, r1 - r0,
                      _lib.ptr(packed), t0, t1, 1 if validate else 0, status.err_ptr, st)
        _, code, idx = status.read()
        _lib.raise_device_error(code, idx, {k: (lambda i, m=m: m) for k, m in _DOMAIN_MSGS.items()})
        return cls(packed, n, p, (t0, t1), dev)

    @classmethod
    def from_votes(cls, votes, p, backend=SERIAL, tiles=None):
        """Dissimilarities of a q x m roll-call matrix (1 yea, -1 nay, 0
        absent) computed on the tensor cores straight into the packed tiles
        (``csrc/mds_votes.cu``; reference votes_to_dissimilarity,
        mds.py:260-283) -- no q x q matrix on the host or the device."""
        torch = _lib.torch_mod()
        dev = backend.torch_device()
        shp = tuple(A.shape_of(votes))
        if len(shp) != 2:
            raise ShapeError(f"vote matrix must be 2-D, got {shp}")
        q, m = shp
        vt = votes if A.is_torch(votes) else torch.from_numpy(np.ascontiguousarray(votes))
        if vt.dtype not in (torch.float32, torch.float64):
            vt = vt.to(torch.float64)
        vt = vt.to(dev).contiguous()
        t0, t1 = tiles if tiles is not None else (0, tile_count(q))
        packed = torch.empty((t1 - t0) * TILE * TILE, dtype=torch.float32, device=dev)
        ws = torch.empty(_lib.ws_bytes("mmk_mds_votes_bytes", q, m), dtype=torch.uint8,
                         device=dev)
        status = _lib.StatusBlock(torch, dev)
        status.clear_error()
        _lib.call("mmk_mds_votes_tri", _lib.dtype_code(vt.dtype), _lib.ptr(vt), q, m,
                  _lib.ptr(packed), t0, t1, _lib.ptr(ws), ws.numel(), status.err_ptr,
                  _lib.stream_handle(torch, dev))
        _, code, idx = status.read()

        def pair(i):
            a, b = divmod(i, q)
            return (f"voters {a} and {b} share no roll call; their dissimilarity "
                    "is undefined")
        _lib.raise_device_error(code, idx, {
            6: lambda i: "votes must be 1 (yea), -1 (nay) or 0 (absent)", 7: pair})
        return cls(packed, q, p, (t0, t1), dev)

    @classmethod
    def from_packed(cls, packed, n, p, backend=SERIAL, tiles=None):
        """Already-packed tiles (this layout, e.g. saved from ``packed`` of an
        earlier problem) as a torch tensor of (t1 - t0) * 128 * 128 fp32
        values, on the device or in (pinned) host memory -- uploaded as is,
        no re-validation."""
        torch = _lib.torch_mod()
        dev = backend.torch_device()
        t0, t1 = tiles if tiles is not None else (0, tile_count(n))
        if not A.is_torch(packed) or packed.dtype != torch.float32 or \
                packed.numel() != (t1 - t0) * TILE * TILE:
            raise ShapeError(f"packed tiles must be an fp32 tensor of {(t1 - t0) * TILE * TILE} "
                             f"values for n={n}, tiles=({t0}, {t1})")
        return cls(packed.reshape(-1).to(dev, non_blocking=True), n, p, (t0, t1), dev)

    @classmethod
    def from_dense(cls, y, p, backend=SERIAL, tiles=None, validate=True):
        """Full n x n dissimilarities (numpy or torch), checked on the device
        for finiteness, sign, zero diagonal and exact symmetry."""
        torch = _lib.torch_mod()
        dev = backend.torch_device()
        shp = tuple(A.shape_of(y))
        if len(shp) != 2 or shp[0] != shp[1]:
            raise ShapeError(f"dissimilarities must be square, got {shp}")
        yt = (y if A.is_torch(y) else torch.from_numpy(np.ascontiguousarray(y)))
        yt = yt.to(device=dev, dtype=torch.float32).contiguous()
        n = shp[0]
        return cls.from_rows(lambda r0, r1: yt[r0:r1], n, p, backend, tiles, block=n,
                             validate=validate)


def _use_tri(problem, backend):
    ok = problem.unit_weights and backend.dtype == "fp32" and problem.p <= 3
    if backend.mds_kernel == "tri":
        if not ok:
            raise ShapeError("the packed-triangle MDS kernel needs unit weights, fp32 and p <= 3")
        return True
    return backend.mds_kernel == "auto" and ok and problem.q >= TRI_MIN_POINTS


def _packed_of(problem, backend):
    """The packed form of a host MdsProblem (cached per device)."""
    key = (str(backend.torch_device()), "tri")
    pk = problem._dev.get(key)
    if pk is None:
        torch = _lib.torch_mod()
        dev = backend.torch_device()
        y = problem.dissimilarities
        pk = PackedMdsProblem.from_rows(
            lambda r0, r1: torch.from_numpy(np.ascontiguousarray(y[r0:r1], dtype=np.float32)
                                            ).to(dev),
            problem.q, problem.p, backend, block=2048)
        problem._dev[key] = pk
    return pk


def _make_mm(problem, backend):
    if isinstance(problem, PackedMdsProblem):
        return _GpuMdsTri(problem, backend)
    if _use_tri(problem, backend):
        return _GpuMdsTri(_packed_of(problem, backend), backend)
    return _GpuMds(problem, backend)


def _check_theta(theta, problem):
    shp = tuple(A.shape_of(theta))
    if len(shp) != 2 or shp != (problem.p, problem.q):
        raise ShapeError(f"configuration must be {problem.p}x{problem.q}, got {shp}")


class _GpuMds(DeviceMm):
    direction = "minimize"

    def __init__(self, problem, backend):
        super().__init__(backend)
        torch = self.torch
        self.problem = problem
        d = problem.device_arrays(backend, torch)
        self.y, self.w, self.wsum = d["y"], d["w"], d["wsum"]
        self.n, self.dim = problem.q, problem.p
        self.ws = torch.zeros(_lib.ws_bytes("mmk_mds_ws_bytes", self.code, self.n, self.dim,
                                            self.n), dtype=torch.uint8, device=self.device)

    def device_state(self, theta):
        return A.to_device(theta, self.backend, self.torch)

    def _alloc_like(self, s):
        return self.torch.empty_like(s)

    def _copy_into(self, dst, src):
        dst.copy_(src)

    def _bytes_per_iter(self):
        k = 1 if self.w is None else 2
        return float(k * self.n * self.n * self.y.element_size())

    def _messages(self):
        return {1: _coincide_msg(self.n)}

    def _iterate(self, theta, out, f_ptr, err_ptr,
                 flags=_lib.MMK_MDS_UPDATE | _lib.MMK_MDS_OBJECTIVE):
        _lib.call("mmk_mds_iter", self.code, _lib.ptr(self.y), _lib.ptr(self.w), self.n,
                  _lib.ptr(self.wsum), _lib.ptr(theta), _lib.ptr(out), self.n, self.dim, self.n,
                  0, self.n, flags, _lib.ptr(self.ws), self.ws.numel(), f_ptr, err_ptr,
                  self.stream())

    def _engine_create(self, a, b, rule, trace, stamp, ctl, eng):
        self._keep = (a, b)
        _lib.call("mmk_mds_engine_create", self.code, _lib.ptr(self.y), _lib.ptr(self.w), self.n,
                  _lib.ptr(self.wsum), _lib.ptr(a), _lib.ptr(b), None, None, self.dim, self.n, 0,
                  self.n, self.n, _lib.ptr(self.ws), self.ws.numel(), None, ctypes.byref(rule),
                  _lib.ptr(trace), _lib.ptr(stamp), _lib.ptr(ctl), self.status.err_ptr,
                  ctypes.byref(eng))

    def stress_only(self, theta):
        out = self.torch.empty_like(theta)
        self._iterate(theta, out, self.status.f_ptr, self.status.err_ptr, _lib.MMK_MDS_OBJECTIVE)
        return self._check_error()

    def update_only(self, theta):
        out = self.torch.empty_like(theta)
        self._iterate(theta, out, self.status.f_ptr, self.status.err_ptr, _lib.MMK_MDS_UPDATE)
        self._check_error()
        return out

    def surrogate(self, state, anchor):
        return mds_surrogate(state, anchor, self.problem)


class _GpuMdsTri(DeviceMm):
    """Packed-triangle MDS (``csrc/mds_tri.cu``); sharded when ``comm`` (an
    NCCL communicator) or ``group`` (a torch process group) is set and the
    problem holds a slice of the tiles: phase A leaves [zs_i, A_i | stress]
    per point, one all-reduce combines the ranks, phase B updates every
    point redundantly."""

    direction = "minimize"

    def __init__(self, packed, backend, comm=None, group=None):
        if backend.dtype != "fp32":
            raise ShapeError("the packed-triangle MDS kernel runs in fp32")
        super().__init__(backend)
        torch = self.torch
        self.problem = packed
        self.pk, self.n, self.dim = packed.packed, packed.n, packed.p
        self.t0, self.t1 = packed.t0, packed.t1
        self.comm, self.group = comm, group
        self.ws = torch.zeros(_lib.ws_bytes("mmk_mds_tri_ws_bytes", self.n, self.dim, self.t0,
                                            self.t1), dtype=torch.uint8, device=self.device)
        self.red = torch.zeros(_lib.load().mmk_mds_tri_reduce_len(self.n, self.dim),
                               dtype=torch.float64, device=self.device)

    def device_state(self, theta):
        return A.to_device(theta, self.backend, self.torch)

    def _alloc_like(self, s):
        return self.torch.empty_like(s)

    def _copy_into(self, dst, src):
        dst.copy_(src)

    def _bytes_per_iter(self):
        return float((self.t1 - self.t0) * TILE * TILE * 4)

    def _messages(self):
        return {1: _coincide_msg(self.n)}

    def _iterate(self, theta, out, f_ptr, err_ptr):
        st = self.stream()
        L = _lib
        if self.group is None and self.comm is None:
            L.call("mmk_mds_tri_iter", L.ptr(self.pk), self.t0, self.t1, L.ptr(theta), L.ptr(out),
                   self.dim, self.n, L.ptr(self.ws), self.ws.numel(), L.ptr(self.red), f_ptr,
                   err_ptr, st)
            return
        L.call("mmk_mds_tri_iter_a", L.ptr(self.pk), self.t0, self.t1, L.ptr(theta), self.dim,
               self.n, L.ptr(self.ws), self.ws.numel(), L.ptr(self.red), err_ptr, st)
        if self.comm is not None:
            L.call("mmk_allreduce_f64", L.ptr(self.red), self.red.numel(),
                   ctypes.c_void_p(self.comm), st)
        else:
            import torch.distributed as dist
            dist.all_reduce(self.red, group=self.group)
        L.call("mmk_mds_tri_iter_b", L.ptr(theta), L.ptr(out), self.dim, self.n, L.ptr(self.red),
               f_ptr, err_ptr, st)

    def _engine_create(self, a, b, rule, trace, stamp, ctl, eng):
        self._keep = (a, b)
        comm = ctypes.c_void_p(self.comm) if self.comm is not None else None
        _lib.call("mmk_mds_tri_engine_create", _lib.ptr(self.pk), self.t0, self.t1, _lib.ptr(a),
                  _lib.ptr(b), self.dim, self.n, _lib.ptr(self.ws), self.ws.numel(),
                  _lib.ptr(self.red), comm, ctypes.byref(rule), _lib.ptr(trace),
                  _lib.ptr(stamp), _lib.ptr(ctl), self.status.err_ptr, ctypes.byref(eng))

    def stress_only(self, theta):
        out = self.torch.empty_like(theta)
        self._iterate(theta, out, self.status.f_ptr, self.status.err_ptr)
        return self._check_error()

    def update_only(self, theta):
        out = self.torch.empty_like(theta)
        self._iterate(theta, out, self.status.f_ptr, self.status.err_ptr)
        self._check_error()
        return out

    def surrogate(self, state, anchor):
        raise NotImplementedError("surrogate is a host helper of dense MdsProblem instances")


def stress(theta, problem, backend=SERIAL):
    """Weighted squared mismatch over unordered pairs."""
    _check_theta(theta, problem)
    mm = _make_mm(problem, backend)
    return mm.stress_only(mm.device_state(theta))


def mds_update(theta, problem, backend=SERIAL):
    """One parallel stress-majorization step (every point moves given the
    previous configuration)."""
    _check_theta(theta, problem)
    mm = _make_mm(problem, backend)
    return A.to_user(mm.update_only(mm.device_state(theta)), theta)


def anchor_configuration(theta):
    """Rigid motion putting object 0 at the origin and zeroing the first p-1
    coordinates of object 1; stress is unchanged (host, O(p^2 q))."""
    was_torch = A.is_torch(theta)
    t = np.ascontiguousarray(_host(theta))
    if t.ndim != 2:
        raise ShapeError(f"configuration must be 2-D, got {t.shape}")
    p, q = t.shape
    out = t - t[:, [0]]
    if p >= 2 and q >= 2:
        u = out[:, 1]
        norm = float(np.sqrt(u @ u))
        if norm != 0.0:
            target = np.zeros(p)
            target[-1] = -norm if u[-1] >= 0.0 else norm
            v = u - target
            vsq = float(v @ v)
            if vsq != 0.0:
                refl = np.eye(p) - (2.0 / vsq) * np.outer(v, v)
                refl[0, :] = -refl[0, :]      # det +1: a rotation
                out = refl @ out
    if was_torch:
        import torch
        return torch.as_tensor(out, device=theta.device, dtype=theta.dtype)
    return out


def mds_run(problem, config, backend=SERIAL, anchor=False, theta0=None):
    """Minimize stress from a uniform[-1, 1] start drawn with ``config.seed``
    (or from ``theta0``); with ``anchor`` the result is rigidly moved to the
    anchoring convention afterwards (trace unchanged)."""
    if theta0 is None:
        theta0 = np.random.default_rng(config.seed).uniform(-1.0, 1.0,
                                                            size=(problem.p, problem.q))
    mm = _make_mm(problem, backend)
    state, trace = run_mm(mm, mm.device_state(theta0), config)
    theta = A.to_user(state, theta0)
    if anchor:
        theta = anchor_configuration(theta)
    return theta, trace


# ---------------------------------------------------------------------------
def _host(a):
    return A.to_user(a, np.empty(0)) if A.is_torch(a) else np.asarray(a, dtype=np.float64)


def _host_d2(theta):
    g = theta.T @ theta
    dg = np.diag(g)
    return np.maximum(dg[:, None] + dg[None, :] - 2.0 * g, 0.0)


def stress_gradient(theta, problem, backend=SERIAL):
    """Analytic stress gradient (mds.py:147-167), on the device: the rows
    kernel with MMK_MDS_GRADIENT.  Coincident points with positive weight
    raise the reference's NumericsError."""
    _check_theta(theta, problem)
    if isinstance(problem, PackedMdsProblem):
        raise ShapeError("stress_gradient takes a dense MdsProblem")
    mm = _GpuMds(problem, backend)
    th = mm.device_state(theta)
    out = mm.torch.empty_like(th)
    mm._iterate(th, out, mm.status.f_ptr, mm.status.err_ptr, _lib.MMK_MDS_GRADIENT)
    mm._check_error()
    return A.to_user(out, theta)


def mds_surrogate(theta, theta_n, problem):
    """Stress majorizer at (theta | theta_n), constants kept (host fp64)."""
    _check_theta(theta, problem)
    _check_theta(theta_n, problem)
    t, tn = _host(theta), _host(theta_n)
    w, y = problem.weights, problem.dissimilarities
    total = 0.0
    for i in range(problem.q):
        for j in range(i + 1, problem.q):
            if w[i, j] == 0.0 and y[i, j] == 0.0:
                continue
            gap_n = tn[:, i] - tn[:, j]
            dist_n = float(np.sqrt(gap_n @ gap_n))
            total += w[i, j] * y[i, j] ** 2
            if w[i, j] * y[i, j] > 0.0:
                if dist_n == 0.0:
                    raise NumericsError(f"objects {i} and {j} coincide at the anchor point")
                total -= 2.0 * w[i, j] * y[i, j] * float((t[:, i] - t[:, j]) @ gap_n) / dist_n
            c = 0.5 * (tn[:, i] + tn[:, j])
            di, dj = t[:, i] - c, t[:, j] - c
            total += 2.0 * w[i, j] * (float(di @ di) + float(dj @ dj))
    return total
