"""Penalized PET reconstruction by Poisson MM, on the GPU.

Drop-in for the reference's reconstruction path (``pkg/src/mmkit/pet.py``):

  PetProblem               pet.py:213-285  same validation + derived arrays
  pet_loglik               pet.py:318-323
  pet_penalized_objective  pet.py:341-346
  pet_update               pet.py:363-417  (EM for mu = 0, positive root else)
  pet_run                  pet.py:477-480  flat start lam = 1
  INTENSITY_FLOOR          pet.py:36       (fp32 storage floors at FLT_MIN)

One MM iteration = one pass over E in libmmk.so (``csrc/pet.cu``): forward
projection, count ratio, loglik, back-projection, pixel update and penalty.
Geometry / phantom / count simulation are host-side input builders
(``datasets``); ``pet_penalized_gradient`` and ``pet_surrogate`` are host
fp64 property-test helpers.
"""

import ctypes
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _arrays as A
from . import _lib
from ._engine import DeviceMm
from .backend import SERIAL
from .datasets import (PetGeometry, build_neighborhoods, build_system_matrix,  # noqa: F401
                       default_phantom, simulate_counts)
from .driver import run_mm
from .errors import DomainError, InputError, NumericsError, ShapeError

__all__ = ["PetGeometry", "PetProblem", "SparsePetProblem", "system_matrix_device", "build_system_matrix", "build_neighborhoods",
           "simulate_counts", "default_phantom", "pet_loglik", "pet_penalized_objective",
           "pet_penalized_gradient", "pet_update", "pet_run", "pet_surrogate"]

INTENSITY_FLOOR = 1e-300

_MSG = {
    1: lambda i: ("a ray with positive counts has zero expected counts; the "
                  f"loglikelihood is -inf (ray {i})"),
    2: lambda j: ("negative discriminant in the penalized intensity update; this indicates "
                  f"a bug, not a data problem (pixel {j})"),
}


@dataclass(frozen=True)
class PetProblem:
    """System matrix E (rays x pixels, unit l1 columns), counts y, penalty mu
    and the pixel adjacency lists."""

    e: Any
    y: Any
    mu: float
    neighborhoods: list

    col_sums: np.ndarray = field(init=False, repr=False)
    degrees: np.ndarray = field(init=False, repr=False)
    nbr_indptr: np.ndarray = field(init=False, repr=False)
    nbr_indices: np.ndarray = field(init=False, repr=False)
    pair_left: np.ndarray = field(init=False, repr=False)
    pair_right: np.ndarray = field(init=False, repr=False)
    _dev: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        e, y = self.e, self.y
        if not A.is_torch(e):
            e = np.ascontiguousarray(np.asarray(e, dtype=np.float64))
        if not A.is_torch(y):
            y = np.asarray(y, dtype=np.float64)
        if e.ndim != 2:
            raise ShapeError(f"system matrix must be 2-D, got {tuple(e.shape)}")
        if y.ndim != 1 or y.shape[0] != e.shape[0]:
            raise ShapeError(f"counts shape {tuple(y.shape)} does not match {e.shape[0]} rays")
        if A.min_value(e) < 0.0:
            raise DomainError("detection coefficients must be nonnegative")
        if A.min_value(y) < 0.0:
            raise DomainError("counts must be nonnegative")
        if self.mu < 0.0:
            raise DomainError(f"penalty constant must be >= 0, got {self.mu}")
        col = (e.double().sum(dim=0).cpu().numpy() if A.is_torch(e) else e.sum(axis=0))
        if np.max(np.abs(col - 1.0)) > 1e-8:
            raise DomainError("system matrix columns must have unit l1 norm "
                              "(normalize as build_system_matrix does)")
        p = e.shape[1]
        if len(self.neighborhoods) != p:
            raise ShapeError(f"{len(self.neighborhoods)} neighborhoods for {p} pixels")
        members = [set(a) for a in self.neighborhoods]
        pairs = set()
        for j, around in enumerate(self.neighborhoods):
            for k in around:
                if k == j:
                    raise DomainError(f"pixel {j} lists itself as a neighbor")
                if j not in members[k]:
                    raise DomainError(f"neighborhood is not symmetric: {k} in N({j}) but "
                                      f"{j} not in N({k})")
                pairs.add((min(j, k), max(j, k)))
        pairs = sorted(pairs)
        indptr = np.zeros(p + 1, dtype=np.int64)
        indptr[1:] = np.cumsum([len(a) for a in self.neighborhoods])
        indices = np.fromiter((k for a in self.neighborhoods for k in a), dtype=np.int64,
                              count=int(indptr[-1]))
        s = object.__setattr__
        s(self, "e", e)
        s(self, "y", y)
        s(self, "col_sums", col)
        s(self, "degrees", np.diff(indptr).astype(np.float64))
        s(self, "nbr_indptr", indptr)
        s(self, "nbr_indices", indices)
        s(self, "pair_left", np.array([a for a, _ in pairs], dtype=np.int64))
        s(self, "pair_right", np.array([b for _, b in pairs], dtype=np.int64))

    @property
    def n_pixels(self):
        return self.e.shape[1]

    @property
    def n_rays(self):
        return self.e.shape[0]

    @property
    def e_t(self):
        """Transposed view of E (the reference stores a dense copy; the GPU
        kernels back-project from E directly)."""
        return self.e.T

    def device_arrays(self, backend, torch, dense=True, rows=None):
        """E (dense only), y, and the neighbour CSR on the device; with
        ``rows = (lo, hi)`` (a ray shard) only those rows of E and y are
        uploaded."""
        lo, hi = rows if rows is not None else (0, self.n_rays)
        key = (str(backend.torch_device()), backend.dtype, dense, lo, hi)
        d = self._dev.get(key)
        if d is None:
            dev = backend.torch_device()
            d = {
                "e": A.to_device(self.e[lo:hi], backend, torch) if dense else None,
                "y": A.to_device(self.y[lo:hi], backend, torch),
                "ptr": torch.from_numpy(self.nbr_indptr.astype(np.int32)).to(dev),
                "idx": torch.from_numpy(self.nbr_indices.astype(np.int32)).to(dev),
            }
            if d["idx"].numel() == 0:
                d["idx"] = torch.zeros(1, dtype=torch.int32, device=dev)
            self._dev[key] = d
        return d


SPARSE_DENSITY = 0.25   # Backend(pet_kernel="auto") switches to CSR/CSC below this


def system_matrix_device(geometry, backend=SERIAL):
    """The Siddon system matrix of ``geometry`` built on the GPU
    (``csrc/pet_siddon.cu``; the reference's Python loop is pet.py:69-132),
    columns scaled to unit l1 norm, as device CSR (by ray) and CSC (by pixel)
    arrays in fp64: {rptr, ridx, rval, cptr, cidx, cval, n_rays, n_pixels}.
    Raises the reference's DomainError for a pixel no ray crosses."""
    from .datasets import PetGeometry
    if not isinstance(geometry, PetGeometry):
        raise InputError("system_matrix_device needs a PetGeometry")
    torch = _lib.torch_mod()
    dev = backend.torch_device()
    side, nd = geometry.grid_side, geometry.n_detectors
    nr, npx = geometry.n_rays, geometry.n_pixels
    det = torch.from_numpy(np.ascontiguousarray(geometry.detector_positions())).to(dev)
    lines = torch.from_numpy(np.linspace(-1.0, 1.0, side + 1)).to(dev)
    cap = 2 * side + 3
    idx = torch.empty((nr, cap), dtype=torch.int32, device=dev)
    val = torch.empty((nr, cap), dtype=torch.float64, device=dev)
    cnt = torch.empty(nr, dtype=torch.int32, device=dev)
    _lib.call("mmk_pet_siddon", _lib.ptr(det), nd, side, _lib.ptr(lines), cap, _lib.ptr(idx),
              _lib.ptr(val), _lib.ptr(cnt), _lib.stream_handle(torch, dev))
    keep = torch.arange(cap, device=dev)[None, :] < cnt[:, None]
    ridx = idx[keep]
    rval = val[keep]
    rows = torch.arange(nr, device=dev, dtype=torch.int32)[:, None].expand(nr, cap)[keep]
    # canonical CSR: pixels ascending within each ray (rays emit in path order)
    key = rows.to(torch.int64) * npx + ridx.to(torch.int64)
    srt = torch.sort(key).indices
    ridx, rval, rows = ridx[srt], rval[srt], rows[srt]
    rptr = torch.zeros(nr + 1, dtype=torch.int64, device=dev)
    rptr[1:] = torch.cumsum(cnt.to(torch.int64), 0)
    order = torch.sort(ridx, stable=True).indices      # by pixel, ray order kept
    cidx = rows[order]
    cval = rval[order]
    ccnt = torch.bincount(ridx.to(torch.int64), minlength=npx)
    cptr = torch.zeros(npx + 1, dtype=torch.int64, device=dev)
    cptr[1:] = torch.cumsum(ccnt, 0)
    col = torch.zeros(npx, dtype=torch.float64, device=dev)
    col.index_add_(0, ridx.to(torch.int64), rval)
    empty = torch.nonzero(col == 0.0)
    if empty.numel():
        raise DomainError(f"pixel {int(empty[0, 0])} is intersected by no ray; its intensity "
                          "is unidentifiable (add detectors or shrink the grid)")
    rval = rval / col[ridx.to(torch.int64)]
    cval = cval / col[torch.repeat_interleave(torch.arange(npx, device=dev), ccnt)]
    i32 = torch.int32
    return {"rptr": rptr.to(i32), "ridx": ridx, "rval": rval, "cptr": cptr.to(i32),
            "cidx": cidx, "cval": cval, "n_rays": nr, "n_pixels": npx}


class SparsePetProblem:
    """A PET problem whose system matrix lives on the GPU in sparse form --
    built by ``system_matrix_device`` for geometries whose dense matrix would
    not fit host memory (a 256 x 256 image with 256 detectors is 32,640 x
    65,536: 17 GB dense in fp64, ~100 MB as CSR + CSC).  Same solver
    semantics as ``PetProblem`` (pet.py:213-285); counts y and the penalty
    lattice as there."""

    def __init__(self, sparse, y, mu, neighborhoods):
        self.sa = sparse
        self.y = y if A.is_torch(y) else np.asarray(y, dtype=np.float64)
        if tuple(A.shape_of(self.y)) != (sparse["n_rays"],):
            raise ShapeError(f"counts shape {tuple(A.shape_of(self.y))} does not match "
                             f"{sparse['n_rays']} rays")
        if A.min_value(self.y) < 0.0:
            raise DomainError("counts must be nonnegative")
        if mu < 0.0:
            raise DomainError(f"penalty constant must be >= 0, got {mu}")
        self.mu = float(mu)
        p = sparse["n_pixels"]
        if len(neighborhoods) != p:
            raise ShapeError(f"{len(neighborhoods)} neighborhoods for {p} pixels")
        indptr = np.zeros(p + 1, dtype=np.int64)
        indptr[1:] = np.cumsum([len(a) for a in neighborhoods])
        self.nbr_indptr = indptr
        self.nbr_indices = np.fromiter((k for a in neighborhoods for k in a), dtype=np.int64,
                                       count=int(indptr[-1]))
        self.e = None
        self._dev = {}

    @property
    def n_pixels(self):
        return self.sa["n_pixels"]

    @property
    def n_rays(self):
        return self.sa["n_rays"]

    def forward(self, lam):
        """E lam (fp64) on the device -- e.g. for simulating counts."""
        torch = _lib.torch_mod()
        sa = self.sa
        with torch.sparse.check_sparse_tensor_invariants():
            e = torch.sparse_csr_tensor(sa["rptr"].to(torch.int64), sa["ridx"].to(torch.int64),
                                        sa["rval"], (sa["n_rays"], sa["n_pixels"]))
        lam_t = lam if A.is_torch(lam) else torch.from_numpy(np.asarray(lam, dtype=np.float64))
        return (e @ lam_t.to(sa["rval"].device, torch.float64)[:, None])[:, 0]

    device_arrays = PetProblem.device_arrays


def _use_sparse(problem, backend):
    if isinstance(problem, SparsePetProblem):
        return True
    if backend.pet_kernel != "auto":
        return backend.pet_kernel == "sparse"
    if A.is_torch(problem.e):
        return False
    nnz = problem._dev.get("nnz")          # E is immutable: count its nonzeros once
    if nnz is None:
        nnz = problem._dev["nnz"] = int(np.count_nonzero(problem.e))
    return nnz < SPARSE_DENSITY * problem.e.size


def _sparse_arrays(e_rows, backend, torch):
    """CSR (by ray) and CSC (by pixel) of a host E block, on the device."""
    import scipy.sparse as sp
    dev, dt = backend.torch_device(), backend.torch_dtype()
    csr = sp.csr_matrix(e_rows)
    csc = csr.tocsc()
    if csr.nnz >= 2 ** 31:
        raise ShapeError("system matrix has too many nonzeros for int32 indices")

    def put(a, dtype):
        a = np.ascontiguousarray(a)
        if a.size == 0:
            a = np.zeros(1, dtype=a.dtype)
        return torch.from_numpy(a.astype(dtype)).to(dev)
    return {"rptr": put(csr.indptr, np.int32), "ridx": put(csr.indices, np.int32),
            "rval": put(csr.data, np.float64).to(dt), "cptr": put(csc.indptr, np.int32),
            "cidx": put(csc.indices, np.int32), "cval": put(csc.data, np.float64).to(dt)}


def _shard_device_sparse(sa, lo, hi, p, torch):
    """Rays [lo, hi) of a device-built system matrix, built on the device:
    the CSR rows (pointers rebased) and the CSC restricted to those rays (ray
    indices rebased to lo).  Boolean selection keeps every pixel's entries in
    ray order, so a shard's per-pixel sums run in the unsharded order."""
    dev = sa["rptr"].device
    rptr = sa["rptr"].to(torch.int64)
    a, b = int(rptr[lo]), int(rptr[hi])
    cidx = sa["cidx"].to(torch.int64)
    cptr = sa["cptr"].to(torch.int64)
    keep = (cidx >= lo) & (cidx < hi)
    col = torch.repeat_interleave(torch.arange(p, device=dev), cptr[1:] - cptr[:-1])
    cptr_s = torch.zeros(p + 1, dtype=torch.int64, device=dev)
    cptr_s[1:] = torch.cumsum(torch.bincount(col[keep], minlength=p), 0)

    def nonempty(t):
        return t if t.numel() else torch.zeros(1, dtype=t.dtype, device=dev)
    return {"rptr": (rptr[lo:hi + 1] - a).to(torch.int32),
            "ridx": nonempty(sa["ridx"][a:b]), "rval": nonempty(sa["rval"][a:b]),
            "cptr": cptr_s.to(torch.int32), "cidx": nonempty((cidx[keep] - lo).to(torch.int32)),
            "cval": nonempty(sa["cval"][keep])}


class _GpuPet(DeviceMm):
    direction = "maximize"

    def __init__(self, problem, backend, rows=None):
        super().__init__(backend)
        torch = self.torch
        self.problem = problem
        self.sparse = _use_sparse(problem, backend)
        lo, hi = rows if rows is not None else (0, problem.n_rays)   # ray shard
        if self.sparse:
            key = (str(backend.torch_device()), backend.dtype, "sparse", lo, hi)
            sa = problem._dev.get(key)
            if sa is None:
                if isinstance(problem, SparsePetProblem):
                    dt = backend.torch_dtype()
                    sa = {k: (v.to(dt) if k in ("rval", "cval") else v)
                          for k, v in problem.sa.items() if k in ("rptr", "ridx", "rval",
                                                                  "cptr", "cidx", "cval")}
                    if (lo, hi) != (0, problem.n_rays):
                        sa = _shard_device_sparse(sa, lo, hi, problem.n_pixels, torch)
                else:
                    e = problem.e if not A.is_torch(problem.e) else problem.e.cpu().numpy()
                    sa = _sparse_arrays(np.asarray(e, dtype=np.float64)[lo:hi], backend, torch)
                problem._dev[key] = sa
            self.sa = sa
        d = problem.device_arrays(backend, torch, dense=not self.sparse, rows=(lo, hi))
        self.e, self.y, self.ptr, self.idx = d["e"], d["y"], d["ptr"], d["idx"]
        self.d, self.p = hi - lo, problem.n_pixels
        self.mu = float(problem.mu)
        name = "mmk_pet_sparse_ws_bytes" if self.sparse else "mmk_pet_ws_bytes"
        self.ws = torch.zeros(_lib.ws_bytes(name, self.code, max(self.d, 1), self.p),
                              dtype=torch.uint8, device=self.device)
        self.red = torch.zeros(_lib.load().mmk_pet_reduce_len(self.p), dtype=torch.float64,
                               device=self.device)

    def device_state(self, lam):
        return A.to_device(lam, self.backend, self.torch)

    def _alloc_like(self, s):
        return self.torch.empty_like(s)

    def _copy_into(self, dst, src):
        dst.copy_(src)

    def _bytes_per_iter(self):
        if self.sparse:
            return float(2 * self.sa["rval"].numel() * (self.sa["rval"].element_size() + 4))
        return float(self.d * self.p * self.e.element_size())

    def _messages(self):
        return _MSG

    def _iterate(self, lam, out, f_ptr, err_ptr, flags=_lib.MMK_PET_UPDATE | _lib.MMK_PET_OBJECTIVE):
        if self.sparse:
            sa, P = self.sa, _lib.ptr
            _lib.call("mmk_pet_sparse_iter", self.code, P(sa["rptr"]), P(sa["ridx"]),
                      P(sa["rval"]), P(sa["cptr"]), P(sa["cidx"]), P(sa["cval"]), P(self.y),
                      P(lam), P(out), self.d, self.p, P(self.ptr), P(self.idx), self.mu, flags,
                      P(self.ws), self.ws.numel(), P(self.red), f_ptr, err_ptr, self.stream())
            return
        _lib.call("mmk_pet_iter", self.code, _lib.ptr(self.e), self.e.stride(0), _lib.ptr(self.y),
                  _lib.ptr(lam), _lib.ptr(out), self.d, self.p, _lib.ptr(self.ptr),
                  _lib.ptr(self.idx), self.mu, flags, _lib.ptr(self.ws), self.ws.numel(),
                  _lib.ptr(self.red), f_ptr, err_ptr, self.stream())

    def _engine_create(self, a, b, rule, trace, stamp, ctl, eng):
        self._keep = (a, b)
        if self.sparse:
            sa, P = self.sa, _lib.ptr
            _lib.call("mmk_pet_sparse_engine_create", self.code, P(sa["rptr"]), P(sa["ridx"]),
                      P(sa["rval"]), P(sa["cptr"]), P(sa["cidx"]), P(sa["cval"]), P(self.y),
                      P(a), P(b), self.d, self.p, P(self.ptr), P(self.idx), self.mu, P(self.ws),
                      self.ws.numel(), P(self.red), self.comm, ctypes.byref(rule), P(trace),
                      P(stamp), P(ctl), self.status.err_ptr, ctypes.byref(eng))
            return
        _lib.call("mmk_pet_engine_create", self.code, _lib.ptr(self.e), self.e.stride(0),
                  _lib.ptr(self.y), _lib.ptr(a), _lib.ptr(b), self.d, self.p, _lib.ptr(self.ptr),
                  _lib.ptr(self.idx), self.mu, _lib.ptr(self.ws), self.ws.numel(),
                  _lib.ptr(self.red), self.comm, ctypes.byref(rule), _lib.ptr(trace),
                  _lib.ptr(stamp), _lib.ptr(ctl), self.status.err_ptr, ctypes.byref(eng))

    def objective_only(self, lam):
        out = self.torch.empty_like(lam)
        self._iterate(lam, out, self.status.f_ptr, self.status.err_ptr, _lib.MMK_PET_OBJECTIVE)
        return self._check_error()

    def update_only(self, lam):
        out = self.torch.empty_like(lam)
        self._iterate(lam, out, self.status.f_ptr, self.status.err_ptr, _lib.MMK_PET_UPDATE)
        self._check_error()
        return out

    def surrogate(self, state, anchor):
        return pet_surrogate(state, anchor, self.problem)


def _check_lam(lam, problem):
    if tuple(A.shape_of(lam)) != (problem.n_pixels,):
        raise ShapeError(f"intensities shape {tuple(A.shape_of(lam))} does not match "
                         f"{problem.n_pixels} pixels")


def pet_penalized_objective(lam, problem, backend=SERIAL):
    """Loglikelihood minus (mu/2) * sum of squared adjacent differences."""
    _check_lam(lam, problem)
    mm = _GpuPet(problem, backend)
    return mm.objective_only(mm.device_state(lam))


def pet_loglik(lam, e, y, backend=SERIAL):
    """Poisson loglikelihood sum_i [y_i ln (E lam)_i - (E lam)_i]."""
    e_arr = e if A.is_torch(e) else np.asarray(e, dtype=np.float64)
    if len(A.shape_of(e_arr)) != 2 or A.shape_of(lam)[0] != e_arr.shape[1]:
        raise ShapeError("system matrix does not match intensities")
    prob = _LooseProblem(e_arr, y)
    mm = _GpuPet(prob, backend)
    return mm.objective_only(mm.device_state(lam))


class _LooseProblem:
    """Unvalidated (E, y) pair for pet_loglik, which the reference also
    accepts without the unit-column check (pet.py:318-323)."""

    def __init__(self, e, y):
        self.e = e
        self.y = y if A.is_torch(y) else np.asarray(y, dtype=np.float64)
        self.mu = 0.0
        self._dev = {}
        p = e.shape[1]
        self.nbr_indptr = np.zeros(p + 1, dtype=np.int64)
        self.nbr_indices = np.zeros(0, dtype=np.int64)

    device_arrays = PetProblem.device_arrays
    n_pixels = PetProblem.n_pixels
    n_rays = PetProblem.n_rays


def pet_update(lam, problem, backend=SERIAL, mean_counts=None):
    """One surrogate-maximization step from strictly positive intensities.
    ``mean_counts`` is accepted for signature compatibility; the device pass
    recomputes E @ lam as part of the same sweep over E."""
    _check_lam(lam, problem)
    lam_np = A.to_user(lam, np.empty(0)) if A.is_torch(lam) else np.asarray(lam, dtype=np.float64)
    if np.min(lam_np) <= 0.0:
        bad = int(np.argmin(lam_np))
        raise DomainError(f"intensities must be strictly positive; pixel {bad} is "
                          f"{lam_np[bad]!r}")
    mm = _GpuPet(problem, backend)
    return A.to_user(mm.update_only(mm.device_state(lam)), lam)


def pet_run(problem, config, backend=SERIAL):
    """Maximize the penalized loglikelihood from the flat start lam = 1."""
    mm = _GpuPet(problem, backend)
    like = problem.e
    state, trace = run_mm(mm, mm.device_state(np.ones(problem.n_pixels)), config)
    return A.to_user(state, like), trace


# ---------------------------------------------------------------------------
# host-side fp64 helpers for property tests (not on the iteration path)
def _host(a):
    return A.to_user(a, np.empty(0)) if A.is_torch(a) else np.asarray(a, dtype=np.float64)


def pet_penalized_gradient(lam, problem, backend=SERIAL):
    """Analytic gradient of the penalized objective (pet.py:349-360) on the
    device: the projection phase (dense or sparse) leaves b = E^T (y / E lam),
    then ``mmk_pet_gradient`` forms b - colsum - mu (deg lam - nbr)."""
    _check_lam(lam, problem)
    mm = _GpuPet(problem, backend)
    ld = mm.device_state(lam)
    st, P = mm.stream(), _lib.ptr
    if mm.sparse:
        sa = mm.sa
        _lib.call("mmk_pet_sparse_iter_a", mm.code, P(sa["rptr"]), P(sa["ridx"]), P(sa["rval"]),
                  P(sa["cptr"]), P(sa["cidx"]), P(sa["cval"]), P(mm.y), P(ld), mm.d, mm.p,
                  P(mm.ws), mm.ws.numel(), P(mm.red), mm.status.err_ptr, st)
    else:
        _lib.call("mmk_pet_iter_a", mm.code, P(mm.e), mm.e.stride(0), P(mm.y), P(ld), mm.d,
                  mm.p, P(mm.ws), mm.ws.numel(), P(mm.red), mm.status.err_ptr, st)
    grad = mm.torch.empty_like(ld)
    _lib.call("mmk_pet_gradient", mm.code, P(ld), P(grad), mm.p, P(mm.ptr), P(mm.idx), mm.mu,
              P(_col_sums_device(problem, mm)), P(mm.red), st)
    mm._check_error()
    return A.to_user(grad, lam)


def _col_sums_device(problem, mm):
    """Column sums of E in fp64 on the device (cached on the problem)."""
    key = (str(mm.device), "colsum")
    cs = problem._dev.get(key)
    if cs is None:
        torch = mm.torch
        if isinstance(problem, SparsePetProblem):
            sa = problem.sa
            cs = torch.zeros(problem.n_pixels, dtype=torch.float64, device=mm.device)
            cs.index_add_(0, sa["ridx"].to(mm.device).long(),
                          sa["rval"].to(device=mm.device, dtype=torch.float64))
        else:
            cs = torch.from_numpy(np.ascontiguousarray(problem.col_sums)).to(mm.device)
        problem._dev[key] = cs
    return cs


def pet_surrogate(lam, lam_n, problem):
    """Minorizing surrogate at (lam | lam_n): Jensen on each log plus the
    even-convex bound on each squared difference (host fp64)."""
    lam, lam_n, e, y = _host(lam), _host(lam_n), _host(problem.e), _host(problem.y)
    mean_n = e @ lam_n
    if np.any((y > 0.0) & (mean_n == 0.0)):
        raise NumericsError("anchor point has zero expected counts on a ray with positive counts")
    value = -float(e.sum(axis=0) @ lam)
    for i in np.flatnonzero(y > 0.0):
        wts = e[i] * lam_n / mean_n[i]
        m = wts > 0.0
        value += y[i] * float(wts[m] @ np.log(e[i, m] * lam[m] / wts[m]))
    if problem.mu > 0.0:
        lj, rk = problem.pair_left, problem.pair_right
        mid = lam_n[lj] + lam_n[rk]
        value -= 0.25 * problem.mu * float(np.sum((2.0 * lam[lj] - mid) ** 2 +
                                                  (2.0 * lam[rk] - mid) ** 2))
    return value
