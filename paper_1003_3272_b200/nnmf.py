"""Nonnegative matrix factorization, Frobenius loss, on the GPU.

Drop-in for the reference's Frobenius path (``pkg/src/mmkit/nnmf.py``):

  NnmfProblem      nnmf.py:40-64   same validation and overcomplete warning
  FactorPair       nnmf.py:67-72
  nnmf_objective   nnmf.py:75-81   ||X - VW||_F^2 (fp64 residual sum)
  nnmf_update_v    nnmf.py:84-96   V <- V * XW^T / (V W W^T + 1e-300)
  nnmf_update_w    nnmf.py:99-110  W <- W * V^T X / (V^T V W + 1e-300)
  nnmf_run         nnmf.py:170-177 uniform(0,1) start from default_rng(seed)
  _initial_factors nnmf.py:162-167 same PCG64 draw order

Poisson log fit (the first "next" row):

  nnmf_poisson_objective nnmf.py:193-209  sum x ln(VW) - VW, 0 ln 0 = 0
  nnmf_poisson_update    nnmf.py:212-242  joint square-root update (V, then W)
  nnmf_poisson_run       nnmf.py:262-265  maximize from the uniform(0,1) start

Every update and objective runs in libmmk.so (``csrc/nnmf.cu``,
``csrc/nnmf_tc.cu``, ``csrc/nnmf_poisson.cu``); one MM iteration is one fused
device pass (see ``_engine.DeviceMm``).  ``cbcl_preprocess`` is provided
host-side in ``datasets``.  ``nnmf_gradient`` / ``nnmf_surrogate`` are host-side fp64
property-test helpers, not part of the iteration.
"""

import ctypes
import warnings
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _arrays as A
from . import _lib
from ._engine import DeviceMm
from .backend import SERIAL
from .driver import run_mm
from .errors import DomainError, ShapeError

__all__ = ["NnmfProblem", "FactorPair", "nnmf_objective", "nnmf_update_v", "nnmf_update_w",
           "nnmf_run", "nnmf_gradient", "nnmf_surrogate", "nnmf_poisson_objective",
           "nnmf_poisson_update", "nnmf_poisson_run"]

DENOM_GUARD = 1e-300


def _require_nonneg(name, m):
    if A.min_value(m) < 0.0:
        raise DomainError(f"{name} must be entrywise nonnegative")


@dataclass(frozen=True)
class NnmfProblem:
    """Nonnegative data matrix X (numpy or a CUDA tensor) and target rank."""

    x: Any
    rank: int
    _dev: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        x = self.x
        if not A.is_torch(x):
            x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        if x.ndim != 2:
            raise ShapeError(f"data matrix must be 2-D, got shape {tuple(x.shape)}")
        if not A.all_finite(x):
            raise DomainError("data matrix contains non-finite entries")
        _require_nonneg("data matrix", x)
        if self.rank < 1:
            raise DomainError(f"rank must be >= 1, got {self.rank}")
        if self.rank > min(x.shape):
            warnings.warn(f"rank {self.rank} exceeds min(data shape) = {min(x.shape)}; "
                          "the factorization is overcomplete", stacklevel=2)
        object.__setattr__(self, "x", x)

    @property
    def shape(self):
        return tuple(self.x.shape)

    @classmethod
    def _unchecked(cls, x, rank):
        """A problem around already-validated data (single-op entry points)."""
        prob = cls.__new__(cls)
        object.__setattr__(prob, "x", x)
        object.__setattr__(prob, "rank", rank)
        object.__setattr__(prob, "_dev", {})
        return prob

    def device_x(self, backend, torch):
        key = (str(backend.torch_device()), backend.dtype)
        t = self._dev.get(key)
        if t is None:
            t = A.to_device(self.x, backend, torch)
            self._dev[key] = t
        return t


@dataclass(frozen=True)
class FactorPair:
    """Left (p x r) and right (r x q) nonnegative factors."""

    v: Any
    w: Any


class _GpuNnmf(DeviceMm):
    direction = "minimize"

    def __init__(self, problem, backend, x_dev=None):
        super().__init__(backend)
        torch = self.torch
        self.x = problem.device_x(backend, torch) if x_dev is None else x_dev
        self.m, self.n = self.x.shape
        self.r = problem.rank
        # everything but the pre-split copy of X is zeroed (mmk_nnmf_ws_clear):
        # at C4 that copy is 8.6 GB a zero fill would write for nothing
        self.ws = torch.empty(_lib.ws_bytes("mmk_nnmf_ws_bytes", self.code, self.m, self.n,
                                            self.r), dtype=torch.uint8, device=self.device)
        _lib.call("mmk_nnmf_ws_clear", self.code, self.m, self.n, self.r, _lib.ptr(self.ws),
                  self.ws.numel(), _lib.stream_handle(torch, self.device))
        self.red = torch.zeros(_lib.load().mmk_nnmf_reduce_len(self.n, self.r),
                               dtype=torch.float64, device=self.device)
        self._problem = problem

    # state helpers
    def device_state(self, s):
        t = self.torch
        return FactorPair(A.to_device(s.v, self.backend, t), A.to_device(s.w, self.backend, t))

    def _alloc_like(self, s):
        return FactorPair(self.torch.empty_like(s.v), self.torch.empty_like(s.w))

    def _copy_into(self, dst, src):
        dst.v.copy_(src.v)
        dst.w.copy_(src.w)

    def _bytes_per_iter(self):
        return 2.0 * self.m * self.n * self.x.element_size()

    def _messages(self):
        return {}

    def _iterate(self, s, out, f_ptr, err_ptr):
        _lib.call("mmk_nnmf_iter", self.code, _lib.ptr(self.x), self.x.stride(0),
                  _lib.ptr(s.v), _lib.ptr(s.w), _lib.ptr(out.v), _lib.ptr(out.w),
                  self.m, self.n, self.r, _lib.ptr(self.ws), self.ws.numel(), _lib.ptr(self.red),
                  f_ptr, err_ptr, self.stream())

    def _engine_create(self, a, b, rule, trace, stamp, ctl, eng):
        self._keep = (a, b)
        # the per-X preparation (tensor-core path) goes to the GPU first, so it
        # runs while the host captures and instantiates the engine's graph
        _lib.call("mmk_nnmf_prepare", self.code, _lib.ptr(self.x), self.x.stride(0), self.m,
                  self.n, self.r, _lib.ptr(self.ws), self.ws.numel(), self.stream())
        _lib.call("mmk_nnmf_engine_create", self.code, _lib.ptr(self.x), self.x.stride(0),
                  _lib.ptr(a.v), _lib.ptr(a.w), _lib.ptr(b.v), _lib.ptr(b.w), self.m, self.n,
                  self.r, _lib.ptr(self.ws), self.ws.numel(), _lib.ptr(self.red), self.comm,
                  ctypes.byref(rule), _lib.ptr(trace), _lib.ptr(stamp), _lib.ptr(ctl),
                  self.status.err_ptr, ctypes.byref(eng))

    def surrogate(self, state, anchor):
        return nnmf_surrogate(self._problem.x, state.v, state.w, anchor.v, anchor.w)


# ---------------------------------------------------------------------------
def _conform(x, v, w):
    xs, vs, ws = A.shape_of(x), A.shape_of(v), A.shape_of(w)
    if len(xs) != 2 or len(vs) != 2 or len(ws) != 2:
        raise ShapeError("x, v and w must all be 2-D")
    if vs[1] != ws[0]:
        raise ShapeError(f"inner dimensions do not agree: v is {vs[0]}x{vs[1]}, "
                         f"w is {ws[0]}x{ws[1]}")
    if (vs[0], ws[1]) != xs:
        raise ShapeError(f"data is {xs} but VW is {(vs[0], ws[1])}")
    return xs[0], xs[1], vs[1]


class _Ops:
    """Scratch for the single-operation entry points."""

    def __init__(self, backend, m, n, r):
        self.torch = _lib.torch_mod()
        torch = self.torch
        self.backend = backend
        self.dev = backend.torch_device()
        self.code = _lib.dtype_code(backend.torch_dtype())
        self.ws = torch.zeros(_lib.ws_bytes("mmk_nnmf_op_ws_bytes", self.code, m, n, r),
                              dtype=torch.uint8, device=self.dev)
        self.red = torch.zeros(_lib.load().mmk_nnmf_reduce_len(n, r), dtype=torch.float64,
                               device=self.dev)
        self.status = _lib.StatusBlock(torch, self.dev)
        self.status.clear_error()

    def stream(self):
        return _lib.stream_handle(self.torch, self.dev)

    def put(self, a):
        return A.to_device(a, self.backend, self.torch)


def nnmf_objective(x, v, w, backend=SERIAL):
    """Squared Frobenius error ||X - VW||_F^2 (fp64 accumulation)."""
    m, n, r = _conform(x, v, w)
    ops = _Ops(backend, m, n, r)
    xd, vd, wd = ops.put(x), ops.put(v), ops.put(w)
    _lib.call("mmk_nnmf_objective", ops.code, _lib.ptr(xd), xd.stride(0), _lib.ptr(vd),
              _lib.ptr(wd), m, n, r, _lib.ptr(ops.ws), ops.ws.numel(), ops.status.f_ptr,
              ops.status.err_ptr, ops.stream())
    return ops.status.read()[0]


def nnmf_update_v(x, v, w, backend=SERIAL):
    """v <- v * (X W^T) / (V W W^T + 1e-300)."""
    for name, mat in (("x", x), ("v", v), ("w", w)):
        _require_nonneg(name, mat)
    m, n, r = _conform(x, v, w)
    ops = _Ops(backend, m, n, r)
    xd, vd, wd = ops.put(x), ops.put(v), ops.put(w)
    out = ops.torch.empty_like(vd)
    _lib.call("mmk_nnmf_update_v", ops.code, _lib.ptr(xd), xd.stride(0), _lib.ptr(vd),
              _lib.ptr(wd), _lib.ptr(out), m, n, r, _lib.ptr(ops.ws), ops.ws.numel(),
              ops.status.err_ptr, ops.stream())
    return A.to_user(out, v)


def nnmf_update_w(x, v, w, backend=SERIAL):
    """w <- w * (V^T X) / (V^T V W + 1e-300)."""
    for name, mat in (("x", x), ("v", v), ("w", w)):
        _require_nonneg(name, mat)
    m, n, r = _conform(x, v, w)
    ops = _Ops(backend, m, n, r)
    xd, vd, wd = ops.put(x), ops.put(v), ops.put(w)
    out = ops.torch.empty_like(wd)
    _lib.call("mmk_nnmf_update_w", ops.code, _lib.ptr(xd), xd.stride(0), _lib.ptr(vd),
              _lib.ptr(wd), _lib.ptr(out), m, n, r, _lib.ptr(ops.ws), ops.ws.numel(),
              _lib.ptr(ops.red), ops.status.err_ptr, ops.stream())
    return A.to_user(out, w)


def _initial_factors(problem, seed):
    rng = np.random.default_rng(seed)
    p, q = problem.shape
    v0 = rng.random((p, problem.rank))
    w0 = rng.random((problem.rank, q))
    return FactorPair(v0, w0)


def nnmf_run(problem, config, backend=SERIAL, state0=None):
    """Factorize X under the Frobenius loss from a uniform(0,1) start drawn
    with ``config.seed`` (or from ``state0``).  Returns (FactorPair, MmTrace);
    factors come back as numpy arrays for a numpy X, device tensors for a
    tensor X."""
    start = _initial_factors(problem, config.seed) if state0 is None else state0
    mm = _GpuNnmf(problem, backend)
    state, trace = run_mm(mm, mm.device_state(start), config)
    return FactorPair(A.to_user(state.v, problem.x), A.to_user(state.w, problem.x)), trace


# ---------------------------------------------------------------------------
# Poisson log fit (nnmf.py:178-265)
def _poisson_messages(n):
    def at(text):
        return lambda idx: text
    return {1: at("zero reconstruction mean at a positive data entry"),
            2: at("reconstruction has zero mean where data is positive")}


class _GpuPoissonNnmf(_GpuNnmf):
    """``_PoissonNnmf`` (nnmf.py:245-259) on the device: objective(state)
    runs one fused pass giving f(state) and the next state."""

    direction = "maximize"

    def __init__(self, problem, backend, x_dev=None):
        DeviceMm.__init__(self, backend)
        torch = self.torch
        self.x = problem.device_x(backend, torch) if x_dev is None else x_dev
        self.m, self.n = self.x.shape
        self.r = problem.rank
        self.ws = torch.zeros(_lib.ws_bytes("mmk_nnmf_poisson_ws_bytes", self.code, self.m,
                                            self.n, self.r), dtype=torch.uint8,
                              device=self.device)
        self.red = torch.zeros(_lib.load().mmk_nnmf_poisson_reduce_len(self.n, self.r),
                               dtype=torch.float64, device=self.device)
        self._problem = problem

    def _messages(self):
        return _poisson_messages(self.n)

    def _iterate(self, s, out, f_ptr, err_ptr):
        _lib.call("mmk_nnmf_poisson_iter", self.code, _lib.ptr(self.x), self.x.stride(0),
                  _lib.ptr(s.v), _lib.ptr(s.w), _lib.ptr(out.v), _lib.ptr(out.w), self.m, self.n,
                  self.r, _lib.ptr(self.ws), self.ws.numel(), _lib.ptr(self.red), f_ptr, err_ptr,
                  self.stream())

    def _engine_create(self, a, b, rule, trace, stamp, ctl, eng):
        self._keep = (a, b)
        _lib.call("mmk_nnmf_poisson_engine_create", self.code, _lib.ptr(self.x),
                  self.x.stride(0), _lib.ptr(a.v), _lib.ptr(a.w), _lib.ptr(b.v), _lib.ptr(b.w),
                  self.m, self.n, self.r, _lib.ptr(self.ws), self.ws.numel(), _lib.ptr(self.red),
                  self.comm, ctypes.byref(rule), _lib.ptr(trace), _lib.ptr(stamp), _lib.ptr(ctl),
                  self.status.err_ptr, ctypes.byref(eng))

    def surrogate(self, state, anchor):
        raise NotImplementedError("the reference defines no Poisson surrogate")


def _poisson_pass(x, v, w, backend):
    """One fused device pass: (f(V, W), V', W') as device tensors."""
    m, n, r = _conform(x, v, w)
    mm = _GpuPoissonNnmf(NnmfProblem._unchecked(x, r), backend)
    s = mm.device_state(FactorPair(v, w))
    out = mm._alloc_like(s)
    mm._iterate(s, out, mm.status.f_ptr, mm.status.err_ptr)
    return mm._check_error(), out


def nnmf_poisson_objective(x, v, w, backend=SERIAL):
    """Poisson-model log fit: sum of x*ln(VW) - VW, with 0 ln 0 = 0."""
    f, _ = _poisson_pass(x, v, w, backend)
    return f


def nnmf_poisson_update(x, v, w, backend=SERIAL):
    """One joint square-root multiplicative update of (V, W): V first, then W
    against the recomputed reconstruction (nnmf.py:212-242)."""
    for name, mat in (("x", x), ("v", v), ("w", w)):
        _require_nonneg(name, mat)
    _, out = _poisson_pass(x, v, w, backend)
    return A.to_user(out.v, v), A.to_user(out.w, w)


def nnmf_poisson_run(problem, config, backend=SERIAL, state0=None):
    """Factorize under the Poisson log fit from a uniform(0,1) start drawn
    with ``config.seed`` (or from ``state0``); returns (FactorPair, MmTrace)."""
    start = _initial_factors(problem, config.seed) if state0 is None else state0
    mm = _GpuPoissonNnmf(problem, backend)
    state, trace = run_mm(mm, mm.device_state(start), config)
    return FactorPair(A.to_user(state.v, problem.x), A.to_user(state.w, problem.x)), trace


def nnmf_gradient(x, v, w, backend=SERIAL):
    """Gradient of ||X - VW||^2 with respect to (V, W) (nnmf.py:113-119):
    (2 (VW - X) W^T, 2 V^T (VW - X)), on the device (``mmk_nnmf_gradient``)."""
    m, n, r = _conform(x, v, w)
    ops = _Ops(backend, m, n, r)
    xd, vd, wd = ops.put(x), ops.put(v), ops.put(w)
    gv, gw = ops.torch.empty_like(vd), ops.torch.empty_like(wd)
    _lib.call("mmk_nnmf_gradient", ops.code, _lib.ptr(xd), xd.stride(0), _lib.ptr(vd),
              _lib.ptr(wd), _lib.ptr(gv), _lib.ptr(gw), m, n, r, _lib.ptr(ops.ws),
              ops.ws.numel(), _lib.ptr(ops.red), ops.status.err_ptr, ops.stream())
    return A.to_user(gv, v), A.to_user(gw, w)


# ---------------------------------------------------------------------------
# host-side fp64 helper for majorization property tests (not on the iteration path)
def nnmf_surrogate(x, v, w, v_n, w_n):
    """Separable majorizer of the Frobenius loss at anchor (v_n, w_n)."""
    x, v, w, v_n, w_n = (np.asarray(A.to_user(a, np.empty(0)) if A.is_torch(a) else a,
                                     dtype=np.float64) for a in (x, v, w, v_n, w_n))
    if np.min(v_n) <= 0.0 or np.min(w_n) <= 0.0:
        raise DomainError("surrogate anchor factors must be strictly positive")
    parts = v_n[:, :, None] * w_n[None, :, :]
    totals = parts.sum(axis=1)
    frac = parts / totals[:, None, :]
    scaled = (totals[:, None, :] / parts) * (v[:, :, None] * w[None, :, :])
    return float(np.sum(frac * (x[:, None, :] - scaled) ** 2))
