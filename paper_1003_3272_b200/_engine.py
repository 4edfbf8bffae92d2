"""Device-resident ``MmProblem`` base shared by the three solvers.

Two ways to drive a solver, identical results:

* **Per-iteration** (the reference protocol, ``driver.py:101-149``):
  ``objective(state)`` enqueues ONE fused iteration that evaluates f(state)
  *and* writes the next state, reads back one 24-byte status record (the
  objective plus the device error record), and caches the next state keyed
  by the identity of ``state``; ``step(state)`` returns that cached state.
  So ``run_mm`` costs one device pass and one device->host read per
  iteration (the pattern of the reference's ``_PetMm._means`` cache,
  ``pet.py:454-471``).
* **Fused** (``run_fused``, picked up by ``run_mm`` when the backend allows
  it): the whole loop runs on the device as one CUDA graph with conditional
  WHILE / IF nodes, two iterations per body on ping-pong state slots
  (``csrc/engine.cu``); the control kernels apply the same stopping rule,
  monotonicity slack and non-finite checks, and the host only drains the
  objective trace every ``batch`` iterations.
"""

import ctypes
import math
import time

import numpy as np

from . import _lib
from .driver import MmProblem, MmTrace
from .errors import MonotonicityError, NonFiniteError

CTL_IT, CTL_REASON, CTL_BATCH_START, CTL_FPREV, CTL_FCUR, CTL_REL, CTL_SLOT, CTL_LEN = (
    0, 1, 2, 3, 4, 5, 6, 16)
STOP_CONVERGED, STOP_CAP, STOP_NONFINITE, STOP_MONOTONE, STOP_DEVICE_ERROR = 1, 2, 3, 4, 5


class StopRule(ctypes.Structure):
    """mirrors ``mmk_stop_rule`` (include/mmk.h)"""
    _fields_ = [("epsilon", ctypes.c_double), ("monotone_tol", ctypes.c_double),
                ("sign", ctypes.c_double), ("max_iters", ctypes.c_int64),
                ("batch", ctypes.c_int64), ("check_monotone", ctypes.c_int32),
                ("pad_", ctypes.c_int32)]


def _as_f64(bits):
    return float(np.array([bits], dtype=np.int64).view(np.float64)[0])


class DeviceMm(MmProblem):
    """Subclasses implement ``_alloc_like``, ``_copy_into``, ``_iterate``,
    ``_engine_create``, ``_messages`` and ``_bytes_per_iter``."""

    comm = None   # NCCL communicator pointer for sharded runs

    def __init__(self, backend):
        self.backend = backend
        self.torch = _lib.torch_mod()
        self.device = backend.torch_device()
        self.dtype = backend.torch_dtype()
        self.code = _lib.dtype_code(self.dtype)
        self.status = _lib.StatusBlock(self.torch, self.device)
        self.status.clear_error()
        self._cache = None
        self.launches_per_iter = 0
        self._fused = bool(backend.fused)

    @property
    def run_fused(self):
        """The fused device loop when the backend allows it (``driver.run_mm``
        picks it up), else None.  A property, not an instance attribute holding
        the bound method: that would be a reference cycle keeping X and the
        workspace alive until the garbage collector happens to run."""
        return self._run_fused if self._fused else None

    # ---- plumbing -----------------------------------------------------------
    def stream(self):
        return _lib.stream_handle(self.torch, self.device)

    def _status_read(self):
        """(f, error code, error index) of the last pass (sharded solvers
        override it to agree on one record across ranks)."""
        return self.status.read()

    def _check_error(self):
        f, code, idx = self._status_read()
        _lib.raise_device_error(code, idx, self._messages())
        return f

    # ---- per-iteration protocol -----------------------------------------------
    def objective(self, state):
        """f(state); the same pass computes the next state, cached for step().
        An error only the update can raise (``_lib.update_only``) is held back
        with it: the reference raises it from step(), which it never calls
        from a converged or final state."""
        nxt = self._alloc_like(state)
        self._iterate(state, nxt, self.status.f_ptr, self.status.err_ptr)
        f, code, idx = self._status_read()
        pending = None
        if code != 0 and _lib.update_only(idx):
            pending = (code, idx)
            self.status.clear_error()
        else:
            _lib.raise_device_error(code, idx, self._messages())
        self._cache = (state, nxt, pending)
        return f

    def step(self, state):
        cached = self._cache
        if cached is not None and cached[0] is state:
            self._cache = None
            if cached[2] is not None:
                _lib.raise_device_error(*cached[2], self._messages())
            return cached[1]
        nxt = self._alloc_like(state)
        self._iterate(state, nxt, self.status.f_ptr, self.status.err_ptr)
        self._check_error()
        return nxt

    # ---- fused device loop ----------------------------------------------------
    def _batch(self, config):
        t_iter = self._bytes_per_iter() / 4.0e12 + 8e-6
        batch = int(min(4096, max(8, 0.05 / t_iter)))
        batch = int(min(batch, config.max_iters + 2))
        return batch + (batch & 1)            # even: pauses fall after the B -> A half

    def _run_fused(self, state0, config):
        torch = self.torch
        sign = 1.0 if self.direction == "maximize" else -1.0
        started = time.perf_counter()
        a = self._alloc_like(state0)
        b = self._alloc_like(state0)
        self._copy_into(a, state0)
        self._copy_into(b, state0)
        batch = self._batch(config)
        dev = self.device
        ctl = torch.zeros(CTL_LEN, dtype=torch.int64, device=dev)
        trace = torch.zeros(batch, dtype=torch.float64, device=dev)
        stamp = torch.zeros(batch, dtype=torch.int64, device=dev)
        ctl_h = torch.zeros(CTL_LEN, dtype=torch.int64, pin_memory=True)
        trace_h = torch.zeros(batch, dtype=torch.float64, pin_memory=True)
        stamp_h = torch.zeros(batch, dtype=torch.int64, pin_memory=True)
        rule = StopRule(config.epsilon, config.monotone_tol, sign, config.max_iters, batch,
                        1 if config.check_monotone else 0, 0)
        eng = ctypes.c_void_p()
        self._engine_create(a, b, rule, trace, stamp, ctl, eng)
        values, stamps = [], []
        try:
            bs = 0
            st = torch.cuda.current_stream(dev)
            while True:
                _lib.call("mmk_engine_run", eng, self.stream())
                ctl_h.copy_(ctl, non_blocking=True)
                trace_h.copy_(trace, non_blocking=True)
                stamp_h.copy_(stamp, non_blocking=True)
                st.synchronize()
                c = ctl_h.numpy()
                reason = int(c[CTL_REASON])
                count = int(c[CTL_IT]) - bs + 1 if reason else batch
                values.extend(trace_h.numpy()[:count].tolist())
                stamps.extend(stamp_h.numpy()[:count].tolist())
                if reason:
                    break
                bs = int(c[CTL_BATCH_START])
        finally:
            _lib.load().mmk_engine_destroy(eng)
        it = len(values) - 1
        if reason == STOP_DEVICE_ERROR:
            self._check_error()
        if reason == STOP_NONFINITE:
            if it == 0:
                raise NonFiniteError(
                    f"objective is non-finite at the initial point: {values[0]!r}")
            raise NonFiniteError(f"objective became non-finite at iteration {it}: {values[-1]!r}")
        if reason == STOP_MONOTONE:
            raise MonotonicityError(it, values[-2], values[-1], self.direction)
        final = b if int(c[CTL_SLOT]) == 1 else a
        ts = np.asarray(stamps, dtype=np.float64)
        trace_obj = MmTrace(
            objective_values=np.array(values),
            cumulative_seconds=(ts - ts[0]) * 1e-9,
            iters=it,
            converged=reason == STOP_CONVERGED,
            wall_time=time.perf_counter() - started,
            final_relative_change=_as_f64(c[CTL_REL]) if it > 0 else math.inf,
        )
        return final, trace_obj
