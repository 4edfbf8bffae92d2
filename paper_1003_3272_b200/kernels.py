"""Generic dense helpers with the reference's names (kernels.py:222-310).

The reference routes every product through these.  Here the solvers never
call them -- their products are fused inside the sm_100a kernels -- so these
exist only so that reference call sites (tests that build inputs with
``matmul(v, w)``, user scripts) keep working.  Products and sums run on the
GPU in fp64 through torch; ``elementwise`` applies the caller's numpy
closure, as in the reference.
"""

import numpy as np

from . import _arrays as A
from .backend import SERIAL, Backend
from .errors import ShapeError

__all__ = ["Backend", "matmul", "matvec", "tree_reduce_sum", "elementwise"]


def _dev(a, backend):
    import torch
    return A.to_device(a, Backend(backend.threads, "fp64", backend.device), torch)


def matmul(a, b, transpose_a=False, transpose_b=False, backend=SERIAL):
    """C = op(A) @ op(B) in fp64 on the device; numpy in -> numpy out."""
    sa, sb = A.shape_of(a), A.shape_of(b)
    if len(sa) != 2 or len(sb) != 2:
        raise ShapeError("matmul operands must be 2-D")
    ta = _dev(a, backend)
    tb = _dev(b, backend)
    ta = ta.T if transpose_a else ta
    tb = tb.T if transpose_b else tb
    if ta.shape[1] != tb.shape[0]:
        raise ShapeError(f"inner dimensions do not agree: {tuple(ta.shape)} x {tuple(tb.shape)}")
    return A.to_user(ta @ tb, a)


def matvec(a, x, transpose_a=False, backend=SERIAL):
    if len(A.shape_of(x)) != 1:
        raise ShapeError(f"x must be 1-D, got shape {A.shape_of(x)}")
    out = matmul(a, np.asarray(x, dtype=np.float64).reshape(-1, 1) if not A.is_torch(x)
                 else x.reshape(-1, 1), transpose_a=transpose_a, backend=backend)
    return out[:, 0]


def tree_reduce_sum(v, backend=SERIAL):
    t = _dev(v, backend).reshape(-1)
    return float(t.sum()) if t.numel() else 0.0


def elementwise(f, *arrays, backend=SERIAL):
    if not arrays:
        raise ShapeError("elementwise needs at least one array")
    arrs = tuple(np.asarray(x, dtype=np.float64) for x in arrays)
    if arrs[0].ndim < 1:
        raise ShapeError("elementwise operands must have at least 1 dimension")
    for k, x in enumerate(arrs[1:], start=1):
        if x.shape != arrs[0].shape:
            raise ShapeError(f"operand {k} has shape {x.shape}, expected {arrs[0].shape}")
    return np.asarray(f(*arrs), dtype=np.float64)
