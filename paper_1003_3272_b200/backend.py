"""Execution target descriptor.

The reference's ``Backend`` (kernels.py:28-56) chose between a serial loop and
a thread pool, with bitwise-identical results either way.  Here the work
always runs on a CUDA device; ``Backend`` selects the device and the state
precision:

* ``dtype="fp64"`` (default) -- IEEE binary64 state and arithmetic, the
  reference's precision; parity target 1e-9 relative.
* ``dtype="fp32"`` -- binary32 state with fp64 objectives / cross-block sums;
  parity target 1e-4 relative (BASELINE.json north star).

``Backend.serial()`` / ``Backend.parallel(threads)`` and the ``threads``,
``is_parallel`` and ``mode`` members are kept so reference call sites run
unchanged; ``threads`` does not change the result (the kernels are
deterministic run to run) and is otherwise ignored.

``fused`` lets ``run_mm`` hand whole runs to the device engine (CUDA graphs,
stopping rule on the device; see ``_engine.py``).  ``fused=False`` keeps the
plain one-iteration-per-host-round-trip loop.

``mds_kernel`` picks the MDS pairwise kernel: ``"rows"`` (full-row tiling,
any weights, fp32/fp64), ``"tri"`` (packed upper triangle, unit weights,
fp32, p <= 3: every pair read once) or ``"auto"`` (tri from
``mds.TRI_MIN_POINTS`` points when it applies).

``pet_kernel`` picks the PET projector: ``"dense"`` (stream E), ``"sparse"``
(CSR/CSC of E's nonzeros) or ``"auto"`` (sparse when E is under
``pet.SPARSE_DENSITY`` nonzero -- the Siddon matrix is ~1 %).
"""

from dataclasses import dataclass
from typing import Optional

from .errors import ShapeError

__all__ = ["Backend", "SERIAL"]


@dataclass(frozen=True)
class Backend:
    threads: int = 1
    dtype: str = "fp64"
    device: Optional[int] = None
    fused: bool = True
    mds_kernel: str = "auto"
    pet_kernel: str = "auto"

    def __post_init__(self):
        if self.threads < 1:
            raise ShapeError(f"backend needs at least 1 thread, got {self.threads}")
        if self.dtype not in ("fp32", "fp64"):
            raise ShapeError(f"dtype must be 'fp32' or 'fp64', got {self.dtype!r}")
        if self.pet_kernel not in ("auto", "dense", "sparse"):
            raise ShapeError(f"pet_kernel must be 'auto', 'dense' or 'sparse', got "
                             f"{self.pet_kernel!r}")
        if self.mds_kernel not in ("auto", "rows", "tri"):
            raise ShapeError(f"mds_kernel must be 'auto', 'rows' or 'tri', got {self.mds_kernel!r}")

    @staticmethod
    def serial(dtype="fp64", device=None):
        return Backend(1, dtype, device)

    @staticmethod
    def parallel(threads, dtype="fp64", device=None):
        return Backend(threads, dtype, device)

    @staticmethod
    def fp32(device=None):
        return Backend(1, "fp32", device)

    @property
    def is_parallel(self):
        return self.threads > 1

    @property
    def mode(self):
        return "parallel" if self.is_parallel else "serial"

    # -- device helpers -----------------------------------------------------
    def torch_dtype(self):
        import torch
        return torch.float32 if self.dtype == "fp32" else torch.float64

    def torch_device(self):
        import torch
        idx = torch.cuda.current_device() if self.device is None else self.device
        return torch.device("cuda", idx)


SERIAL = Backend.serial()
