"""Host/device array conversion for the drop-in API.

Reference functions take and return numpy float64 arrays.  The GPU solvers
accept numpy arrays or torch tensors; results come back in the caller's
container: numpy in -> numpy float64 out (exactly what reference callers
expect), torch in -> torch tensor on the device out (no host round trip, for
large problems that never leave HBM).
"""

import numpy as np


def is_torch(a):
    mod = type(a).__module__
    return mod.startswith("torch")


def to_device(a, backend, torch):
    """Contiguous tensor on the backend device with the backend dtype."""
    if is_torch(a):
        t = a.to(device=backend.torch_device(), dtype=backend.torch_dtype())
    else:
        arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        t = torch.from_numpy(arr).to(device=backend.torch_device(), dtype=backend.torch_dtype())
    return t.contiguous()


def to_user(t, like):
    """Return ``t`` in the container type of ``like``."""
    if is_torch(like):
        return t if like.device == t.device else t.to(like.device)
    return t.detach().to("cpu", dtype=__import__("torch").float64).numpy()


def shape_of(a):
    return tuple(a.shape) if hasattr(a, "shape") else np.shape(a)


def min_value(a):
    if is_torch(a):
        return float(a.min()) if a.numel() else np.inf
    a = np.asarray(a, dtype=np.float64)
    return float(np.min(a)) if a.size else np.inf


def all_finite(a):
    if is_torch(a):
        import torch
        return bool(torch.isfinite(a).all())
    return bool(np.all(np.isfinite(np.asarray(a, dtype=np.float64))))
