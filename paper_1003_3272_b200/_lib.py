"""ctypes binding of libmmk.so (include/mmk.h) and the device plumbing the
solver modules share: dtype mapping, workspaces, the per-iteration status
read-back and the device error record -> exception translation.

There is deliberately no fallback: if the library or a GPU is missing every
solver entry point raises ``DeviceError``.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError, DomainError, NumericsError, raise_for_status

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libmmk.so")
# tcgen05 self-test and tuning microbenchmarks (include/mmk_diag.h): a separate
# library, not part of the solver ABI
DIAG_PATH = os.path.join(_PKG, "libmmk_diag.so")
ABI_VERSION = 1

MMK_F32, MMK_F64 = 0, 1
MMK_PET_UPDATE, MMK_PET_OBJECTIVE, MMK_PET_CHECK_POSITIVE = 1, 2, 4
MMK_MDS_UPDATE, MMK_MDS_OBJECTIVE, MMK_MDS_GRADIENT = 1, 2, 4
ERR_SITE_SHIFT = 48   # include/mmk.h: err index = site << 48 | offending index

_lock = threading.Lock()
_lib = None

_c = ctypes
_vp, _i64, _i32, _dbl, _sz = _c.c_void_p, _c.c_int64, _c.c_int, _c.c_double, _c.c_size_t
_SIGS = {
    "mmk_abi_version": ([], _i32),
    "mmk_last_error": ([], _c.c_char_p),
    "mmk_prof_enable": ([_i32], _i32),
    "mmk_prof_report": ([_c.c_char_p, _sz], _i32),
    "mmk_f64_to_f32": ([_vp, _vp, _i64, _vp], _i32),
    "mmk_nnmf_gradient": ([_i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp,
                           _vp, _vp], _i32),
    "mmk_pet_gradient": ([_i32, _vp, _vp, _i64, _vp, _vp, _dbl, _vp, _vp, _vp], _i32),
    "mmk_nnmf_ws_bytes": ([_i32, _i64, _i64, _i64, _c.POINTER(_sz)], _i32),
    "mmk_nnmf_op_ws_bytes": ([_i32, _i64, _i64, _i64, _c.POINTER(_sz)], _i32),
    "mmk_nnmf_ws_clear": ([_i32, _i64, _i64, _i64, _vp, _sz, _vp], _i32),
    "mmk_nnmf_prepare": ([_i32, _vp, _i64, _i64, _i64, _i64, _vp, _sz, _vp], _i32),
    "mmk_nnmf_reduce_len": ([_i64, _i64], _i64),
    "mmk_nnmf_iter_a": ([_i32, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp, _vp,
                         _vp], _i32),
    "mmk_nnmf_iter_b": ([_i32, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp], _i32),
    "mmk_nnmf_iter": ([_i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp, _vp,
                       _vp, _vp], _i32),
    "mmk_nnmf_objective": ([_i32, _vp, _i64, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp, _vp,
                            _vp], _i32),
    "mmk_nnmf_update_v": ([_i32, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp,
                           _vp], _i32),
    "mmk_nnmf_update_w": ([_i32, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp, _vp,
                           _vp], _i32),
    "mmk_nnmf_poisson_ws_bytes": ([_i32, _i64, _i64, _i64, _c.POINTER(_sz)], _i32),
    "mmk_nnmf_poisson_reduce_len": ([_i64, _i64], _i64),
    "mmk_nnmf_poisson_iter_a": ([_i32, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz, _vp,
                                 _vp, _vp], _i32),
    "mmk_nnmf_poisson_iter_b": ([_i32, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp], _i32),
    "mmk_nnmf_poisson_iter": ([_i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz,
                               _vp, _vp, _vp, _vp], _i32),
    "mmk_nnmf_poisson_engine_create": ([_i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                                        _vp, _sz, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "mmk_pet_ws_bytes": ([_i32, _i64, _i64, _c.POINTER(_sz)], _i32),
    "mmk_pet_reduce_len": ([_i64], _i64),
    "mmk_pet_iter_a": ([_i32, _vp, _i64, _vp, _vp, _i64, _i64, _vp, _sz, _vp, _vp, _vp], _i32),
    "mmk_pet_iter_b": ([_i32, _vp, _vp, _i64, _vp, _vp, _dbl, _i32, _vp, _vp, _sz, _vp, _vp,
                        _vp], _i32),
    "mmk_pet_iter": ([_i32, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _dbl, _i32, _vp, _sz,
                      _vp, _vp, _vp, _vp], _i32),
    "mmk_pet_sparse_ws_bytes": ([_i32, _i64, _i64, _c.POINTER(_sz)], _i32),
    "mmk_pet_sparse_iter_a": ([_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _sz,
                               _vp, _vp, _vp], _i32),
    "mmk_pet_sparse_iter": ([_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp,
                             _vp, _dbl, _i32, _vp, _sz, _vp, _vp, _vp, _vp], _i32),
    "mmk_pet_sparse_engine_create": ([_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                                      _i64, _vp, _vp, _dbl, _vp, _sz, _vp, _vp, _vp, _vp, _vp,
                                      _vp, _vp, _vp], _i32),
    "mmk_pet_siddon": ([_vp, _i32, _i32, _vp, _i32, _vp, _vp, _vp, _vp], _i32),
    "mmk_mds_ws_bytes": ([_i32, _i64, _i64, _i64, _c.POINTER(_sz)], _i32),
    "mmk_mds_iter": ([_i32, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i32,
                      _vp, _sz, _vp, _vp, _vp], _i32),
    "mmk_mds_unpack": ([_i32, _vp, _vp, _i64, _i64, _i64, _vp], _i32),
    "mmk_mds_votes_bytes": ([_i64, _i64, _c.POINTER(_sz)], _i32),
    "mmk_mds_votes_tri": ([_i32, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _sz, _vp, _vp], _i32),
    "mmk_mds_tri_ntiles": ([_i64], _i64),
    "mmk_mds_tri_reduce_len": ([_i64, _i64], _i64),
    "mmk_mds_tri_ws_bytes": ([_i64, _i64, _i64, _i64, _c.POINTER(_sz)], _i32),
    "mmk_mds_tri_pack": ([_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _vp], _i32),
    "mmk_mds_tri_iter_a": ([_vp, _i64, _i64, _vp, _i64, _i64, _vp, _sz, _vp, _vp, _vp], _i32),
    "mmk_mds_tri_iter_b": ([_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp], _i32),
    "mmk_mds_tri_iter": ([_vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _sz, _vp, _vp, _vp, _vp],
                         _i32),
    "mmk_mds_tri_engine_create": ([_vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _sz, _vp, _vp, _vp,
                                   _vp, _vp, _vp, _vp, _vp], _i32),
    "mmk_nccl_available": ([], _i32),
    "mmk_allreduce_f64": ([_vp, _i64, _vp, _vp], _i32),
    "mmk_allgather": ([_vp, _vp, _i64, _i32, _vp, _vp], _i32),
    "mmk_nnmf_engine_create": ([_i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _sz,
                                _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "mmk_pet_engine_create": ([_i32, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _dbl, _vp,
                               _sz, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "mmk_mds_engine_create": ([_i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                               _i64, _i64, _vp, _sz, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "mmk_engine_run": ([_vp, _vp], _i32),
    "mmk_engine_destroy": ([_vp], None),
}


_DIAG_SIGS = {
    "mmk_selftest_tc": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp], _i32),
    "mmk_tc_mma_bench": ([_i32, _i32, _vp, _vp], _i32),
    "mmk_tc_mma2_bench": ([_i32, _i32, _vp, _vp], _i32),
    "mmk_tc_pingpong": ([_i32, _vp, _vp], _i32),
}
_diag = None


def load_diag(path=DIAG_PATH):
    """The diagnostics library (self-test, MMA microbenchmarks)."""
    global _diag
    with _lock:
        if _diag is None:
            if not os.path.exists(path):
                raise DeviceError(f"{path} is missing; build it with "
                                  "`python -m paper_1003_3272_b200.build`")
            lib = ctypes.CDLL(path)
            for name, (args, res) in _DIAG_SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _diag = lib
        return _diag


def call_diag(name, *args):
    rc = getattr(load_diag(), name)(*args)
    if rc != 0:
        raise_for_status(rc, f"{name}: {load_diag().mmk_last_error().decode(errors='replace')}")


def exported_symbols():
    """Every entry point include/mmk.h declares (checked by the CPU tests)."""
    return sorted(_SIGS)


def load(path=LIB_PATH):
    """Load and type the library.  Needs no GPU (used by the CPU tests)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is missing; build it with `python -m paper_1003_3272_b200.build`")
        lib = ctypes.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.mmk_abi_version() != ABI_VERSION:
            raise DeviceError(f"libmmk ABI {lib.mmk_abi_version()} != expected {ABI_VERSION}")
        _lib = lib
        return lib


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise_for_status(rc, f"{name}: {lib.mmk_last_error().decode(errors='replace')}")


# ---------------------------------------------------------------------------
def torch_mod():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device is visible; the MM kernels run only on the GPU "
                          "(there is no CPU fallback)")
    load()
    return torch


def dtype_code(torch_dtype):
    import torch
    if torch_dtype == torch.float32:
        return MMK_F32
    if torch_dtype == torch.float64:
        return MMK_F64
    raise DeviceError(f"unsupported dtype {torch_dtype}")


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def stream_handle(torch, device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ws_bytes(name, *args):
    out = ctypes.c_size_t(0)
    call(name, *args, ctypes.byref(out))
    return out.value


class StatusBlock:
    """Device record [f (fp64 bits), err code, err index] plus its pinned
    host mirror; ``read()`` is the single device->host transfer of an
    iteration."""

    def __init__(self, torch, device):
        self.torch = torch
        self.dev = torch.zeros(3, dtype=torch.int64, device=device)
        self.host = torch.zeros(3, dtype=torch.int64, pin_memory=True)
        self.f_ptr = ctypes.c_void_p(self.dev.data_ptr())
        self.err_ptr = ctypes.c_void_p(self.dev.data_ptr() + 8)

    def clear_error(self):
        self.dev[1:].zero_()
        self.dev[2] = np.iinfo(np.int64).max

    def read(self):
        self.host.copy_(self.dev, non_blocking=True)
        self.torch.cuda.current_stream(self.dev.device).synchronize()
        raw = self.host.numpy()
        f = float(raw[:1].view(np.float64)[0])
        return f, int(raw[1]), int(raw[2])


def prof_report():
    """{kernel name: (launches, total_ms)} since the last report."""
    lib = load()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.mmk_prof_report(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split("\t")
        out[name] = (int(cnt), float(ms))
    return out


UPDATE_SITE = 16   # csrc/mmk_common.cuh kUpdateSite: sites 16..31 are update-only errors


def update_only(index):
    """True for an error the reference raises only from its update (step):
    MDS coincident pairs, PET negative discriminant / non-positive
    intensities, the Poisson update's zero mean."""
    return UPDATE_SITE <= (index >> ERR_SITE_SHIFT) < 2 * UPDATE_SITE


def split_site(index):
    """(site, offending index); update-only sites map to their base site."""
    site = index >> ERR_SITE_SHIFT
    if UPDATE_SITE <= site < 2 * UPDATE_SITE:
        site -= UPDATE_SITE
    return site, index & ((1 << ERR_SITE_SHIFT) - 1)


def raise_device_error(code, index, messages):
    """Map a device error record to the reference exception + message.
    ``messages`` maps site -> callable(idx) -> str."""
    if code == 0:
        return
    site, idx = split_site(index)
    text = messages.get(site, lambda i: f"device invariant violated at index {i}")(idx)
    cls = {2: DomainError, 3: NumericsError}.get(code, NumericsError)
    raise cls(text)
