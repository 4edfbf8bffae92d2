"""The C-ABI library loads without a GPU and exports every entry point
include/mmk.h declares; ctypes signatures cover all of them."""

import os
import re

import pytest

from paper_1003_3272_b200 import _lib, build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "mmk.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mmk_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    path = B.build()
    assert os.path.exists(path)
    lib = _lib.load()
    assert lib.mmk_abi_version() == _lib.ABI_VERSION


def test_every_declared_symbol_is_exported_and_typed():
    lib = _lib.load()
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(declared) == _lib.exported_symbols()


def test_workspace_queries_are_host_only():
    lib = _lib.load()
    assert _lib.ws_bytes("mmk_nnmf_ws_bytes", 0, 2429, 361, 10) > 0
    assert _lib.ws_bytes("mmk_pet_ws_bytes", 0, 2016, 4096) > 0
    assert _lib.ws_bytes("mmk_mds_ws_bytes", 0, 401, 3, 401) > 0
    assert lib.mmk_nnmf_reduce_len(361, 10) == 3610 + 100 + 2   # [P | G | f | error flag]
    assert lib.mmk_pet_reduce_len(4096) == 4098   # [b | loglik | error flag]


def test_shape_errors_map_to_exceptions():
    from paper_1003_3272_b200.errors import ShapeError
    with pytest.raises(ShapeError):
        _lib.ws_bytes("mmk_nnmf_ws_bytes", 0, 10, 10, 0)


def test_sass_has_no_legacy_fallback_symbols():
    # the product library is CUDA-only: no host compute entry points
    lib = _lib.load()
    assert not hasattr(lib, "ora_matmul")


def test_nnmf_tc_workspace_policy():
    """Only a full-iteration fp32 workspace of rank 17..128 holds the
    tensor-core region (the pre-split copy of X: fp16 hi / lo, row-major, 4
    bytes per element), and only while that copy stays within 96 GiB; fp64,
    ranks <= 16 and the single operations (mmk_nnmf_op_ws_bytes) never
    reserve it (a zero-filled 16 GiB region per single-op call)."""
    ws = _lib.ws_bytes
    copy = 4 * 131072 * 16384
    c4 = ws("mmk_nnmf_ws_bytes", 0, 131072, 16384, 64)
    assert copy <= c4 < copy + (1 << 30)
    # ranks 17..63 run on the rank-64 kernels (zero-padded): same region
    assert copy <= ws("mmk_nnmf_ws_bytes", 0, 131072, 16384, 32) < copy + (1 << 30)
    for args in ((1, 131072, 16384, 64), (0, 131072, 16384, 16), (1, 131072, 16384, 128)):
        assert ws("mmk_nnmf_ws_bytes", *args) < (1 << 30)
    # ranks 65..128 run on the rank-128 kernels: the same copy plus the
    # rank-128 operands and the V step's Q rows (m x 256 fp32, 128 MiB here)
    for r in (65, 128):
        assert copy <= ws("mmk_nnmf_ws_bytes", 0, 131072, 16384, r) < copy + (1 << 30)
    assert ws("mmk_nnmf_op_ws_bytes", 0, 131072, 16384, 64) < (1 << 30)
    # 524288 x 65536: the copy would be 128 GiB -- SIMT path, no region
    assert ws("mmk_nnmf_ws_bytes", 0, 524288, 65536, 64) < (1 << 33)


def test_diagnostics_live_outside_the_solver_library():
    """The tcgen05 self-test and MMA microbenchmarks are in libmmk_diag.so
    (include/mmk_diag.h), not in the product library."""
    text = open(os.path.join(ROOT, "include", "mmk_diag.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    diag = sorted(set(re.findall(r"\b(mmk_[a-z0-9_]+)\s*\(", text)))
    assert diag and not set(diag) & set(header_functions())
    dl = _lib.load_diag()
    for name in diag:
        assert hasattr(dl, name), name
    lib = _lib.load()
    for name in diag + ["mmk_tc_set_trace"]:
        assert not hasattr(lib, name), name
