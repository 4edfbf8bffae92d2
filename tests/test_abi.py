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
    assert lib.mmk_nnmf_reduce_len(361, 10) == 3610 + 100 + 1
    assert lib.mmk_pet_reduce_len(4096) == 4097


def test_shape_errors_map_to_exceptions():
    from paper_1003_3272_b200.errors import ShapeError
    with pytest.raises(ShapeError):
        _lib.ws_bytes("mmk_nnmf_ws_bytes", 0, 10, 10, 0)


def test_sass_has_no_legacy_fallback_symbols():
    # the product library is CUDA-only: no host compute entry points
    lib = _lib.load()
    assert not hasattr(lib, "ora_matmul")


@pytest.mark.parametrize("env,presplit", [(None, True), ("0", False), ("1", True)])
def test_nnmf_tc_presplit_workspace_policy(env, presplit):
    """The tensor-core NNMF workspace holds the pre-split copy of X (fp16 hi / lo,
    row-major + transposed: 8 bytes per element) unless MMK_TC_PRESPLIT=0, and by
    default only while that copy stays within 48 GiB (read once per process,
    hence the subprocess)."""
    import subprocess
    import sys
    code = ("from paper_1003_3272_b200 import _lib\n"
            "print(_lib.ws_bytes('mmk_nnmf_ws_bytes', 0, 131072, 16384, 64),"
            " _lib.ws_bytes('mmk_nnmf_ws_bytes', 0, 262144, 65536, 64))")
    e = dict(os.environ)
    e.pop("MMK_TC_PRESPLIT", None)
    if env is not None:
        e["MMK_TC_PRESPLIT"] = env
    out = subprocess.run([sys.executable, "-c", code], env=e, cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    c4, big = (int(v) for v in out.stdout.split())
    copy = 8 * 131072 * 16384
    assert (c4 >= copy) == presplit and c4 < copy + (1 << 30)
    # 262144 x 65536: the copy would be 128 GiB -- only when forced
    assert (big >= 8 * 262144 * 65536) == (env == "1")
