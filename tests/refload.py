"""Load the read-only reference package as ``mmkit_ref`` (fixture generation
and CPU-side cross-checks only; /root/reference is absent on the GPU box).
Numba's cache and bytecode are redirected so nothing is written under
/root/reference."""

import importlib.util
import os
import sys
import tempfile

REF_SRC = "/root/reference/pkg/src/mmkit"


def available():
    return os.path.isdir(REF_SRC)


def load():
    if "mmkit_ref" in sys.modules:
        return sys.modules["mmkit_ref"]
    os.environ.setdefault("NUMBA_CACHE_DIR",
                          os.path.join(tempfile.gettempdir(), "mmk_numba_cache"))
    sys.dont_write_bytecode = True
    spec = importlib.util.spec_from_file_location(
        "mmkit_ref", os.path.join(REF_SRC, "__init__.py"),
        submodule_search_locations=[REF_SRC])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["mmkit_ref"] = mod
    spec.loader.exec_module(mod)
    return mod
