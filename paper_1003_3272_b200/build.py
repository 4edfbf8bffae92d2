"""Build libmmk.so in-tree for sm_100a (nvcc, no JIT cache).

    python -m paper_1003_3272_b200.build            # incremental
    python -m paper_1003_3272_b200.build --force

Objects go to build/ (git-ignored); the shared library lands next to this
file so it travels with the source tree to the GPU box.
"""

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libmmk.so")
DIAG = os.path.join(PKG, "libmmk_diag.so")   # self-test + microbenchmarks (include/mmk_diag.h)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]
# tuning experiments only (e.g. MMK_NVCC_EXTRA="-DMMK_TC_XST=5"); empty by default
FLAGS += os.environ.get("MMK_NVCC_EXTRA", "").split()


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _diag_sources():
    return sorted(glob.glob(os.path.join(CSRC, "diag", "*.cu")))


def _deps():
    return _sources() + _diag_sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _up_to_date():
    if not (os.path.exists(LIB) and os.path.exists(DIAG)):
        return False
    t = min(os.path.getmtime(LIB), os.path.getmtime(DIAG))
    return all(os.path.getmtime(p) <= t for p in _deps())


def _compile(src):
    sub = "diag_" if os.path.basename(os.path.dirname(src)) == "diag" else ""
    obj = os.path.join(OBJ, sub + os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{proc.stderr}")
    return obj, proc.stderr


def build(force=False, verbose=False):
    """Compile every .cu under csrc/ and link libmmk.so (returns its path)."""
    if not force and _up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    srcs, dsrcs = _sources(), _diag_sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, srcs + dsrcs))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results[:len(srcs)]]
    subprocess.run([NVCC, *ARCH, "-shared", "-o", LIB, *objs], check=True)
    # the diagnostics library reuses the host helpers of mmk_abi.cu and tma_maps.cu
    dobjs = [o for o, _ in results[len(srcs):]] + [o for o in objs if o.endswith(("mmk_abi.o", "tma_maps.o"))]
    subprocess.run([NVCC, *ARCH, "-shared", "-o", DIAG, *dobjs], check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
