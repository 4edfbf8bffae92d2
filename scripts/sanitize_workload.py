"""Small invocations of every kernel family in libmmk.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; scripts/sanitize.sh).

  nnmf   SIMT (r = 10, fp32 + fp64), tensor cores (r = 64, fp32: pre-split X,
         V step with the residual pipeline, W step, split-K reduction),
         register-blocked tiles (fp64 r = 40 / 100, fp32 r = 72, Poisson
         r = 24), fp64 single ops in the reference's order, Poisson, the
         persistent small engine and the graph engine
  pet    dense and sparse projectors, device Siddon builder, persistent engine
  mds    rows kernel (fp32/fp64, weights), packed-triangle kernel (bulk-copy
         ring), votes -> packed tiles on the tensor cores
  mmx    fp64 -> fp32 narrowing
Each solver runs a few iterations per path; correctness is the test suite's
job -- this only has to execute every kernel.

    python scripts/sanitize_workload.py <nnmf|pet|mds|mmx|all> [graph|iter|both]

`iter` runs every solver through the per-iteration path (direct kernel
launches); `graph` through the device-loop engines (CUDA graphs with
conditional nodes, persistent cooperative kernels)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1003_3272_b200 as M  # noqa: E402
from paper_1003_3272_b200 import Backend, MmConfig  # noqa: E402
from paper_1003_3272_b200.mds import PackedMdsProblem  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main(which, paths):
    rng = np.random.default_rng(0)
    fused_modes = {"graph": (True,), "iter": (False,), "both": (True, False)}[paths]
    cfg = MmConfig(max_iters=4, epsilon=1e-300, monotone_tol=1e-6)
    if which in ("all", "nnmf"):
        x = f32(rng.random((300, 200)))
        for dt in ("fp32", "fp64"):
            for fused in fused_modes:
                M.nnmf_run(M.NnmfProblem(x=x, rank=10), cfg, Backend(dtype=dt, fused=fused),
                           state0=M.FactorPair(f32(rng.random((300, 10))),
                                               f32(rng.random((10, 200)))))
        xt = f32(rng.random((520, 392)))   # 5 row tiles (ragged), 7 K-blocks (ragged)
        st0 = M.FactorPair(f32(rng.random((520, 64))), f32(rng.random((64, 392))))
        for fused in fused_modes:
            M.nnmf_run(M.NnmfProblem(x=xt, rank=64), cfg, Backend(dtype="fp32", fused=fused),
                       state0=st0)
        # rank-128 tensor-core tile (one Q set copied out, vfinish_kernel, one
        # W-step block per item): r = 128 and r = 100 (zero-padded), ragged tiles
        for r in (128, 100):
            st1 = M.FactorPair(f32(rng.random((520, r))), f32(rng.random((r, 392))))
            for fused in fused_modes:
                M.nnmf_run(M.NnmfProblem(x=xt, rank=r), cfg, Backend(dtype="fp32", fused=fused),
                           state0=st1)
        xp = np.floor(rng.random((120, 90)) * 5)
        for fused in fused_modes:
            M.nnmf_poisson_run(M.NnmfProblem(x=xp, rank=4), cfg, Backend(dtype="fp32", fused=fused))
        # register-blocked tiles (round 2): fp64 r = 40 and r = 100 (DMMA), fp32 off
        # the tensor cores (ragged m, n), Poisson r = 24 and r = 100
        for dt, r in (("fp64", 40), ("fp64", 100), ("fp32", 72)):
            xr = f32(rng.random((131, 97)))
            for fused in fused_modes:
                M.nnmf_run(M.NnmfProblem(x=xr, rank=r), cfg, Backend(dtype=dt, fused=fused),
                           state0=M.FactorPair(f32(rng.random((131, r))), f32(rng.random((r, 97)))))
        for pr in (24, 100):
            for fused in fused_modes:
                M.nnmf_poisson_run(M.NnmfProblem(x=np.floor(rng.random((130, 70)) * 4), rank=pr),
                                   cfg, Backend(dtype="fp64", fused=fused))
        # fp64 single ops in the reference's order (nnmf_ref.cu)
        vv, ww = rng.random((300, 10)), rng.random((10, 200))
        M.nnmf_update_v(x, vv, ww, backend=Backend(dtype="fp64"))
        M.nnmf_update_w(x, vv, ww, backend=Backend(dtype="fp64"))
        M.nnmf_gradient(x, vv, ww, backend=Backend(dtype="fp64"))
        M.nnmf_update_v(x, f32(rng.random((300, 10))), f32(rng.random((10, 200))),
                        backend=Backend(dtype="fp32"))
        M.nnmf_objective(x, f32(rng.random((300, 10))), f32(rng.random((10, 200))),
                         backend=Backend(dtype="fp64"))
    if which in ("all", "pet"):
        geo = M.PetGeometry(8, 12)
        e = M.build_system_matrix(geo)
        y = M.simulate_counts(M.default_phantom(8) + 0.5, e, 3)
        nb = M.build_neighborhoods(8)
        for kern in ("dense", "sparse"):
            for fused in fused_modes:
                M.pet_run(M.PetProblem(e=e, y=y, mu=1e-3, neighborhoods=nb), cfg,
                          Backend(dtype="fp32", pet_kernel=kern, fused=fused))
        sa = M.system_matrix_device(M.PetGeometry(16, 24))
        ys = M.simulate_counts(M.default_phantom(16) + 0.5, M.build_system_matrix(
            M.PetGeometry(16, 24)), 4)
        for fused in fused_modes:
            M.pet_run(M.SparsePetProblem(sa, ys, 1e-4, M.build_neighborhoods(16)), cfg,
                      Backend(dtype="fp32", fused=fused))
    if which in ("all", "mds"):
        n = 150
        yy = rng.random((n, n))
        yy = f32((yy + yy.T) / 2.0)
        np.fill_diagonal(yy, 0.0)
        th0 = f32(rng.uniform(-1, 1, (3, n)))
        w = np.ones((n, n)) - np.eye(n)
        for dt in ("fp32", "fp64"):
            for fused in fused_modes:
                M.mds_run(M.MdsProblem(weights=w, dissimilarities=yy, p=3), cfg,
                          Backend(dtype=dt, mds_kernel="rows", fused=fused), theta0=th0)
        n2 = 300
        y2 = rng.random((n2, n2))
        y2 = f32((y2 + y2.T) / 2.0)
        np.fill_diagonal(y2, 0.0)
        for fused in fused_modes:
            M.mds_run(M.MdsProblem(weights=np.ones((n2, n2)) - np.eye(n2), dissimilarities=y2,
                                   p=3), cfg, Backend(dtype="fp32", mds_kernel="tri", fused=fused),
                      theta0=f32(rng.uniform(-1, 1, (3, n2))))
        votes = rng.choice([-1.0, 0.0, 1.0], size=(200, 64))
        PackedMdsProblem.from_votes(votes, p=3, backend=Backend(dtype="fp32"))
    if which in ("all", "mmx"):
        from paper_1003_3272_b200 import _lib
        src = torch.rand(1000, dtype=torch.float64, device="cuda")
        dst = torch.empty(1000, dtype=torch.float32, device="cuda")
        _lib.call("mmk_f64_to_f32", _lib.ptr(src), _lib.ptr(dst), 1000,
                  _lib.stream_handle(torch, src.device))
    torch.cuda.synchronize()
    print(f"sanitize workload '{which}' ({paths}) done")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all", sys.argv[2] if len(sys.argv) > 2 else "both")
