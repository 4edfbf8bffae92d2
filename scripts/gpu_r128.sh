timeout 900 python -m pytest tests/test_nnmf_tile_gpu.py tests/test_edge_gpu.py tests/test_parity_gpu.py -x -q 2>&1 | tail -2
python - <<'PY'
import torch, time, paper_1003_3272_b200 as M
from paper_1003_3272_b200 import _lib
for dt, tdt in (("fp32", torch.float32), ("fp64", torch.float64)):
    m, n, r = 65536, 16384, 128
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(m, n, device="cuda", generator=g, dtype=tdt)
    v0 = torch.rand(m, r, device="cuda", generator=g, dtype=tdt); w0 = torch.rand(r, n, device="cuda", generator=g, dtype=tdt)
    prob = M.NnmfProblem(x=x, rank=r)
    run = lambda k: M.nnmf_run(prob, M.MmConfig(max_iters=k, epsilon=1e-300), M.Backend(dtype=dt), state0=M.FactorPair(v0, w0))
    run(2); torch.cuda.synchronize()
    lib = _lib.load(); _lib.prof_report(); lib.mmk_prof_enable(1)
    st, tr = M.nnmf_run(prob, M.MmConfig(max_iters=3, epsilon=1e-300), M.Backend(dtype=dt, fused=False), state0=M.FactorPair(v0, w0))
    torch.cuda.synchronize(); lib.mmk_prof_enable(0)
    rep = _lib.prof_report()
    t0 = time.perf_counter(); run(10); torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(dt, "r=128 65536x16384: %.2f it/s" % (10 / t), {k: round(v[1] / v[0], 3) for k, v in rep.items() if "tile" in k})
PY
