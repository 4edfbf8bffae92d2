python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
cat > /tmp/pois_probe.py <<'PY'
import sys, time
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_1003_3272_b200 as M
import golden_io as G
x, v0, w0 = G.poisson_c1_inputs()
prob = M.NnmfProblem(x=x, rank=10)
be = M.Backend(dtype="fp32")
cfg = M.MmConfig(max_iters=1000, epsilon=1e-300, monotone_tol=1e-6)
M.nnmf_poisson_run(prob, cfg, be, state0=M.FactorPair(v0, w0))
torch.cuda.synchronize(); t = time.perf_counter()
_, tr = M.nnmf_poisson_run(prob, cfg, be, state0=M.FactorPair(v0, w0))
torch.cuda.synchronize(); print(f"poisson-c1: {1e6*(time.perf_counter()-t)/1000:.1f} us/iter")
PY
python /tmp/pois_probe.py; MMK_SMALL_ENGINE=0 python /tmp/pois_probe.py
