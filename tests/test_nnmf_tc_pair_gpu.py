"""CTA-pair (cta_group::2) form of the tensor-core V step (MMK_TC_PAIR=1,
csrc/nnmf_tc.cu nnmf_vstep_tc<true>): one iteration against fp64 on even and
odd tile counts (an odd count leaves the last pair's peer tile past m: its
TMA boxes are zero-filled and its rows are skipped), and a 30-iteration run
against the single-CTA form.  The switch is read once per process, so each
case runs in a subprocess."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

SNIPPET = r"""
import sys, torch
sys.path.insert(0, {here!r}); sys.path.insert(0, {root!r})
import test_nnmf_tc_gpu as T
import paper_1003_3272_b200 as M
m, n = {m}, {n}
g = torch.Generator(device="cuda").manual_seed(m + n)
x = torch.rand(m, n, device="cuda", generator=g)
v = torch.rand(m, 64, device="cuda", generator=g)
w = torch.rand(64, n, device="cuda", generator=g)
(vt, wt, ft), used = T.tc_launched(lambda: T.one_iter(x, v, w, force_simt=False))
assert used
vr, wr, fr = T.reference_iter(x, v, w)
rel = lambda a, b: float((a.double() - b).norm() / b.norm())
print("RESULT", abs(ft - fr) / fr, rel(vt, vr), rel(wt, wr))
import numpy as np
cfg = M.MmConfig(max_iters=30, epsilon=1e-300)
be = M.Backend(dtype="fp32")
st, tr = M.nnmf_run(M.NnmfProblem(x=x.cpu().numpy(), rank=64), cfg, be,
                    state0=M.FactorPair(v.cpu().numpy(), w.cpu().numpy()))
np.save({out!r}, np.asarray(tr.objective_values))
"""


def _run(pair, m, n, out):
    env = dict(os.environ, MMK_TC_PAIR="1" if pair else "0")
    code = SNIPPET.format(here=HERE, root=os.path.dirname(HERE), m=m, n=n, out=out)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT")][0]
    return [float(t) for t in line.split()[1:]]


@pytest.mark.parametrize("m,n", [(1024, 512), (4104, 392), (1160, 2176)])
def test_pair_vstep_matches_fp64_and_single_cta(m, n, tmp_path):
    import numpy as np
    fa, va, wa = _run(True, m, n, str(tmp_path / "pair.npy"))
    assert fa < 2e-6 and va < 3e-5 and wa < 3e-5, (fa, va, wa)
    _run(False, m, n, str(tmp_path / "single.npy"))
    tp, ts = np.load(tmp_path / "pair.npy"), np.load(tmp_path / "single.npy")
    assert np.all(np.diff(tp) <= 1e-6 * np.abs(tp[:-1]))
    assert np.max(np.abs(tp - ts) / ts) < 1e-5
