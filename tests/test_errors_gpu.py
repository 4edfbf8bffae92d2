"""Errors the reference raises only from its UPDATE (step), not while
evaluating the objective: MDS coupled coincident pairs (mds.py:105-111),
PET non-positive intensities and negative discriminants (pet.py:374-405),
the Poisson update's zero mean (nnmf.py:180-183).  A fused pass evaluates
f(state) and the update together; such an error must surface only when the
run actually steps from that state (csrc/mmk_common.cuh kUpdateSite, the
stopping rule mm_step, _engine.DeviceMm.objective/step)."""

import numpy as np
import pytest

import paper_1003_3272_b200 as M
from oracle import oracle as O
from paper_1003_3272_b200 import Backend, MmConfig
from paper_1003_3272_b200 import mds as MD

pytestmark = pytest.mark.gpu

PER_ITER = Backend(dtype="fp64", fused=False)


def _coincident_mds(n=9, p=2, seed=3):
    rng = np.random.default_rng(seed)
    y = rng.random((n, n))
    y = (y + y.T) / 2.0
    np.fill_diagonal(y, 0.0)
    theta = rng.uniform(-1.0, 1.0, size=(p, n))
    theta[:, 1] = theta[:, 0]          # objects 0 and 1 coincide, coupled (y01 > 0)
    return M.MdsProblem(weights=1.0 - np.eye(n), dissimilarities=y, p=p), theta


def test_mds_coincidence_raised_by_step_not_objective():
    prob, theta = _coincident_mds()
    mm = MD._make_mm(prob, PER_ITER)
    st = mm.device_state(theta)
    f = mm.objective(st)                          # the reference's stress() does not raise
    want = O.mds_stress(theta, O.MdsData(prob.weights, prob.dissimilarities, prob.p))
    assert abs(f - want) <= 1e-12 * abs(want)
    with pytest.raises(M.NumericsError, match="objects 0 and 1 coincide"):
        mm.step(st)
    # the device record was cleared when the error was held back: a valid
    # state evaluates and steps normally afterwards
    ok = theta.copy()
    ok[:, 1] += 0.25
    s2 = mm.device_state(ok)
    assert np.isfinite(mm.objective(s2))
    mm.step(s2)


def test_mds_coincidence_still_stops_a_run_that_steps():
    prob, theta = _coincident_mds()
    for be in (Backend(dtype="fp64"), PER_ITER):
        with pytest.raises(M.NumericsError, match="objects 0 and 1 coincide"):
            M.mds_run(prob, MmConfig(max_iters=5, epsilon=1e-300), be, theta0=theta)
