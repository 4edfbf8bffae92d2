"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py
from the reference itself) and the seeded input recipes they were made on."""

import hashlib
import os

import numpy as np

from paper_1003_3272_b200 import datasets as D

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(HERE, name + ".npz"))


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def c1_inputs():
    x = f32(np.random.default_rng(0).random((2429, 361)))
    g = np.random.default_rng(1)
    return x, f32(g.random((2429, 10))), f32(g.random((10, 361)))


def poisson_c1_inputs():
    """Count data of the CBCL shape, rank 10 (tests/golden/make_golden.py)."""
    x = np.floor(np.random.default_rng(21).random((2429, 361)) * 6.0)
    g = np.random.default_rng(22)
    return x, f32(g.random((2429, 10))), f32(g.random((10, 361)))


_C2 = {}


def c2_inputs():
    if not _C2:
        e = D.build_system_matrix(D.PetGeometry(64, 64))
        y = D.simulate_counts(D.default_phantom(64), e, 20260811)
        _C2.update(e=e, y=y, nbrs=D.build_neighborhoods(64))
    return _C2["e"], _C2["y"], _C2["nbrs"]


def c3_inputs(dim):
    diss = f32(D.votes_to_dissimilarity(D.synthetic_votes(401, 671, 0)))
    theta0 = f32(np.random.default_rng(1).uniform(-1.0, 1.0, size=(dim, 401)))
    return diss, theta0


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def rel_elem(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def _outer_sum(a, b):
    """a @ b as a fixed-order sum of outer products (BLAS summation order
    depends on the machine's thread count; this does not)."""
    out = np.zeros((a.shape[0], b.shape[1]))
    for k in range(a.shape[1]):
        out += np.outer(a[:, k], b[k])
    return out


def r64_inputs(kind):
    """Rank-64 tensor-core-eligible NNMF inputs (tests/golden/make_golden.py
    r64_inputs): 'uniform' or 'wellfit' (rank-64 product with 1 % noise,
    start within 20 % of the truth, ||X||^2 / f ~ 1e4)."""
    m, n, r = 1024, 2048, 64
    if kind == "uniform":
        g = np.random.default_rng(41)
        return f32(g.random((m, n))), f32(g.random((m, r))), f32(g.random((r, n)))
    g = np.random.default_rng(31)
    vt, wt = g.random((m, r)), g.random((r, n))
    x = f32(np.maximum(_outer_sum(vt, wt) * (1.0 + 0.01 * g.standard_normal((m, n))), 0.0))
    g2 = np.random.default_rng(32)
    return x, f32(vt * (1.0 + 0.2 * g2.random((m, r)))), f32(wt * (1.0 + 0.2 * g2.random((r, n))))
