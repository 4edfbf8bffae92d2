"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference solvers' per-iteration arithmetic
(``/root/reference/pkg/src/mmkit``), used as the parity checker for the CUDA
path and as the timed CPU baseline in ``bench.py``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this module; the product package never does.

The dense products and sums go through ``liboracle.so`` (``mmk_oracle.c``),
which reproduces the reference's tree-summation order bit for bit; the
element-wise maps are the same numpy expressions the reference evaluates.
The oracle is therefore expected to agree with the reference *bitwise*;
``tests/test_oracle.py`` pins that against golden vectors produced by the
reference itself (``tests/golden/make_golden.py``).

Every function cites the reference line it restates.
"""

import ctypes
import math
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

NNMF_DENOM_GUARD = 1e-300      # nnmf.py:32
PET_INTENSITY_FLOOR = 1e-300   # pet.py:36


class OracleError(Exception):
    """Raised where the reference raises; ``kind`` names the reference
    exception class (DomainError, NumericsError, ...)."""

    def __init__(self, kind, message):
        self.kind = kind
        super().__init__(message)


def build():
    """Compile liboracle.so from mmk_oracle.c (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        L.ora_matmul.argtypes = [dp, dp, dp, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.ora_matmul.restype = ctypes.c_int
        L.ora_tree_sum.argtypes = [dp, ctypes.c_int64]
        L.ora_tree_sum.restype = ctypes.c_double
        L.ora_max_threads.restype = ctypes.c_int
        _LIB = L
    return _LIB


def default_threads():
    return max(1, os.cpu_count() or 1)


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# --------------------------------------------------------------------------
# kernels.py restatement
def matmul(a, b, ta=False, tb=False, threads=1):
    """kernels.matmul (kernels.py:222-241) via the tree-summed C loops."""
    a = _f64(a)
    b = _f64(b)
    rows, inner = (a.shape[1], a.shape[0]) if ta else a.shape
    inner_b, cols = (b.shape[1], b.shape[0]) if tb else b.shape
    if inner != inner_b:
        raise OracleError("ShapeError", "inner dimensions do not agree")
    out = np.empty((rows, cols))
    lib().ora_matmul(_ptr(a), _ptr(b), _ptr(out), rows, inner, cols, int(ta),
                     int(tb), int(threads))
    return out


def matvec(a, x, ta=False, threads=1):
    """kernels.matvec (kernels.py:244-250)."""
    return matmul(a, _f64(x).reshape(-1, 1), ta=ta, threads=threads)[:, 0]


def tree_sum(v):
    """kernels.tree_reduce_sum (kernels.py:259-282); same order for any
    backend."""
    v = _f64(v).ravel()
    if v.size == 0:
        return 0.0
    return float(lib().ora_tree_sum(_ptr(v), v.size))


# --------------------------------------------------------------------------
# NNMF (Frobenius), nnmf.py
def _require_nonneg(name, m):                         # nnmf.py:35-37
    if np.min(m) < 0.0:
        raise OracleError("DomainError", f"{name} must be entrywise nonnegative")


def nnmf_objective(x, v, w, threads=1):               # nnmf.py:75-81
    recon = matmul(v, w, threads=threads)
    a = _f64(x)
    return tree_sum((a - recon) * (a - recon))


def nnmf_update_v(x, v, w, threads=1):                # nnmf.py:84-96
    for name, m in (("x", x), ("v", v), ("w", w)):
        _require_nonneg(name, m)
    numer = matmul(x, w, tb=True, threads=threads)
    recon = matmul(v, w, threads=threads)
    denom = matmul(recon, w, tb=True, threads=threads)
    return _f64(v) * (numer / (denom + NNMF_DENOM_GUARD))


def nnmf_update_w(x, v, w, threads=1):                # nnmf.py:99-110
    for name, m in (("x", x), ("v", v), ("w", w)):
        _require_nonneg(name, m)
    numer = matmul(v, x, ta=True, threads=threads)
    recon = matmul(v, w, threads=threads)
    denom = matmul(v, recon, ta=True, threads=threads)
    return _f64(w) * (numer / (denom + NNMF_DENOM_GUARD))


def nnmf_gradient(x, v, w, threads=1):                # nnmf.py:113-119
    recon = matmul(v, w, threads=threads)
    resid = recon - _f64(x)
    return (2.0 * matmul(resid, w, tb=True, threads=threads),
            2.0 * matmul(v, resid, ta=True, threads=threads))


def nnmf_step(x, v, w, threads=1):                    # nnmf.py:153-156
    v2 = nnmf_update_v(x, v, w, threads)
    return v2, nnmf_update_w(x, v2, w, threads)


# --------------------------------------------------------------------------
# NNMF (Poisson log fit), nnmf.py:178-265
def _masked_ratio(x, b):                              # nnmf.py:178-190
    if np.any((x > 0.0) & (b == 0.0)):
        raise OracleError("NumericsError",
                          "reconstruction has zero mean where data is positive")
    out = np.zeros_like(x)
    m = x > 0.0
    out[m] = x[m] / b[m]
    return out


def nnmf_poisson_objective(x, v, w, threads=1):       # nnmf.py:193-209
    b = matmul(v, w, threads=threads)
    x = _f64(x)
    if np.any((x > 0.0) & (b == 0.0)):
        raise OracleError("NumericsError", "zero reconstruction mean at a positive data entry")
    out = -b.copy()
    m = x > 0.0
    out[m] += x[m] * np.log(b[m])
    return tree_sum(out)


def nnmf_poisson_update(x, v, w, threads=1):          # nnmf.py:212-242
    for name, m in (("x", x), ("v", v), ("w", w)):
        _require_nonneg(name, m)
    x, v, w = _f64(x), _f64(v), _f64(w)
    p, q = x.shape
    b = matmul(v, w, threads=threads)
    ratio = _masked_ratio(x, b)
    numer_v = matmul(ratio, w, tb=True, threads=threads)
    w_sums = matvec(w, np.ones(q), threads=threads)
    v_next = v * np.sqrt(numer_v / (np.broadcast_to(w_sums, (p, len(w_sums))) +
                                    NNMF_DENOM_GUARD))
    b = matmul(v_next, w, threads=threads)
    ratio = _masked_ratio(x, b)
    numer_w = matmul(v_next, ratio, ta=True, threads=threads)
    v_sums = matvec(v_next, np.ones(p), ta=True, threads=threads)
    w_next = w * np.sqrt(numer_w / (np.broadcast_to(v_sums[:, None], (len(v_sums), q)) +
                                    NNMF_DENOM_GUARD))
    return v_next, w_next


# --------------------------------------------------------------------------
# PET, pet.py
class PetData:
    """The arrays ``PetProblem`` derives (pet.py:231-277)."""

    def __init__(self, e, y, mu, neighborhoods):
        self.e = _f64(e)
        self.y = _f64(y)
        self.mu = float(mu)
        self.degrees = np.array([float(len(a)) for a in neighborhoods])
        self.nbr_lists = [list(a) for a in neighborhoods]
        pairs = sorted({(min(j, k), max(j, k))
                        for j, a in enumerate(neighborhoods) for k in a})
        self.pair_left = np.array([a for a, _ in pairs], dtype=np.int64)
        self.pair_right = np.array([b for _, b in pairs], dtype=np.int64)

    @property
    def n_pixels(self):
        return self.e.shape[1]


def _pet_check_means(y, means):                       # pet.py:291-293, 305-306
    if np.any((y > 0.0) & (means == 0.0)):
        raise OracleError("NumericsError",
                          "a ray with positive counts has zero expected counts")


def pet_loglik_from_means(y, means):                  # pet.py:304-315
    _pet_check_means(y, means)
    out = -means.copy()
    m = y > 0.0
    out[m] += y[m] * np.log(means[m])
    return tree_sum(out)


def pet_penalty(lam, pd):                             # pet.py:326-331
    if pd.pair_left.size == 0:
        return 0.0
    d = lam[pd.pair_left] - lam[pd.pair_right]
    return tree_sum(d * d)


def pet_objective_from_means(lam, means, pd):         # pet.py:334-338
    value = pet_loglik_from_means(pd.y, means)
    if pd.mu > 0.0:
        value -= 0.5 * pd.mu * pet_penalty(lam, pd)
    return value


def pet_objective(lam, pd, threads=1):                # pet.py:341-346
    lam = _f64(lam)
    return pet_objective_from_means(lam, matvec(pd.e, lam, threads=threads), pd)


def pet_update(lam, pd, means=None, threads=1):       # pet.py:363-417
    lam = _f64(lam)
    if np.min(lam) <= 0.0:
        bad = int(np.argmin(lam))
        raise OracleError("DomainError",
                          f"intensities must be strictly positive; pixel {bad} is {lam[bad]!r}")
    if means is None:
        means = matvec(pd.e, lam, threads=threads)
    _pet_check_means(pd.y, means)
    ratio = np.zeros_like(pd.y)
    pos = pd.y > 0.0
    ratio[pos] = pd.y[pos] / means[pos]
    backproj = matvec(pd.e, ratio, ta=True, threads=threads)
    totals = lam * backproj
    if pd.mu == 0.0:
        return np.maximum(totals, PET_INTENSITY_FLOOR)
    nbr = np.array([sum_seq(lam, a) for a in pd.nbr_lists])
    mu = pd.mu
    a = -2.0 * mu * pd.degrees
    b = mu * (pd.degrees * lam + nbr) - 1.0
    disc = b * b - 4.0 * a * totals
    if np.any(disc < 0.0):
        raise OracleError("NumericsError", "negative discriminant")
    sq = np.sqrt(disc)
    neg = b < 0.0
    out = np.where(neg, 2.0 * totals / np.where(neg, sq - b, 1.0),
                   (-b - sq) / np.where(a < 0.0, 2.0 * a, -1.0))
    return np.maximum(out, PET_INTENSITY_FLOOR)


def sum_seq(lam, idx):                                # pet.py:204-210
    s = 0.0
    for k in idx:
        s += lam[k]
    return s


def pet_gradient(lam, pd, threads=1):                 # pet.py:349-360
    lam = _f64(lam)
    means = matvec(pd.e, lam, threads=threads)
    _pet_check_means(pd.y, means)
    ratio = np.zeros_like(pd.y)
    pos = pd.y > 0.0
    ratio[pos] = pd.y[pos] / means[pos]
    grad = matvec(pd.e, ratio, ta=True, threads=threads) - pd.e.sum(axis=0)
    if pd.mu > 0.0:
        nbr = np.array([sum_seq(lam, a) for a in pd.nbr_lists])
        grad -= pd.mu * (pd.degrees * lam - nbr)
    return grad


# --------------------------------------------------------------------------
# MDS, mds.py
class MdsData:
    """Arrays ``MdsProblem`` derives (mds.py:35-63)."""

    def __init__(self, weights, dissimilarities, dim):
        self.w = _f64(weights)
        self.y = _f64(dissimilarities)
        self.dim = int(dim)
        self.wy = self.w * self.y
        self.wsum = self.w.sum(axis=1)

    @property
    def n(self):
        return self.w.shape[0]


def _pair_d2(theta, threads=1):                       # mds.py:79-89
    gram = matmul(theta, theta, ta=True, threads=threads)
    diag = np.diag(gram).copy()
    return np.maximum(diag[:, None] + diag[None, :] - 2.0 * gram, 0.0)


def mds_stress(theta, md, threads=1):                 # mds.py:92-102
    d2 = _pair_d2(_f64(theta), threads)
    iu, ju = np.triu_indices(md.n, k=1)
    resid = md.y[iu, ju] - np.sqrt(d2[iu, ju])
    return tree_sum(md.w[iu, ju] * resid * resid)


def mds_update(theta, md, threads=1):                 # mds.py:114-144
    theta = _f64(theta)
    d2 = _pair_d2(theta, threads)
    coupling = md.wy * ~np.eye(md.n, dtype=bool)
    bad = np.nonzero((d2 <= 0.0) & (coupling > 0.0))
    if bad[0].size:
        raise OracleError("NumericsError",
                          f"objects {int(bad[0][0])} and {int(bad[1][0])} coincide")
    z = np.zeros_like(coupling)
    m = coupling > 0.0
    z[m] = coupling[m] / np.sqrt(d2[m])
    z_sums = matvec(z, np.ones(md.n), threads=threads)
    spread = matmul(theta, md.w - z, threads=threads)
    return (theta * (md.wsum + z_sums)[None, :] + spread) / (2.0 * md.wsum)[None, :]


def mds_stress_gradient(theta, md, threads=1):         # mds.py:147-167
    theta = _f64(theta)
    d2 = _pair_d2(theta, threads)
    w_off = md.w * ~np.eye(md.n, dtype=bool)
    bad = np.nonzero((d2 <= 0.0) & (w_off > 0.0))
    if bad[0].size:
        raise OracleError("NumericsError",
                          f"objects {int(bad[0][0])} and {int(bad[1][0])} coincide")
    coef = np.zeros_like(w_off)
    m = w_off > 0.0
    coef[m] = w_off[m] * (1.0 - md.y[m] / np.sqrt(d2[m]))
    row = matvec(coef, np.ones(md.n), threads=threads)
    pulled = matmul(theta, coef, threads=threads)
    return 2.0 * (theta * row[None, :] - pulled)


# --------------------------------------------------------------------------
# driver restatement (driver.py:101-149) for fixed-count parity runs
def run(objective, step, state0, direction, max_iters, epsilon=1e-300,
        monotone_tol=1e-12, check_monotone=True):
    """Returns (state, trace values ndarray, converged)."""
    sign = 1.0 if direction == "maximize" else -1.0
    f_prev = float(objective(state0))
    vals = [f_prev]
    state = state0
    converged = False
    for it in range(1, max_iters + 1):
        state = step(state)
        f_new = float(objective(state))
        if not math.isfinite(f_new):
            raise OracleError("NonFiniteError", f"non-finite at {it}")
        if check_monotone and sign * (f_new - f_prev) < -monotone_tol * (1.0 + abs(f_prev)):
            raise OracleError("MonotonicityError", f"iteration {it}")
        rel = abs(f_new - f_prev) / (abs(f_prev) + 1.0)
        vals.append(f_new)
        f_prev = f_new
        if rel < epsilon:
            converged = True
            break
    return state, np.array(vals), converged


def nnmf_run(x, v0, w0, max_iters, threads=1, **kw):
    """_FrobeniusNnmf under run_mm (nnmf.py:143-177) from a given start."""
    x = _f64(x)
    return run(lambda s: nnmf_objective(x, s[0], s[1], threads),
               lambda s: nnmf_step(x, s[0], s[1], threads),
               (_f64(v0), _f64(w0)), "minimize", max_iters, **kw)


def nnmf_poisson_run(x, v0, w0, max_iters, threads=1, **kw):
    """_PoissonNnmf under run_mm (nnmf.py:245-265) from a given start."""
    x = _f64(x)
    return run(lambda s: nnmf_poisson_objective(x, s[0], s[1], threads),
               lambda s: nnmf_poisson_update(x, s[0], s[1], threads),
               (_f64(v0), _f64(w0)), "maximize", max_iters, **kw)


def pet_run(pd, max_iters, threads=1, lam0=None, **kw):
    """_PetMm under run_mm from lam = 1 (pet.py:448-480), including the
    identity-keyed forward-projection cache."""
    cache = {}

    def means_of(lam):
        if cache.get("key") is lam:
            return cache["m"]
        m = matvec(pd.e, lam, threads=threads)
        cache["key"], cache["m"] = lam, m
        return m

    def objective(lam):
        return pet_objective_from_means(lam, means_of(lam), pd)

    def step(lam):
        return pet_update(lam, pd, means=means_of(lam), threads=threads)

    start = np.ones(pd.n_pixels) if lam0 is None else _f64(lam0)
    return run(objective, step, start, "maximize", max_iters, **kw)


def mds_run(md, theta0, max_iters, threads=1, **kw):
    """_MdsMm under run_mm (mds.py:228-257) from a given start."""
    return run(lambda t: mds_stress(t, md, threads),
               lambda t: mds_update(t, md, threads),
               _f64(theta0), "minimize", max_iters, **kw)


def timed(fn, *args, **kw):
    t0 = time.perf_counter()
    out = fn(*args, **kw)
    return out, time.perf_counter() - t0
