"""Host-side input construction: scanner geometry, phantom, counts, lattice
neighbourhoods, roll-call data and the synthetic matrices used by the
benchmarks.

None of this is on the per-iteration path (SURVEY.md section 2.1 rows 3-4:
"one-time input generation"); it exists so that the GPU solvers can be fed
the *same* inputs the reference builds, without the reference installed.
Each builder reproduces the reference's arithmetic so the arrays agree bit
for bit; ``tests/test_datasets.py`` checks that against the reference (when
present) and against committed digests.

Reference anchors:
  PetGeometry             pet.py:39-66
  build_system_matrix     pet.py:69-132 (Siddon chord lengths, unit columns)
  build_neighborhoods     pet.py:135-152
  simulate_counts         pet.py:155-170 (PCG64 Poisson, tree-summed means)
  default_phantom         pet.py:173-192
  votes_to_dissimilarity  mds.py:260-283
  synthetic_votes         cli.py:257-266
  cbcl_preprocess         nnmf.py:268-288
"""

import logging
import math
from dataclasses import dataclass

import numpy as np

from .errors import DomainError, InputError, ShapeError

log = logging.getLogger(__name__)

__all__ = ["PetGeometry", "build_system_matrix", "build_neighborhoods",
           "default_phantom", "simulate_counts", "votes_to_dissimilarity",
           "synthetic_votes", "cbcl_preprocess", "tree_row_sums", "distance_rows"]


# ---------------------------------------------------------------------------
def tree_row_sums(products):
    """Row sums of a 2-D array in the reference's pairwise-halving order
    (kernels.py:112-130 applied to every row at once, odd tail carried)."""
    buf = np.array(products, dtype=np.float64, copy=True)
    n = buf.shape[1]
    if n == 0:
        return np.zeros(buf.shape[0])
    while n > 1:
        half = n // 2
        nxt = buf[:, 0:2 * half:2] + buf[:, 1:2 * half:2]
        if n & 1:
            nxt = np.concatenate([nxt, buf[:, n - 1:n]], axis=1)
        buf = nxt
        n = buf.shape[1]
    return buf[:, 0].copy()


# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class PetGeometry:
    """Square grid of ``grid_side**2`` pixels inside [-1,1]^2, detectors on
    the circumscribed circle, one line of flight per unordered pair."""

    grid_side: int
    n_detectors: int

    def __post_init__(self):
        if self.grid_side < 1:
            raise InputError(f"grid_side must be >= 1, got {self.grid_side}")
        if self.n_detectors < 2:
            raise InputError(f"need at least 2 detectors, got {self.n_detectors}")

    @property
    def n_pixels(self):
        return self.grid_side ** 2

    @property
    def n_rays(self):
        return self.n_detectors * (self.n_detectors - 1) // 2

    def detector_positions(self):
        ang = 2.0 * np.pi * (np.arange(self.n_detectors) + 0.5) / self.n_detectors
        rad = math.sqrt(2.0)
        return np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1)


def _clip_interval(p0, d):
    """Parameter interval [lo, hi] of p0 + t*d inside the square, or None."""
    lo, hi = 0.0, 1.0
    for axis in (0, 1):
        s, dd = p0[axis], d[axis]
        if dd == 0.0:
            if s < -1.0 or s > 1.0:
                return None
            continue
        ta = (-1.0 - s) / dd
        tb = (1.0 - s) / dd
        lo = max(lo, min(ta, tb))
        hi = min(hi, max(ta, tb))
    return (lo, hi) if lo < hi else None


def _chord_row(p0, p1, side, grid_lines, row):
    d = (p1[0] - p0[0], p1[1] - p0[1])
    span = _clip_interval(p0, d)
    if span is None:
        return
    lo, hi = span
    length = math.hypot(d[0], d[1])
    knots = [np.array([lo, hi])]
    for axis in (0, 1):
        if d[axis] != 0.0:
            t = (grid_lines - p0[axis]) / d[axis]
            knots.append(t[(t > lo) & (t < hi)])
    t = np.unique(np.concatenate(knots))
    a, b = t[:-1], t[1:]
    keep = b > a
    a, b = a[keep], b[keep]
    mid = 0.5 * (a + b)
    h = 2.0 / side
    ix = np.minimum(((p0[0] + mid * d[0] + 1.0) / h).astype(np.int64), side - 1)
    iy = np.minimum(((1.0 - (p0[1] + mid * d[1])) / h).astype(np.int64), side - 1)
    np.add.at(row, iy * side + ix, (b - a) * length)


def build_system_matrix(geometry):
    """Dense ``n_rays x n_pixels`` chord-length matrix, columns scaled to unit
    l1 norm (pet.py:110-132).  Raises DomainError naming the first pixel no
    ray crosses."""
    det = geometry.detector_positions()
    side = geometry.grid_side
    grid_lines = np.linspace(-1.0, 1.0, side + 1)
    e = np.zeros((geometry.n_rays, geometry.n_pixels))
    ray = 0
    for i in range(geometry.n_detectors):
        for j in range(i + 1, geometry.n_detectors):
            _chord_row(det[i], det[j], side, grid_lines, e[ray])
            ray += 1
    col = e.sum(axis=0)
    empty = np.flatnonzero(col == 0.0)
    if empty.size:
        raise DomainError(
            f"pixel {empty[0]} is intersected by no ray; its intensity "
            "is unidentifiable (add detectors or shrink the grid)")
    return e / col


def build_neighborhoods(grid_side):
    """Sorted 4-neighbour lists of the row-major pixel lattice."""
    if grid_side < 1:
        raise InputError(f"grid_side must be >= 1, got {grid_side}")
    s = grid_side
    out = []
    for j in range(s * s):
        iy, ix = divmod(j, s)
        cand = []
        if iy > 0:
            cand.append(j - s)
        if ix > 0:
            cand.append(j - 1)
        if ix < s - 1:
            cand.append(j + 1)
        if iy < s - 1:
            cand.append(j + s)
        out.append(sorted(cand))
    return out


def default_phantom(grid_side):
    """Warm square (1) with a hot disk (4) and a cold disk (0)."""
    s = grid_side
    h = 2.0 / s
    iy, ix = np.divmod(np.arange(s * s), s)
    x = -1.0 + (ix + 0.5) * h
    y = 1.0 - (iy + 0.5) * h
    lam = np.ones(s * s)
    lam[(x + 0.25) ** 2 + (y + 0.2) ** 2 < 0.55 ** 2] = 4.0
    lam[(x - 0.35) ** 2 + (y - 0.35) ** 2 < 0.22 ** 2] = 0.0
    return lam


def simulate_counts(lambda_true, e, seed):
    """Seeded Poisson counts with means E @ lambda_true, the means summed in
    the reference's tree order so a seed gives the reference's dataset."""
    lam = np.asarray(lambda_true, dtype=np.float64)
    e = np.asarray(e, dtype=np.float64)
    if lam.ndim != 1 or e.ndim != 2 or e.shape[1] != lam.shape[0]:
        raise ShapeError(f"system matrix {e.shape} does not match intensities {lam.shape}")
    if np.min(lam) < 0.0:
        raise DomainError("true intensities must be nonnegative")
    means = tree_row_sums(e * lam[None, :])
    return np.random.default_rng(seed).poisson(means).astype(np.float64)


# ---------------------------------------------------------------------------
def votes_to_dissimilarity(votes):
    """Fraction of commonly attended roll calls on which two voters split."""
    v = np.asarray(votes, dtype=np.float64)
    if v.ndim != 2:
        raise ShapeError(f"vote matrix must be 2-D, got {v.shape}")
    if not np.all((v == 1.0) | (v == -1.0) | (v == 0.0)):
        raise DomainError("votes must be 1 (yea), -1 (nay) or 0 (absent)")
    att = (v != 0.0).astype(np.float64)
    shared = att @ att.T
    off = ~np.eye(v.shape[0], dtype=bool)
    miss = (shared == 0.0) & off
    if miss.any():
        i, j = (int(k[0]) for k in np.nonzero(miss))
        raise DomainError(
            f"voters {i} and {j} share no roll call; their dissimilarity is undefined")
    net = v @ v.T
    diss = (shared - net) / (2.0 * np.where(off, shared, 1.0))
    np.fill_diagonal(diss, 0.0)
    return diss


def synthetic_votes(q, m, seed):
    """Two-bloc yea/nay/absent matrix with the reference's RNG draw order."""
    rng = np.random.default_rng(seed)
    second_bloc = np.arange(q) >= q // 2
    line = rng.choice([-1.0, 1.0], size=m)
    votes = np.where(second_bloc[:, None], line[None, :], -line[None, :])
    votes = np.where(rng.random((q, m)) < 0.15, -votes, votes)
    votes[rng.random((q, m)) < 0.05] = 0.0
    return votes


def cbcl_preprocess(raw):
    """Rows rescaled to mean 0.25 / population std 0.25, clipped to [0, 1]."""
    raw = np.asarray(raw, dtype=np.float64)
    if raw.ndim != 2:
        raise ShapeError(f"expected a 2-D image matrix, got shape {raw.shape}")
    mu = raw.mean(axis=1)
    sd = raw.std(axis=1)
    flat = np.flatnonzero(sd == 0.0)
    if flat.size:
        raise DomainError(f"row {flat[0]} is constant; its scaling is undefined")
    scaled = (raw - mu[:, None]) / sd[:, None] * 0.25 + 0.25
    out = np.clip(scaled, 0.0, 1.0)
    frac = float(np.mean(out != scaled))
    if frac > 0.0:
        log.info("cbcl_preprocess clamped %.3f%% of entries into [0, 1]", 100.0 * frac)
    return out


# ---------------------------------------------------------------------------
def distance_rows(n, seed=0, latent_dim=10, noise=0.05, device="cuda"):
    """Device generator of large synthetic MDS dissimilarities (BASELINE
    config 5): latent points z ~ N(0, I_latent) (torch
    generator ``seed``), Y_ij = ||z_i - z_j|| (1 + noise * e_ij) with e_ij in
    [-1, 1) from an integer hash of the unordered pair (exactly symmetric),
    zero diagonal.  Returns ``rows(r0, r1)`` -> fp32 tensor of rows [r0, r1);
    nothing n x n is ever materialised at once (feed it to
    ``PackedMdsProblem.from_rows``).  The n = 65536 matrix does not fit a
    numpy PCG64 recipe in host memory, hence a device hash instead of
    ``default_rng(1)``."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    z = torch.randn(n, latent_dim, generator=g, device=device, dtype=torch.float32)
    jj = torch.arange(n, device=device, dtype=torch.int64)

    def rows(r0, r1):
        d = torch.cdist(z[r0:r1], z)
        ii = torch.arange(r0, r1, device=device, dtype=torch.int64)[:, None]
        lo, hi = torch.minimum(ii, jj), torch.maximum(ii, jj)
        h = (lo * 0x9E3779B1 + hi * 0x85EBCA77 + seed) & 0xFFFFFF
        e = h.to(torch.float32) / float(1 << 23) - 1.0
        y = d * (1.0 + noise * e)
        y[torch.arange(r1 - r0, device=device), torch.arange(r0, r1, device=device)] = 0.0
        return y
    return rows
