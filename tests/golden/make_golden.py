"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package (/root/reference/pkg/src/mmkit) in this container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [names...]

The fixtures pin both the CPU oracle (tests/test_oracle.py, bitwise) and the
CUDA path (tests/test_parity_gpu.py, 1e-9 fp64 / 1e-4 fp32).  Inputs are
regenerated from seeds by the tests (paper_1003_3272_b200.datasets /
numpy PCG64), so only outputs and input digests are stored.

Input recipes follow SURVEY.md section 8(d):
  C1 NNMF  X = default_rng(0).random((2429, 361)); V0, W0 from default_rng(1);
           all rounded to fp32 (so fp32 and fp64 GPU modes see the same data)
  C2 PET   E = build_system_matrix(PetGeometry(64, 64)) exact (fp64),
           y = simulate_counts(default_phantom(64), E, 20260811), lam0 = 1
  C3 MDS   Y = votes_to_dissimilarity(_synthetic_votes(401, 671, 0)) rounded
           to fp32, W = 1 - I, theta0 = default_rng(1).uniform(-1, 1,
           (dim, 401)) rounded to fp32
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import refload  # noqa: E402

R = refload.load()
THREADS = os.cpu_count() or 1


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def c1_inputs():
    x = f32(np.random.default_rng(0).random((2429, 361)))
    g = np.random.default_rng(1)
    v0 = f32(g.random((2429, 10)))
    w0 = f32(g.random((10, 361)))
    return x, v0, w0


def c2_inputs():
    e = R.build_system_matrix(R.PetGeometry(grid_side=64, n_detectors=64))
    y = R.simulate_counts(R.default_phantom(64), e, seed=20260811)
    return e, y, R.build_neighborhoods(64)


def c3_inputs(dim):
    import importlib
    cli = importlib.import_module("mmkit_ref.cli")
    diss = f32(R.votes_to_dissimilarity(cli._synthetic_votes(401, 671, 0)))
    theta0 = f32(np.random.default_rng(1).uniform(-1.0, 1.0, size=(dim, 401)))
    return diss, theta0


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)", flush=True)


def gen_nnmf_c1():
    x, v0, w0 = c1_inputs()
    problem = R.NnmfProblem(x=x, rank=10)
    import importlib
    nn = importlib.import_module("mmkit_ref.nnmf")
    mm = nn._FrobeniusNnmf(problem, R.Backend.parallel(THREADS))
    state, tr = R.run_mm(mm, nn.FactorPair(v0, w0), R.MmConfig(max_iters=1000, epsilon=1e-300))
    save("nnmf_c1", trace=tr.objective_values, v=state.v, w=state.w,
         x_digest=digest(x), v0_digest=digest(v0), w0_digest=digest(w0))


def gen_nnmf_small():
    rng = np.random.default_rng(11)
    x = rng.random((12, 9))
    problem = R.NnmfProblem(x=x, rank=3)
    state, tr = R.nnmf_run(problem, R.MmConfig(max_iters=25, seed=5))
    save("nnmf_small", x=x, trace=tr.objective_values, v=state.v, w=state.w)


def gen_pet_c2():
    e, y, nbrs = c2_inputs()
    out = {"e_digest": digest(e), "y": y}
    for mu in (0.0, 1e-7, 1e-6, 1e-5):
        problem = R.PetProblem(e=e, y=y, mu=mu, neighborhoods=nbrs)
        lam, tr = R.pet_run(problem, R.MmConfig(max_iters=1000, epsilon=1e-300),
                            backend=R.Backend.parallel(THREADS))
        out[f"trace_{mu:g}"] = tr.objective_values
        out[f"lam_{mu:g}"] = lam
    save("pet_c2", **out)


def gen_pet_c2_converge():
    e, y, nbrs = c2_inputs()
    problem = R.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=nbrs)
    lam, tr = R.pet_run(problem, R.MmConfig(), backend=R.Backend.parallel(THREADS))
    save("pet_c2_converge", trace=tr.objective_values, lam=lam,
         iters=np.array(tr.iters), converged=np.array(tr.converged))


def gen_pet_small():
    geo = R.PetGeometry(grid_side=5, n_detectors=8)
    e = R.build_system_matrix(geo)
    y = R.simulate_counts(R.default_phantom(5) + 0.5, e, seed=3)
    out = {"e": e, "y": y}
    for mu in (0.0, 1e-7, 1e-6, 1e-5):
        problem = R.PetProblem(e=e, y=y, mu=mu, neighborhoods=R.build_neighborhoods(5))
        lam, tr = R.pet_run(problem, R.MmConfig(max_iters=150))
        out[f"trace_{mu:g}"] = tr.objective_values
        out[f"lam_{mu:g}"] = lam
    save("pet_small", **out)


def gen_mds_c3():
    out = {}
    for dim in (2, 3, 4, 5, 10):
        diss, theta0 = c3_inputs(dim)
        problem = R.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=dim)
        import importlib
        md = importlib.import_module("mmkit_ref.mds")
        theta, tr = R.run_mm(md._MdsMm(problem, R.Backend.parallel(THREADS)), theta0,
                             R.MmConfig(max_iters=1000, epsilon=1e-300))
        out[f"trace_{dim}"] = tr.objective_values
        out[f"theta_{dim}"] = theta
        out["diss_digest"] = digest(diss)
    save("mds_c3", **out)


def gen_mds_small():
    rng = np.random.default_rng(10)
    q, p = 9, 3
    y = rng.random((q, q)) * 2.0
    y = (y + y.T) / 2.0
    np.fill_diagonal(y, 0.0)
    problem = R.MdsProblem(weights=np.ones((q, q)) - np.eye(q), dissimilarities=y, p=p)
    theta, tr = R.mds_run(problem, R.MmConfig(max_iters=40, seed=2))
    anchored, tr2 = R.mds_run(problem, R.MmConfig(max_iters=40, seed=2), anchor=True)
    save("mds_small", y=y, trace=tr.objective_values, theta=theta, anchored=anchored)


def poisson_c1_inputs():
    """Count data of the CBCL shape (2429 x 361), rank 10 start; fp32-exact."""
    x = np.floor(np.random.default_rng(21).random((2429, 361)) * 6.0)
    g = np.random.default_rng(22)
    return x, f32(g.random((2429, 10))), f32(g.random((10, 361)))


def gen_poisson_small():
    rng = np.random.default_rng(12)
    x = np.floor(rng.random((12, 9)) * 6.0)
    problem = R.NnmfProblem(x=x, rank=3)
    state, tr = R.nnmf_poisson_run(problem, R.MmConfig(max_iters=40, seed=4))
    save("poisson_small", x=x, trace=tr.objective_values, v=state.v, w=state.w)


def gen_poisson_c1():
    x, v0, w0 = poisson_c1_inputs()
    problem = R.NnmfProblem(x=x, rank=10)
    import importlib
    nn = importlib.import_module("mmkit_ref.nnmf")
    mm = nn._PoissonNnmf(problem, R.Backend.parallel(THREADS))
    state, tr = R.run_mm(mm, nn.FactorPair(v0, w0), R.MmConfig(max_iters=100, epsilon=1e-300))
    save("poisson_c1", trace=tr.objective_values, v=state.v, w=state.w,
         x_digest=digest(x), v0_digest=digest(v0), w0_digest=digest(w0))


def gen_gradients():
    """Analytic gradients (nnmf.py:113-119, pet.py:349-360, mds.py:147-167) at
    the config starts and at the 1000-iteration goldens (near-stationary)."""
    import importlib
    out = {}
    nn = importlib.import_module("mmkit_ref.nnmf")
    pt = importlib.import_module("mmkit_ref.pet")
    x, v0, w0 = c1_inputs()
    c1 = np.load(os.path.join(HERE, "nnmf_c1.npz"))
    for tag, (v, w) in (("start", (v0, w0)), ("it1000", (c1["v"], c1["w"]))):
        gv, gw = nn.nnmf_gradient(x, v, w, backend=R.Backend.parallel(THREADS))
        out[f"nnmf_gv_{tag}"], out[f"nnmf_gw_{tag}"] = gv, gw
    e, y, nbrs = c2_inputs()
    c2 = np.load(os.path.join(HERE, "pet_c2.npz"))
    for mu in (0.0, 1e-5):
        problem = R.PetProblem(e=e, y=y, mu=mu, neighborhoods=nbrs)
        for tag, lam in (("start", np.ones(4096)), ("it1000", c2[f"lam_{mu:g}"])):
            out[f"pet_g_{mu:g}_{tag}"] = pt.pet_penalized_gradient(
                lam, problem, backend=R.Backend.parallel(THREADS))
    md = importlib.import_module("mmkit_ref.mds")
    c3 = np.load(os.path.join(HERE, "mds_c3.npz"))
    diss, theta0 = c3_inputs(3)
    problem = R.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=3)
    for tag, th in (("start", theta0), ("it1000", c3["theta_3"])):
        out[f"mds_g_{tag}"] = md.stress_gradient(th, problem, backend=R.Backend.parallel(THREADS))
    save("gradients", **out)


def _outer_sum(a, b):
    """a @ b as a fixed-order sum of outer products (BLAS summation order
    depends on the machine's thread count; this does not)."""
    out = np.zeros((a.shape[0], b.shape[1]))
    for k in range(a.shape[1]):
        out += np.outer(a[:, k], b[k])
    return out


def r64_inputs(kind):
    """Rank-64 NNMF on a tensor-core-eligible shape (1024 x 2048: 8 row tiles,
    16 column blocks, 32 K-blocks of the tcgen05 kernels), fp32-exact.
    uniform : X, V0, W0 ~ U[0, 1) (SURVEY 8(d) C4 recipe at a reduced shape)
    wellfit : X = (Vt Wt)(1 + 0.01 N(0, 1)) clipped at 0, a rank-64 product
              with 1 % noise, started from Vt, Wt perturbed by up to 20 %:
              ||X||^2 / f ~ 1e4 over the run, the regime where the Gram-trace
              objective cancels."""
    m, n, r = 1024, 2048, 64
    if kind == "uniform":
        g = np.random.default_rng(41)
        return f32(g.random((m, n))), f32(g.random((m, r))), f32(g.random((r, n)))
    g = np.random.default_rng(31)
    vt, wt = g.random((m, r)), g.random((r, n))
    x = f32(np.maximum(_outer_sum(vt, wt) * (1.0 + 0.01 * g.standard_normal((m, n))), 0.0))
    g2 = np.random.default_rng(32)
    return x, f32(vt * (1.0 + 0.2 * g2.random((m, r)))), f32(wt * (1.0 + 0.2 * g2.random((r, n))))


def _gen_r64(kind, iters):
    import importlib
    nn = importlib.import_module("mmkit_ref.nnmf")
    x, v0, w0 = r64_inputs(kind)
    mm = nn._FrobeniusNnmf(R.NnmfProblem(x=x, rank=64), R.Backend.parallel(THREADS))
    state, tr = R.run_mm(mm, nn.FactorPair(v0, w0),
                         R.MmConfig(max_iters=iters, epsilon=1e-300))
    save(f"nnmf_r64_{kind}", trace=tr.objective_values, v=state.v, w=state.w,
         x_digest=digest(x), v0_digest=digest(v0), w0_digest=digest(w0))


def gen_nnmf_r64_uniform():
    _gen_r64("uniform", 500)


def gen_nnmf_r64_wellfit():
    _gen_r64("wellfit", 1000)


GENERATORS = {
    "nnmf_r64_uniform": gen_nnmf_r64_uniform, "nnmf_r64_wellfit": gen_nnmf_r64_wellfit,
    "gradients": gen_gradients,
    "poisson_small": gen_poisson_small, "poisson_c1": gen_poisson_c1,
    "nnmf_small": gen_nnmf_small, "pet_small": gen_pet_small, "mds_small": gen_mds_small,
    "mds_c3": gen_mds_c3, "pet_c2": gen_pet_c2, "nnmf_c1": gen_nnmf_c1,
    "pet_c2_converge": gen_pet_c2_converge,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(GENERATORS)
    for n in names:
        t = time.perf_counter()
        GENERATORS[n]()
        print(f"{n}: {time.perf_counter() - t:.1f}s", flush=True)
