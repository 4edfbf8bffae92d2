#!/usr/bin/env python
"""MM iterations/sec on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload nnmf-large|mds-large|pet-large|nnmf-mid|nnmf-r128]

--gpus N > 1 without a torchrun environment re-launches this script under
torch.distributed.run with N ranks on this node (one per GPU; on a box with
fewer GPUs than N the ranks share devices over a gloo group -- a functional
check of the sharded path, not a throughput number).

A "step" is one MM iteration: the objective at the current state plus the
full update (one fused device pass).  Default workload = BASELINE config 4,
NNMF 131072 x 16384, rank 64, fp32 (the largest single-GPU config; X is
8.6 GB, larger than L2, so no flush is needed between steps).  Under
torchrun the rows of X are sharded across ranks (strong scaling of a fixed
problem, NCCL all-reduce of the W-step partials).

value    device-timed iterations/s of the whole job through the public API
         (nnmf_run / nnmf_run_sharded, mds_run / mds_run_sharded), inputs
         resident in HBM (CUDA events on the compute stream, max over ranks)
e2e      the same metric through the public API (nnmf_run on a pinned host
         tensor: H2D of X and the start, K iterations with per-batch trace
         reads, D2H of the factors) -- the headline against --impl reference
roofline dominant kernel (CUDA events on its own launches) vs
         MEASURED_PEAKS.json
cpu_baseline  the CPU oracle (oracle/, bit-exact restatement of the reference)
         on a bounded sample of the same workload, all host cores
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "nnmf-large": dict(solver="nnmf", m=131072, n=16384, r=64, label="BASELINE config 4"),
    "nnmf-r128": dict(solver="nnmf", m=131072, n=16384, r=128,
                      label="BASELINE config 4's X at rank 128 (the rank-128 tensor-core tile)"),
    "nnmf-mid": dict(solver="nnmf", m=16384, n=4096, r=64,
                     label="BASELINE config 4 at 1/32 of the size (CI of the sharded path)"),
    "mds-large": dict(solver="mds", n=65536, dim=3, label="BASELINE config 5"),
    "nnmf-c1": dict(solver="nnmf", m=2429, n=361, r=10, label="BASELINE config 1"),
    "poisson-c1": dict(solver="poisson", m=2429, n=361, r=10,
                       label="Poisson NNMF at the config-1 shape (SURVEY 8f)"),
    "pet-c2": dict(solver="pet", grid=64, detectors=64, mu=1e-5, label="BASELINE config 2"),
    "pet-large": dict(solver="pet", grid=256, detectors=256, mu=1e-6,
                      label="PET at a larger shape: 256x256 image, 256 detectors (32,640 rays), "
                            "device-built sparse system matrix"),
    "mds-c3": dict(solver="mds", n=401, dim=3, label="BASELINE config 3"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="nnmf-large", choices=sorted(WORKLOADS))
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a moment to start: the timed region begins once
            # it reports (a short region would otherwise go unsampled)
            t0 = time.perf_counter()
            while not self.samples and time.perf_counter() - t0 < 3.0:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        import statistics
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_info():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- CPU arm
def host_cpu():
    """lscpu model name, physical cores and logical CPUs of this host
    (state the core count the CPU number was taken on)."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        sockets = int(kv.get("Socket(s)", "1"))
        cores = int(kv.get("Core(s) per socket", "0"))
        info["physical_cores"] = sockets * cores or None
    except (OSError, ValueError, subprocess.SubprocessError):
        pass
    return info



def cpu_sample(workload, seconds):
    """Time the CPU oracle on a bounded sample of `workload`; returns the
    extrapolated full-size iterations/s plus a description."""
    import numpy as np
    from oracle import oracle as O
    threads = O.default_threads()
    W = WORKLOADS[workload]
    rng = np.random.default_rng(0)
    if W["solver"] == "nnmf":
        m, n, r = W["m"], W["n"], W["r"]
        rows = m
        if m * n * r > 5e8:
            rows = 256
        x = rng.random((rows, n), dtype=np.float32).astype(np.float64)
        v = rng.random((rows, r))
        w = rng.random((r, n))
        t0 = time.perf_counter()
        iters = 0
        while True:
            O.nnmf_objective(x, v, w, threads)
            v, w = O.nnmf_step(x, v, w, threads)
            iters += 1
            if time.perf_counter() - t0 > seconds or iters >= 50:
                break
        dt = (time.perf_counter() - t0) / iters
        scale = m / rows
        return 1.0 / (dt * scale), threads, (
            f"{iters} oracle MM iteration(s) (objective + V,W update) on {rows} of {m} rows "
            f"(n={n}, r={r}, fp64 tree-summed); per-iteration time scaled linearly in rows"
            if rows < m else f"{iters} oracle MM iterations at full size (fp64)")
    if W["solver"] == "poisson":
        x = np.floor(rng.random((W["m"], W["n"])) * 6.0)
        v = rng.random((W["m"], W["r"]))
        w = rng.random((W["r"], W["n"]))
        t0 = time.perf_counter()
        iters = 0
        while True:
            O.nnmf_poisson_objective(x, v, w, threads)
            v, w = O.nnmf_poisson_update(x, v, w, threads)
            iters += 1
            if time.perf_counter() - t0 > seconds or iters >= 50:
                break
        dt = (time.perf_counter() - t0) / iters
        return 1.0 / dt, threads, f"{iters} oracle Poisson MM iterations at full size (fp64)"
    if W["solver"] == "mds":
        n, dim = W["n"], W["dim"]
        ns = n if n <= 2048 else 1024
        y = rng.random((ns, ns))
        y = (y + y.T) / 2.0
        np.fill_diagonal(y, 0.0)
        md = O.MdsData(1.0 - np.eye(ns), y, dim)
        th = rng.uniform(-1, 1, size=(dim, ns))
        t0 = time.perf_counter()
        iters = 0
        while True:
            O.mds_stress(th, md, threads)
            th = O.mds_update(th, md, threads)
            iters += 1
            if time.perf_counter() - t0 > seconds or iters >= 50:
                break
        dt = (time.perf_counter() - t0) / iters
        scale = (n / ns) ** 2
        return 1.0 / (dt * scale), threads, (
            f"{iters} oracle MM iterations at n={ns}" +
            (f", scaled by (n/{ns})^2 to n={n}" if ns < n else ""))
    # pet (the dense oracle at the 64 x 64 paper shape, scaled by d * p for
    # larger geometries whose dense matrix does not fit host memory)
    from paper_1003_3272_b200 import datasets as D
    if W["grid"] > 64:
        v, thr, smp = cpu_sample("pet-c2", seconds)
        g2 = D.PetGeometry(W["grid"], W["detectors"])
        scale = (g2.n_rays * g2.n_pixels) / (2016.0 * 4096.0)
        return v / scale, thr, (f"{smp} at 64x64, scaled by d*p ({scale:.0f}x) to "
                                f"{W['grid']}x{W['grid']} (extrapolated: the dense oracle "
                                f"needs {g2.n_rays * g2.n_pixels * 8 / 1e9:.0f} GB)")
    e = D.build_system_matrix(D.PetGeometry(W["grid"], W["detectors"]))
    y = D.simulate_counts(D.default_phantom(W["grid"]), e, 20260811)
    pd = O.PetData(e, y, W["mu"], D.build_neighborhoods(W["grid"]))
    lam = np.ones(e.shape[1])
    t0 = time.perf_counter()
    iters = 0
    while True:
        m = O.matvec(pd.e, lam, threads=threads)
        O.pet_objective_from_means(lam, m, pd)
        lam = O.pet_update(lam, pd, means=m, threads=threads)
        iters += 1
        if time.perf_counter() - t0 > seconds or iters >= 200:
            break
    dt = (time.perf_counter() - t0) / iters
    return 1.0 / dt, threads, f"{iters} oracle MM iterations at full size (fp64)"


def run_reference(args):
    world, rank, _ = dist_info()
    if rank != 0:
        return
    W = WORKLOADS[args.workload]
    vals = []
    threads, sample = None, None
    for _ in range(max(1, args.warmup // 3)):
        cpu_sample(args.workload, min(args.cpu_seconds, 5.0))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, threads, sample = cpu_sample(args.workload, args.cpu_seconds / max(args.steps, 1))
        vals.append(v)
    elapsed = time.perf_counter() - t0
    value = sum(vals) / len(vals)
    line = {
        "impl": "reference", "metric": "MM iterations/sec", "value": value,
        "unit": "iterations/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, W, world),
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": threads,
                         "kind": "port", "sample": sample, "host": host_cpu()},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": elapsed,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, W, world=1):
    cfg = {"workload": args.workload, "what": W["label"]}
    cfg.update({k: v for k, v in W.items() if k not in ("solver", "label")})
    kind = {"mds": "tiles-sharded", "pet": "replicas"}.get(W["solver"], "rows-sharded")
    cfg["parallelism"] = f"{kind} x{world}" if world > 1 else "single-gpu"
    cfg["l2"] = ("inputs larger than L2" if args.workload in ("nnmf-large", "nnmf-r128",
                                                               "mds-large")
                 else "L2-resident (no flush: the solver re-reads a cache-sized matrix "
                      "every iteration by design)")
    return cfg


# ----------------------------------------------------------------------------- GPU arm
def bench_nnmf_large(args, torch, world, rank, dev):
    """BASELINE config 4: rows of X (and V) sharded across ranks, W
    replicated.  `value` times the public API on X resident in HBM --
    nnmf_run at one rank, nnmf_run_sharded (the device-loop engine with the
    NCCL all-reduce captured in its graph) across ranks; the per-kernel
    breakdown and the roofline come from a separate launch-profiled loop of
    the same iteration through the C ABI (phase A, all-reduce, phase B)."""
    import torch.distributed as dist

    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200.parallel import ShardedNnmf, nnmf_run_sharded, shard_rows
    W = WORKLOADS[args.workload]
    m, n, r = W["m"], W["n"], W["r"]
    lo, hi = shard_rows(m, world, rank)
    be = M.Backend(dtype=args.dtype, device=dev.index)
    dt = be.torch_dtype()
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    x = torch.rand(hi - lo, n, generator=g, device=dev, dtype=torch.float32).to(dt)
    g.manual_seed(7)
    w0 = torch.rand(r, n, generator=g, device=dev, dtype=torch.float32).to(dt)
    g.manual_seed(2000 + rank)
    v0 = torch.rand(hi - lo, r, generator=g, device=dev, dtype=torch.float32).to(dt)

    # 1) the public API (the headline value)
    group = dist.group.WORLD if world > 1 else None
    prob = M.NnmfProblem(x=x, rank=r)

    def api_run(iters):
        # (kernel timing experiments that disable parts of the objective turn
        # the descent check off; they never produce a bench number)
        cfg = M.MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6,
                         check_monotone="MMK_TC_EXP" not in os.environ)
        if world > 1:
            return nnmf_run_sharded(x, r, cfg, be, group=group, state0=(v0, w0))
        return M.nnmf_run(prob, cfg, be, state0=M.FactorPair(v0, w0))

    timing = time_region(args, torch, dev, lambda: api_run(args.warmup),
                         lambda: api_run(args.steps), world)

    # 2) launch-profiled per-iteration loop (kernel breakdown, roofline)
    sh = ShardedNnmf(x, v0.clone(), w0.clone(), r, be, group=group)
    loop = time_steps(args, torch, dev, lambda: sh.iterate(world), world)
    prof = loop["prof"]
    es = x.element_size()
    ml = hi - lo
    alg = {  # algorithmic HBM bytes per launch
        "nnmf_vstep": ml * n * es + 2 * ml * r * es + r * n * es,
        "nnmf_wpart": ml * n * es + ml * r * es,
        # X once (as X_hi + X_lo) + V read + V' written + V_h read + W_hi/W_lo chunks;
        # rank 128: the Q rows [q | q2] written instead of V' (nnmf_vfinish_tc
        # reads them and V, writes V')
        "nnmf_vstep_tc": (ml * n * 4 + 2 * ml * r * 4 + ml * r * 2 + 2 * r * n * 4 if r <= 64
                          else ml * n * 4 + ml * r * 4 + ml * r * 2 + 2 * r * n * 4 +
                          ml * 2 * r * 4),
        "nnmf_vfinish_tc": ml * 2 * r * 4 + 2 * ml * r * 4,
        # X once + V'_hi/V'_lo read + fp32 split-K partials written
        "nnmf_wstep_tc": ml * n * 4 + 2 * ml * r * 4,
        # CUDA-core tile kernels (ranks 17..64, fp64): algorithmic FLOPs --
        # Q = X W^T and the residual V W (2 x 2 m n r), P = V'^T X (2 m n r)
        "nnmf_vstep_tile": 4 * ml * n * r,
        "nnmf_wpart_tile": 2 * ml * n * r,
    }
    launches = sum(c for c, _ in prof.values()) // args.steps
    roof = roofline(prof, alg, "hbm", args.workload)
    e2e = None
    if not args.no_e2e and world == 1:
        e2e = nnmf_e2e(args, torch, be, x, v0, w0, r)
    kernels = {k: {"launches_per_step": c // args.steps, "avg_ms": ms / c}
               for k, (c, ms) in prof.items()}
    return timing, roof, launches, e2e, {
        "kernels": kernels, "kernel_loop_ms_per_step": loop["ms_total"] / args.steps,
        "value_path": sharded_path("nnmf", world) +
                      " on X resident in HBM; one timed run of `steps` iterations after a "
                      "`warmup`-iteration run"}


def sharded_path(name, world):
    """How the timed run is driven: the in-graph NCCL all-reduce when every
    rank has its own device, else (ranks sharing a device, gloo) run_mm's
    per-iteration protocol with a host all-reduce per iteration -- that line
    measures the protocol on one GPU, not the scaling."""
    import torch.distributed as dist
    if world == 1:
        return f"{name}_run (device-loop engine)"
    if dist.get_backend() == "nccl":
        return f"{name}_run_sharded (device-loop engine, NCCL all-reduce in its graph)"
    return (f"{name}_run_sharded (per-iteration protocol, gloo all-reduce on the host; "
            f"{world} ranks share one device)")


def nnmf_e2e(args, torch, be, x_dev, v0_dev, w0_dev, r):
    import paper_1003_3272_b200 as M
    xh = torch.empty(x_dev.shape, dtype=x_dev.dtype, pin_memory=True)
    xh.copy_(x_dev)
    vh = v0_dev.cpu().pin_memory()
    wh = w0_dev.cpu().pin_memory()
    prob = M.NnmfProblem(x=xh, rank=r)   # validation outside the timed region
    cfg = M.MmConfig(max_iters=args.steps, epsilon=1e-300, monotone_tol=1e-6)

    def run():
        prob._dev.clear()                   # no cached device copy: X is uploaded in the run
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st, tr = M.nnmf_run(prob, cfg, be, state0=M.FactorPair(vh, wh))
        torch.cuda.synchronize()
        return st, tr, time.perf_counter() - t0

    # one untimed warm-up run (first-touch of the caching allocators, host and
    # device), then the timed run -- the steady state of a serving process
    st, tr, dt0 = run()
    del st, tr
    st, tr, dt = run()
    K = tr.iters
    h2d = xh.numel() * xh.element_size() + vh.numel() * 4 + wh.numel() * 4
    d2h = (st.v.numel() + st.w.numel()) * st.v.element_size() + 8 * (K + 1)
    return {"value": K / dt, "unit": "iterations/s", "h2d_bytes_per_step": h2d // max(K, 1),
            "d2h_bytes_per_step": d2h // max(K, 1), "iters": K,
            "phases_ms": {"total": 1e3 * dt, "device_loop": 1e3 * tr.wall_time,
                          "upload_setup_readback": 1e3 * (dt - tr.wall_time),
                          "warmup_run_total": 1e3 * dt0},
            "path": "nnmf_run(NnmfProblem(pinned host X), fused device loop) -> host factors; "
                    "second of two runs (the first warms the allocators)"}


def bench_mds_large(args, torch, world, rank, dev):
    """BASELINE config 5: MDS n = 65536, dim 3, unit weights, packed upper
    triangle; tiles split evenly across ranks (one all-reduce of the
    per-point accumulators per iteration).  `value` times the public API
    (mds_run / mds_run_sharded) with the tiles resident in HBM; the kernel
    breakdown comes from a launch-profiled loop of the same iteration; `e2e`
    uploads the packed tiles from pinned host memory inside the timed run."""
    import torch.distributed as dist

    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import datasets as D
    from paper_1003_3272_b200.mds import PackedMdsProblem, _GpuMdsTri, tile_count
    from paper_1003_3272_b200.parallel import mds_run_sharded, tile_range
    W = WORKLOADS[args.workload]
    n, dim = W["n"], W["dim"]
    be = M.Backend(dtype="fp32", device=dev.index, mds_kernel="tri")
    nt = tile_count(n)
    t0, t1 = tile_range(nt, world, rank)
    prob = PackedMdsProblem.from_rows(D.distance_rows(n, seed=0), n, dim, be, tiles=(t0, t1))
    group = dist.group.WORLD if world > 1 else None
    g = torch.Generator(device=dev)
    g.manual_seed(2)
    th0 = torch.rand(dim, n, generator=g, device=dev) * 2 - 1

    def api_run(iters, problem=prob):
        cfg = M.MmConfig(max_iters=iters, epsilon=1e-300, monotone_tol=1e-6)
        if world > 1:
            return mds_run_sharded(problem, cfg, be, group=group, theta0=th0)
        return M.mds_run(problem, cfg, be, theta0=th0)

    timing = time_region(args, torch, dev, lambda: api_run(args.warmup),
                         lambda: api_run(args.steps), world)
    # launch-profiled loop (kernel breakdown, roofline)
    mm = _GpuMdsTri(prob, be, group=group)
    th = [th0.clone(), torch.empty_like(th0)]
    cur = [0]

    def step():
        a = cur[0]
        mm._iterate(th[a], th[1 - a], mm.status.f_ptr, mm.status.err_ptr)
        cur[0] = 1 - a

    prof = time_steps(args, torch, dev, step, world)["prof"]
    alg = {"mds_tri": (t1 - t0) * 128 * 128 * 4 + 2 * dim * n * 4}
    launches = sum(c for c, _ in prof.values()) // args.steps
    roof = roofline(prof, alg, "hbm", args.workload)
    kernels = {k: {"launches_per_step": c // args.steps, "avg_ms": ms / c}
               for k, (c, ms) in prof.items()}
    mm._check_error()
    e2e = None
    if not args.no_e2e and world == 1:
        host = torch.empty(prob.packed.numel(), dtype=torch.float32, pin_memory=True)
        host.copy_(prob.packed)
        del mm, th

        def run():
            torch.cuda.synchronize()
            t_0 = time.perf_counter()
            p2 = PackedMdsProblem.from_packed(host, n, dim, be, tiles=(t0, t1))
            cfg = M.MmConfig(max_iters=args.steps, epsilon=1e-300, monotone_tol=1e-6)
            th_out, tr = M.mds_run(p2, cfg, be, theta0=th0.cpu().numpy())
            th_h = th_out.cpu() if hasattr(th_out, "cpu") else th_out
            torch.cuda.synchronize()
            return tr, th_h, time.perf_counter() - t_0

        run()
        tr, th_h, dt = run()
        K = tr.iters
        h2d = host.numel() * 4 + dim * n * 8
        d2h = dim * n * 8 + 8 * (K + 1)
        e2e = {"value": K / dt, "unit": "iterations/s", "h2d_bytes_per_step": h2d // max(K, 1),
               "d2h_bytes_per_step": d2h // max(K, 1), "iters": K,
               "phases_ms": {"total": 1e3 * dt, "device_loop": 1e3 * tr.wall_time,
                             "upload_setup_readback": 1e3 * (dt - tr.wall_time)},
               "path": "PackedMdsProblem.from_packed(pinned host tiles) + mds_run(host theta0) "
                       "-> host theta; second of two runs"}
    return timing, roof, launches, e2e, {
        "kernels": kernels,
        "value_path": sharded_path("mds", world) +
                      " on the packed tiles resident in HBM",
        "data": "synthetic (Y_ij = ||z_i - z_j||(1 + 0.05 e_ij), z ~ N(0, I_10), e from a "
                "symmetric pair hash; theta0 uniform[-1,1]; datasets.distance_rows)"}


def bench_pet_large(args, torch, world, rank, dev):
    """PET at a larger shape: device-built Siddon matrix (CSR + CSC), counts
    simulated from the default phantom, penalized MM in fp32.  Replicas only
    across GPUs (the exchange is an all-reduce of the p-vector)."""
    import numpy as np
    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import _lib
    from paper_1003_3272_b200.pet import _GpuPet
    W = WORKLOADS[args.workload]
    geo = M.PetGeometry(W["grid"], W["detectors"])
    be = M.Backend(dtype="fp32", device=dev.index)
    sa = M.system_matrix_device(geo, be)
    nb = M.build_neighborhoods(W["grid"])
    lam_true = torch.from_numpy(M.default_phantom(W["grid"])).to(dev)
    means = M.SparsePetProblem(sa, np.zeros(geo.n_rays), 0.0, nb).forward(lam_true)
    g = torch.Generator(device=dev)
    g.manual_seed(20260811)
    y = torch.poisson(means * 50.0, generator=g)
    prob = M.SparsePetProblem(sa, y, W["mu"], nb)
    mm = _GpuPet(prob, be)
    lam = [torch.ones(geo.n_pixels, device=dev), torch.empty(geo.n_pixels, device=dev)]
    cur = [0]

    def step():
        a = cur[0]
        mm._iterate(lam[a], lam[1 - a], mm.status.f_ptr, mm.status.err_ptr)
        cur[0] = 1 - a

    timing = time_steps(args, torch, dev, step, world)
    prof = timing["prof"]
    nnz = int(sa["rval"].numel())
    # streamed bytes of each projector (values fp32 + int32 indices + the
    # row/column pointers); the gathers of lam / ratio hit L2 and are excluded
    alg = {"pet_sfwd": nnz * 8 + (geo.n_rays + 1) * 4 + geo.n_rays * 12,
           "pet_sback_pixel": nnz * 8 + (geo.n_pixels + 1) * 4 + geo.n_pixels * 8}
    launches = sum(c for c, _ in prof.values()) // args.steps
    roof = roofline(prof, alg, "hbm", args.workload)
    kernels = {k: {"launches_per_step": c // args.steps, "avg_ms": ms / c}
               for k, (c, ms) in prof.items()}
    mm._check_error()
    e2e = None
    if not args.no_e2e and world == 1:
        e2e = pet_e2e(args, torch, be, geo, y.cpu().numpy(), W["mu"], nb)
    return timing, roof, launches, e2e, {
        "kernels": kernels,
        "data": f"synthetic (Poisson counts of 50 x E default_phantom(256), torch generator; "
                f"E = device Siddon matrix, {nnz} nonzeros)"}


def pet_e2e(args, torch, be, geo, y_host, mu, nb):
    """The public API end to end: the geometry -> the system matrix built on
    the device, the host counts and the penalty lattice uploaded, pet_run for
    `steps` iterations, the image read back to the host.  The problem object
    (host validation, neighbour CSR) is built outside the timed region, as
    nnmf_e2e builds NnmfProblem."""
    import numpy as np
    import paper_1003_3272_b200 as M
    prob = M.SparsePetProblem(M.system_matrix_device(geo, be), y_host, mu, nb)
    cfg = M.MmConfig(max_iters=args.steps, epsilon=1e-300, monotone_tol=1e-6)

    def run():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prob.sa = M.system_matrix_device(geo, be)   # E from the geometry, on the device
        prob._dev.clear()                            # counts and lattice uploaded in the run
        lam, tr = M.pet_run(prob, cfg, be)
        lam = np.asarray(lam)                        # host image
        torch.cuda.synchronize()
        return lam, tr, time.perf_counter() - t0

    lam, tr, dt0 = run()   # warms the allocators; the second run is timed
    lam, tr, dt = run()
    K = tr.iters
    h2d = y_host.nbytes + prob.nbr_indptr.nbytes + prob.nbr_indices.nbytes
    d2h = lam.nbytes + 8 * (K + 1)
    return {"value": K / dt, "unit": "iterations/s", "h2d_bytes_per_step": h2d // max(K, 1),
            "d2h_bytes_per_step": d2h // max(K, 1), "iters": K,
            "phases_ms": {"total": 1e3 * dt, "device_loop": 1e3 * tr.wall_time,
                          "build_upload_readback": 1e3 * (dt - tr.wall_time),
                          "warmup_run_total": 1e3 * dt0},
            "path": "system_matrix_device(geometry) + SparsePetProblem(host counts) + pet_run "
                    "-> host image; second of two runs"}


def time_region(args, torch, dev, warm, run, world):
    """Time ONE call of `run` (a whole public-API run of args.steps
    iterations) between CUDA events on the compute stream, after `warm`
    (args.warmup iterations through the same API); barrier + synchronize on
    both sides, max over ranks; nvidia-smi clocks sampled meanwhile."""
    import torch.distributed as dist
    warm()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with Clocks(dev.index) as clk:
        start.record(stream)
        run()
        end.record(stream)
        torch.cuda.synchronize(dev)
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    return {"ms_total": ms, "clocks": clk.summary()}


def time_steps(args, torch, dev, step, world):
    """Warm-up, then exactly args.steps timed steps between CUDA events on the
    compute stream (barrier + synchronize on both sides, max over ranks).
    The library's launch profiler records an event pair around every kernel
    launch of the timed region on its launch stream; ``prof`` holds
    {kernel: (launches, total ms)} for the roofline of the dominant kernel."""
    import torch.distributed as dist
    from paper_1003_3272_b200 import _lib
    lib = _lib.load()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    _lib.prof_report()                     # drop anything recorded earlier
    with Clocks(dev.index) as clk:
        lib.mmk_prof_enable(1)
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize(dev)
        lib.mmk_prof_enable(0)
    prof = _lib.prof_report()
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms = float(t.item())
    return {"ms_total": ms, "clocks": clk.summary(), "prof": prof}


FP64_PEAK_TFLOPS = 40.0
FLOP_KERNELS = {"nnmf_vstep_tile": True, "nnmf_wpart_tile": True}


def roofline(prof, alg, bound, workload):
    hbm, bf16, kind = peaks()
    name = max(prof, key=lambda k: prof[k][1])
    cnt, ms = prof[name]
    avg_ms = ms / cnt
    flops = FLOP_KERNELS.get(name)
    if flops is not None and name in alg:
        # CUDA-core fp64 kernels (csrc/nnmf_tile.cu) are bound by the FP64 FMA
        # rate, not HBM: algorithmic flops / time against the nominal B200
        # FP64 peak (no measured figure in MEASURED_PEAKS.json)
        achieved = alg[name] / (avg_ms * 1e-3) / 1e12
        return {"kernel": name, "bound": "fp64", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                "alg_flops": alg[name], "avg_ms": avg_ms,
                "peak_kind": "nominal (B200 FP64, 40 TFLOP/s)"}
    if name not in alg:
        return {"kernel": name, "bound": bound, "achieved": None, "peak": hbm, "unit": "GB/s",
                "frac": None, "traffic": None, "peak_kind": kind}
    achieved = alg[name] / (avg_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            t = json.load(fh)
        # per-workload captures ("kernel@workload"); the bare kernel names are
        # the captures of the headline workloads
        traffic = t.get(f"{name}@{workload}",
                        t.get(name) if workload in ("nnmf-large", "mds-large", "pet-large")
                        else None)
    return {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "alg_bytes": alg[name],
            "avg_ms": avg_ms, "peak_kind": kind}


def suite(args, torch, dev):
    """Paper shapes (BASELINE configs 1-3) through the public API with host
    numpy inputs, 1000 fixed iterations each, next to the CPU oracle; plus the
    time to the reference's default tolerance (epsilon 1e-9, at most 100,000
    iterations) for C1 / C2 / C3, the CPU time estimated from the oracle's
    iteration rate."""
    import numpy as np

    import paper_1003_3272_b200 as M
    from paper_1003_3272_b200 import datasets as D
    out = {}
    be = M.Backend(dtype="fp32", device=dev.index)
    cfg = M.MmConfig(max_iters=1000, epsilon=1e-300, monotone_tol=1e-6)

    def timed(fn):
        fn()   # warm (graph build, uploads cached per problem object)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = fn()
        torch.cuda.synchronize()
        return res, time.perf_counter() - t0

    x = np.random.default_rng(0).random((2429, 361)).astype(np.float32).astype(np.float64)
    g = np.random.default_rng(1)
    s0 = M.FactorPair(g.random((2429, 10)), g.random((10, 361)))
    prob = M.NnmfProblem(x=x, rank=10)
    (_, tr), dt = timed(lambda: M.nnmf_run(prob, cfg, be, state0=s0))
    cpu, thr, _ = cpu_sample("nnmf-c1", 3.0)
    out["nnmf-c1"] = {"gpu_it_s": tr.iters / dt, "cpu_it_s": cpu, "cpu_threads": thr,
                      "speedup": tr.iters / dt / cpu}
    xc = np.floor(np.random.default_rng(21).random((2429, 361)) * 6.0)
    g = np.random.default_rng(22)
    sc0 = M.FactorPair(g.random((2429, 10)), g.random((10, 361)))
    cprob = M.NnmfProblem(x=xc, rank=10)
    (_, tr), dt = timed(lambda: M.nnmf_poisson_run(cprob, cfg, be, state0=sc0))
    cpu, thr, _ = cpu_sample("poisson-c1", 3.0)
    out["poisson-c1"] = {"gpu_it_s": tr.iters / dt, "cpu_it_s": cpu, "cpu_threads": thr,
                         "speedup": tr.iters / dt / cpu}
    e = D.build_system_matrix(D.PetGeometry(64, 64))
    y = D.simulate_counts(D.default_phantom(64), e, 20260811)
    pprob = M.PetProblem(e=e, y=y, mu=1e-5, neighborhoods=D.build_neighborhoods(64))
    (_, tr), dt = timed(lambda: M.pet_run(pprob, cfg, be))
    cpu, thr, _ = cpu_sample("pet-c2", 3.0)
    out["pet-c2"] = {"gpu_it_s": tr.iters / dt, "cpu_it_s": cpu, "cpu_threads": thr,
                     "speedup": tr.iters / dt / cpu}
    # time to the reference's default tolerance (epsilon 1e-9; the reference
    # converges at 3,266 iterations here)
    conv = M.MmConfig(max_iters=100000, epsilon=1e-9, monotone_tol=1e-6)
    (_, tr), dt = timed(lambda: M.pet_run(pprob, conv, be))
    out["pet-c2-to-tolerance"] = {"iters": tr.iters, "converged": bool(tr.converged),
                                  "gpu_s": dt, "cpu_s_est": tr.iters / cpu,
                                  "speedup": tr.iters / cpu / dt}
    diss = D.votes_to_dissimilarity(D.synthetic_votes(401, 671, 0))
    mprob = M.MdsProblem(weights=1.0 - np.eye(401), dissimilarities=diss, p=3)
    th0 = np.random.default_rng(1).uniform(-1, 1, size=(3, 401))
    (_, tr), dt = timed(lambda: M.mds_run(mprob, cfg, be, theta0=th0))
    cpu, thr, _ = cpu_sample("mds-c3", 3.0)
    out["mds-c3"] = {"gpu_it_s": tr.iters / dt, "cpu_it_s": cpu, "cpu_threads": thr,
                     "speedup": tr.iters / dt / cpu}
    (_, tr), dt = timed(lambda: M.mds_run(mprob, conv, be, theta0=th0))
    out["mds-c3-to-tolerance"] = {"iters": tr.iters, "converged": bool(tr.converged),
                                  "gpu_s": dt, "cpu_s_est": tr.iters / cpu,
                                  "speedup": tr.iters / cpu / dt}
    cpu_n = out["nnmf-c1"]["cpu_it_s"]
    (_, tr), dt = timed(lambda: M.nnmf_run(prob, conv, be, state0=s0))
    out["nnmf-c1-to-tolerance"] = {"iters": tr.iters, "converged": bool(tr.converged),
                                   "gpu_s": dt, "cpu_s_est": tr.iters / cpu_n,
                                   "speedup": tr.iters / cpu_n / dt}
    return out


def relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N ranks on this node (rank 0 prints the line)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_ours(args):
    import torch
    import torch.distributed as dist
    world, rank, local = dist_info()
    ndev = torch.cuda.device_count()
    # one rank per GPU over NCCL; more ranks than GPUs (a functional check of
    # the sharded path on a small box) share devices over gloo
    backend = "nccl" if world <= ndev else "gloo"
    dev = torch.device("cuda", local % ndev if world > 1 else 0)
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    from paper_1003_3272_b200 import build as B
    B.build()
    W = WORKLOADS[args.workload]
    if args.workload in ("nnmf-large", "nnmf-mid", "nnmf-r128"):
        timing, roof, launches, e2e, extra = bench_nnmf_large(args, torch, world, rank, dev)
    elif args.workload == "mds-large":
        timing, roof, launches, e2e, extra = bench_mds_large(args, torch, world, rank, dev)
    elif args.workload == "pet-large":
        timing, roof, launches, e2e, extra = bench_pet_large(args, torch, world, rank, dev)
    else:
        raise SystemExit(f"workload {args.workload} runs inside the suite (see --workload help)")
    extra = extra or {}
    ms = timing["ms_total"]
    # sharded workloads (NNMF rows, MDS tiles): every rank advances the same
    # iteration -> job throughput = steps / time (strong scaling of a fixed
    # problem).  PET runs replicas: N independent reconstructions.
    replicas = args.workload == "pet-large"
    value = (world if replicas else 1) * args.steps / (ms / 1000.0)
    cpu = None
    suite_res = None
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        v, thr, sample = cpu_sample(args.workload, args.cpu_seconds)
        cpu = {"value": v, "unit": "iterations/s", "cores": thr, "kind": "port",
               "sample": sample, "host": host_cpu()}
        if not args.no_suite:
            suite_res = suite(args, torch, dev)
    if rank == 0:
        line = {
            "metric": "MM iterations/sec", "value": value, "unit": "iterations/s",
            "n_gpus": world, "devices": min(world, ndev), "collectives": backend,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak (replicas)" if replicas else "strong",
            "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32" else "f64",
            "data": extra.get("data", "synthetic (uniform [0,1) X, uniform start; "
                                      "torch.Generator seeded)"),
            "config": workload_config(args, W, world),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches * args.steps, "clocks": timing["clocks"],
            "timing_note": "kernel times from CUDA events around every launch of the timed "
                           "region (library launch profiler); value from events bracketing "
                           "the region",
            "suite": suite_res,
            "kernels": extra.get("kernels"),
        }
        for k in ("kernel_loop_ms_per_step", "value_path", "e2e_note"):
            if k in extra:
                line[k] = extra[k]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
