"""bench.py's reference arm (the CPU oracle, no GPU needed): one JSON line
with the contract's keys -- impl, metric / unit / higher_is_better, the
cpu_baseline object and an e2e object with zero copied bytes."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "nnmf-c1",
                          "--steps", "2", "--warmup", "1", "--cpu-seconds", "1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    ln = lines[0]
    assert ln["impl"] == "reference" and ln["metric"] == "MM iterations/sec"
    assert ln["unit"] == "iterations/s" and ln["higher_is_better"] is True
    assert ln["value"] > 0 and ln["steps"] == 2 and ln["warmup"] == 1
    cb = ln["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == ln["value"]
    assert ln["e2e"] == {"value": ln["value"], "unit": "iterations/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}
    assert ln["config"]["workload"] == "nnmf-c1"
