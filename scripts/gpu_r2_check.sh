# round-2 re-entry check: GPU tests + default bench line + launch list + full ncu of the top kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_line.json'))
for k in ['value','ms_per_step','roofline','e2e','gpu_launches','clocks','cpu_baseline']: print(k, '=', json.dumps(d.get(k)))
for k,v in d.get('kernels',{}).items(): print(k, v)
PY
timeout 900 python bench.py --workload mds-large > gpurun_out/bench_mds.log 2>&1; echo mds rc=$?
tail -1 gpurun_out/bench_mds.log | cut -c1-1500
