# full GPU test suite + default bench line
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-suite > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_full.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','roofline','e2e','gpu_launches','clocks']: print(k, '=', json.dumps(d[k]))
for k,v in d['kernels'].items(): print(k, v)"
