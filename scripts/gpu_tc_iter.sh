# tensor-core NNMF iteration loop: TC tests + a short C4 bench line
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_nnmf_tc_gpu.py tests/test_nnmf_c4_gpu.py tests/test_tc_gpu.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_tc.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_tc.log
timeout 600 python bench.py --no-suite --no-e2e --steps 30 --cpu-seconds 0 > gpurun_out/bench_tc.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_tc.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', d['value'], 'ms', d['ms_per_step'], 'clocks', d['clocks'])
for k,v in d['kernels'].items(): print(k, v)"
