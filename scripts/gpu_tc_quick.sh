# quick tensor-core check: TC tests (not the C4 size) + a short bench line
timeout 600 python -m pytest tests/test_nnmf_tc_gpu.py tests/test_nnmf_c4_gpu.py -x -q -k "not c4" 2>&1 | tail -3
for i in 1 2; do
timeout 300 python bench.py --no-suite --no-e2e --steps 30 --cpu-seconds 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('it/s', round(d['value'],1), 'vstep', round(k['nnmf_vstep_tc']['avg_ms'],4), 'wstep', round(k['nnmf_wstep_tc']['avg_ms'],4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
