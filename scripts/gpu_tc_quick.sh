# quick tensor-core check: TC tests + determinism + bench lines (kernel loop)
timeout 900 python -m pytest tests/test_nnmf_tc_gpu.py tests/test_nnmf_c4_gpu.py -x -q 2>&1 | tail -3
python scripts/tc_det2.py 131072 16384 20
for i in $(seq ${REPS:-3}); do
timeout 300 python bench.py --no-suite --no-e2e --steps ${STEPS:-50} --cpu-seconds 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('it/s', round(d['value'],1), 'loop ms', round(d['kernel_loop_ms_per_step'],4), 'vstep', round(k['nnmf_vstep_tc']['avg_ms'],4), 'wstep', round(k['nnmf_wstep_tc']['avg_ms'],4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
