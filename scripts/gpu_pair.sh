# CTA-pair V step: quick correctness, then the TC tests, then A/B bench lines
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 120 python -m pytest tests/test_nnmf_tc_gpu.py -x -q -k "test_tc_iteration_matches_fp64" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_nnmf_tc_gpu.py tests/test_nnmf_c4_gpu.py -x -q 2>&1 | tail -3
for v in 1 0 1 0; do
MMK_TC_PAIR=$v timeout 300 python bench.py --no-suite --no-e2e --steps ${STEPS:-50} --cpu-seconds 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('PAIR=$v it/s', round(d['value'],1), 'vstep', round(k['nnmf_vstep_tc']['avg_ms'],4), 'wstep', round(k['nnmf_wstep_tc']['avg_ms'],4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
