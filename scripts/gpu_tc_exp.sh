# timing experiment: V-step time with parts of the residual disabled (MMK_TC_EXP bits:
# 1 no residual MMAs, 2 no residual compute, 4 no correction terms)
for e in ${EXPS:-0 1 2 3}; do
  MMK_TC_EXP=$e timeout 300 python bench.py --no-suite --no-e2e --steps 20 --cpu-seconds 0 > gpurun_out/exp_$e.log 2>&1
  tail -1 gpurun_out/exp_$e.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('exp', $e, 'vstep', round(k['nnmf_vstep_tc']['avg_ms'],4), 'wstep', round(k['nnmf_wstep_tc']['avg_ms'],4), 'clk', d['clocks']['sm_mhz'])"
done
