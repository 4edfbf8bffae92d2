python -c "from paper_1003_3272_b200 import build; build.build()"
for d in 0 1 2 3 4 6; do
  MMK_TC_DBG=$d timeout 300 python scripts/tctrace.py > gpurun_out/tctrace_$d.log 2>&1
  echo "dbg=$d"; grep steady gpurun_out/tctrace_$d.log
  MMK_TC_DBG=$d timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-suite --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('  vstep %.3f wstep %.3f total %.3f' % (k['nnmf_vstep_tc']['avg_ms'], k['nnmf_wstep_tc']['avg_ms'], d['ms_per_step']))"
done
