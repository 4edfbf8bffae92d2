# rank-128 bench line + ncu captures of its V step and V' pass
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --steps 20 --warmup 5 --workload nnmf-r128 --no-suite --cpu-seconds 0 > gpurun_out/bench_r128.log 2>&1; tail -1 gpurun_out/bench_r128.log > gpurun_out/bench_line_r128.json
python -c "import json; d=json.load(open('gpurun_out/bench_line_r128.json')); print(d['value'], d['ms_per_step'], d['roofline'], d['e2e'] and d['e2e']['value'], {k: round(v['avg_ms'],4) for k, v in d['kernels'].items() if v['avg_ms'] > 0.02})"
B="python bench.py --workload nnmf-r128 --steps 3 --warmup 1 --no-e2e --no-suite --cpu-seconds 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'nnmf_vstep_tc|vfinish' -s 2 -c 2 \
  -o gpurun_out/prof_r128 $B > /dev/null 2>&1; echo fr rc=$?
