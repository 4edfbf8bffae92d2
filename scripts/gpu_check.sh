# full GPU suite + smoke + C4 bench line (driver arguments)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-suite > gpurun_out/bench_nnmf.log 2>&1; tail -1 gpurun_out/bench_nnmf.log > gpurun_out/bench_line.json
python -c "import json; d=json.load(open('gpurun_out/bench_line.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], {k: round(v['avg_ms'],4) for k, v in d['kernels'].items() if v['avg_ms'] > 0.02})"
