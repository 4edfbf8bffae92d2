# fp64 DMMA tile kernels: parity tests + the fp64 C4 bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_nnmf_tile_gpu.py tests/test_edge_gpu.py tests/test_parity_gpu.py -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 --dtype fp64 --no-suite --no-e2e --cpu-seconds 0 > gpurun_out/bench_fp64.log 2>&1; tail -1 gpurun_out/bench_fp64.log > gpurun_out/bench_line_fp64.json
python -c "import json; d=json.load(open('gpurun_out/bench_line_fp64.json')); print(d['value'], d['roofline'], {k: round(v['avg_ms'],3) for k, v in d['kernels'].items() if v['avg_ms'] > 0.05})"
