# round-2 baseline: GPU tests + default bench line on the round-1 tree
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-suite > gpurun_out/bench_base.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/bench_base.log
