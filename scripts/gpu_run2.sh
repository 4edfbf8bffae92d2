python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload mds-large --steps 10 --warmup 3 --cpu-seconds 0 --no-suite > gpurun_out/bench_mds.log 2>&1; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_mds.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernels'])"
timeout 300 python scripts/tctrace.py > gpurun_out/tctrace.log 2>&1; echo trace rc=$?
cat gpurun_out/tctrace.log | grep -E "steady|cols" 
