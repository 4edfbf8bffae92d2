python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_mds_tri_gpu.py -x -q -p no:cacheprovider > gpurun_out/tri_tests.log 2>&1; echo tri rc=$?
tail -30 gpurun_out/tri_tests.log
timeout 600 python bench.py --workload mds-large --steps 10 --warmup 3 --cpu-seconds 0 --no-suite > gpurun_out/bench_mds.log 2>&1; echo bench rc=$?
tail -c 1500 gpurun_out/bench_mds.log
