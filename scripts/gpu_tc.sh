python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_mds_tri_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python bench.py --workload mds-large --steps 30 --warmup 3 --no-e2e --no-suite --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('total %.3f ms' % d['ms_per_step']); [print('  %-22s %d %.4f' % (n, v['launches_per_step'], v['avg_ms'])) for n, v in k.items()]"
