python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_pet_sparse_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "pet" 2>&1 | tail -2
timeout 300 python bench.py --workload pet-large --steps 200 --no-e2e --no-suite --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value %.1f total %.4f ms' % (d['value'], d['ms_per_step'])); [print('  %-22s %d %.4f' % (n, v['launches_per_step'], v['avg_ms'])) for n, v in k.items()]"
python scripts/suite_probe.py 2>&1
