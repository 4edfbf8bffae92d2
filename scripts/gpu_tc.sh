python -c "from paper_1003_3272_b200 import build; build.build()"
for w in nnmf-large mds-large pet-large; do
timeout 300 python bench.py --workload $w --no-e2e --no-suite --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$w value %.1f total %.3f ms' % (d['value'], d['ms_per_step']), d['clocks'], 'roof', round(d['roofline']['frac'],3), d['gpu_launches']); [print('  %-22s %d %.4f' % (n, v['launches_per_step'], v['avg_ms'])) for n, v in k.items()]"
done
