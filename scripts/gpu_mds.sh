# packed-triangle MDS: tests + C5 bench (kernel time of mds_tri_kernel)
timeout 900 python -m pytest tests/test_mds_tri_gpu.py -x -q 2>&1 | tail -3
for i in 1 2; do
timeout 600 python bench.py --workload mds-large --no-suite --no-e2e --steps 30 --cpu-seconds 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('it/s', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'tri', {a: round(b['avg_ms'],4) for a,b in k.items() if 'tri' in a}, 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
