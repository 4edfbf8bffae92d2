python -c "from paper_1003_3272_b200 import build; build.build()"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
for i in 1 2; do
timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-suite --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('total %.3f ms' % d['ms_per_step'], d['clocks']); [print('  %-22s %d %.4f' % (n, v['launches_per_step'], v['avg_ms'])) for n, v in k.items() if v['avg_ms'] > 0.02]"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
