python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
tail -c 1500 gpurun_out/bench_ref.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo ours rc=$?
tail -1 gpurun_out/bench_full.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','roofline','e2e','gpu_launches','clocks','suite']: print(k, '=', json.dumps(d[k]))"
