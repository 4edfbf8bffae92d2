python -c "from paper_1003_3272_b200 import build; build.build()"
MMK_TC_PAIR=1 timeout 300 python -m pytest tests/test_nnmf_tc_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
MMK_TC_PAIR=1 timeout 200 python scripts/tctrace.py | grep steady
MMK_TC_PAIR=1 timeout 300 python bench.py --steps 30 --no-e2e --no-suite --cpu-seconds 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('PAIR value %.1f frac %.3f clk %s vstep %.3f wstep %.3f' % (d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], k['nnmf_vstep_tc']['avg_ms'], k['nnmf_wstep_tc']['avg_ms']))"
