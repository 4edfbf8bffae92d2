python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max --cache-control none --clock-control none -s 400 -c 60 --csv --log-file gpurun_out/warm_c1.csv python scripts/suite_probe.py > gpurun_out/ncu_warm.log 2>&1; echo ncu rc=$?
