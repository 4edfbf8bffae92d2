python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'mds_tri_kernel|mds_tri_accum' -s 2 -c 2 -o gpurun_out/prof_mds_tri python bench.py --workload mds-large --steps 2 --warmup 1 --no-e2e --no-suite --cpu-seconds 0 > gpurun_out/prof_tri.log 2>&1; echo ncu rc=$?
