# round evidence: full bench line, launch lists and ncu --set full captures of the top kernels (one GPU)
set -x
python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
tail -c 4000 gpurun_out/bench_full.log
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-suite --cpu-seconds 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_nnmf_large.csv $B > gpurun_out/launches.log 2>&1; echo launches rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_mds_large.csv $B --workload mds-large > gpurun_out/launches2.log 2>&1; echo launches2 rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'nnmf_(v|w)step_tc' -s 2 -c 2 \
  -o gpurun_out/prof_nnmf_large $B > gpurun_out/prof.log 2>&1; echo full rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'mds_tri_kernel' -s 1 -c 1 \
  -o gpurun_out/prof_mds_large $B --workload mds-large > gpurun_out/prof2.log 2>&1; echo full2 rc=$?
