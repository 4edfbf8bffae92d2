# round evidence: full bench line, launch lists and ncu --set full captures of the top kernels (one GPU)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
B="python bench.py --steps 3 --warmup 1 --no-e2e --no-suite --cpu-seconds 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'nnmf|pois|gram|presplit|vprep|wreduce|wmax|split_w|sumsq|objective' --csv \
  --log-file gpurun_out/launches_nnmf_large.csv $B > gpurun_out/launches.log 2>&1; echo l1 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'mds' --csv \
  --log-file gpurun_out/launches_mds_large.csv $B --workload mds-large > gpurun_out/launches2.log 2>&1; echo l2 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'pet' --csv \
  --log-file gpurun_out/launches_pet_large.csv $B --workload pet-large > gpurun_out/launches3.log 2>&1; echo l3 rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'nnmf_(v|w)step_tc' -s 2 -c 2 \
  -o gpurun_out/prof_nnmf_large $B > gpurun_out/prof.log 2>&1; echo full rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'mds_tri_kernel' -s 1 -c 1 \
  -o gpurun_out/prof_mds_large $B --workload mds-large > gpurun_out/prof2.log 2>&1; echo full2 rc=$?
timeout 1500 ncu --set full --clock-control none -k regex:'pet_s' -s 4 -c 2 \
  -o gpurun_out/prof_pet_large $B --workload pet-large > gpurun_out/prof3.log 2>&1; echo full3 rc=$?
