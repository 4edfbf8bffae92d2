# round-2 final evidence: GPU tests, smoke, bench lines (driver's args), launch lists, ncu captures
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_nnmf.log 2>&1; tail -1 gpurun_out/bench_nnmf.log > gpurun_out/bench_line.json
timeout 900 python bench.py --steps 20 --warmup 5 --workload mds-large --no-suite > gpurun_out/bench_mds.log 2>&1; tail -1 gpurun_out/bench_mds.log > gpurun_out/bench_line_mds.json
timeout 900 python bench.py --steps 20 --warmup 5 --workload pet-large --no-suite > gpurun_out/bench_pet.log 2>&1; tail -1 gpurun_out/bench_pet.log > gpurun_out/bench_line_pet.json
timeout 900 python bench.py --steps 5 --warmup 3 --dtype fp64 --no-suite --no-e2e --cpu-seconds 0 > gpurun_out/bench_fp64.log 2>&1; tail -1 gpurun_out/bench_fp64.log > gpurun_out/bench_line_fp64.json
timeout 900 python bench.py --steps 20 --warmup 5 --workload nnmf-r128 --no-suite --cpu-seconds 0 > gpurun_out/bench_r128.log 2>&1; tail -1 gpurun_out/bench_r128.log > gpurun_out/bench_line_r128.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_line_ref.json
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --workload nnmf-mid --no-suite --no-e2e --cpu-seconds 0 > gpurun_out/bench_2rank.log 2>&1; tail -1 gpurun_out/bench_2rank.log > gpurun_out/bench_line_2rank.json
B="python bench.py --steps 3 --warmup 1 --no-e2e --no-suite --cpu-seconds 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'nnmf|gram|presplit|vprep|wreduce|wmax|split|xmax|objective|control|mmk' --csv \
  --log-file gpurun_out/launches_nnmf_large.csv $B > /dev/null 2>&1; echo l1 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'mds' --csv \
  --log-file gpurun_out/launches_mds_large.csv $B --workload mds-large > /dev/null 2>&1; echo l2 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'pet' --csv \
  --log-file gpurun_out/launches_pet_large.csv $B --workload pet-large > /dev/null 2>&1; echo l3 rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'nnmf_vstep_tc' -s 1 -c 1 \
  -o gpurun_out/prof_vstep $B > /dev/null 2>&1; echo fv rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'nnmf_wstep_tc|vprep_gram|gram32|wreduce_tc|wfinish|split_v|split_w|wmax' -s 8 -c 8 \
  -o gpurun_out/prof_wstep_helpers $B > /dev/null 2>&1; echo fw rc=$?
timeout 1500 ncu --set full --clock-control none -k regex:'dmma' -s 2 -c 2 \
  -o gpurun_out/prof_fp64_tile python bench.py --steps 2 --warmup 1 --dtype fp64 --no-e2e --no-suite --cpu-seconds 0 > /dev/null 2>&1; echo f64 rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'mds_tri_kernel' -s 1 -c 1 \
  -o gpurun_out/prof_mds_large $B --workload mds-large > /dev/null 2>&1; echo fm rc=$?
timeout 1500 ncu --set full --clock-control none -k regex:'pet_s' -s 4 -c 2 \
  -o gpurun_out/prof_pet_large $B --workload pet-large > /dev/null 2>&1; echo fp rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'nnmf_vstep_tc|vfinish' -s 2 -c 2 \
  -o gpurun_out/prof_r128 $B --workload nnmf-r128 > /dev/null 2>&1; echo fr rc=$?
