# one ncu --set full capture of the V step at C4
B="python bench.py --steps 3 --warmup 1 --no-e2e --no-suite --cpu-seconds 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'nnmf_vstep_tc' -s 2 -c 1 \
  -o gpurun_out/prof_v $B > gpurun_out/prof_v.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/prof_v.log
