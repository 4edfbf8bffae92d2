# ncu evidence for the headline bench (one GPU): launch list + full capture of the TC kernels
set -x
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-suite --cpu-seconds 0"
python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_nnmf_large.csv $B > gpurun_out/launches.log 2>&1; echo launches rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'nnmf_(v|w)step_tc|nnmf_gram64|nnmf_vgw' -s 8 -c 6 \
  -o gpurun_out/prof_nnmf_large $B > gpurun_out/prof.log 2>&1; echo full rc=$?
ls -la gpurun_out
