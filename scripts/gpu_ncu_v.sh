# ncu --set full of one V step launch (single CTA and pair forms) at C4
for v in 0 1; do
MMK_TC_PAIR=$v ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'nnmf_vstep_tc' -s 2 -c 1 \
  -o gpurun_out/prof_vstep_p$v python scripts/vstep_time.py > gpurun_out/ncu_v$v.log 2>&1; echo ncu$v rc=$?
done
