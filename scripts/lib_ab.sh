# A/B of prebuilt library variants (paper_1003_3272_b200/libmmk_<tag>.so) at C4,
# interleaved, sustained (STEPS, default 150): bash scripts/lib_ab.sh x4 x5 ...
P=paper_1003_3272_b200
cp $P/libmmk.so /tmp/libmmk_orig.so
for rep in 1 2; do
  for tag in "$@"; do
    cp $P/libmmk_$tag.so $P/libmmk.so
    echo "== [$tag]"
    timeout 300 python bench.py --steps ${STEPS:-150} --warmup 3 --no-e2e --no-suite --cpu-seconds 0 ${WORKLOAD:+--workload $WORKLOAD} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['frac'], d['clocks'], {k: round(v['avg_ms'],3) for k,v in d['kernels'].items() if 'step_tc' in k or 'mds_tri_kernel' in k})"
  done
done
cp /tmp/libmmk_orig.so $P/libmmk.so
