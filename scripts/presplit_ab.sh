# A/B of the NNMF tensor-core variants at C4 (one GPU), interleaved; pass the
# env settings to compare as arguments (default: pre-split X vs split warps)
B="python bench.py --steps ${STEPS:-30} --warmup 3 --no-e2e --no-suite --cpu-seconds 0"
[ $# -eq 0 ] && set -- "" "MMK_TC_PRESPLIT=0"
for rep in 1 2; do
  for v in "$@"; do
    echo "== [$v]"
    env $v timeout 300 $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['frac'], d['clocks'], {k: round(v['avg_ms'],3) for k,v in d['kernels'].items() if 'step_tc' in k or 'presplit' in k})"
  done
done
