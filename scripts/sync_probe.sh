# synccheck of one small tensor-core run per rank tile (and the CTA-pair form)
CS=/usr/local/cuda/bin/compute-sanitizer
for R in 64 128 100; do
  echo "== R=$R: $(R=$R timeout 300 $CS --tool synccheck python scripts/sync_probe.py 2>&1 | grep -E 'ERROR SUMMARY|probe done' | tr '\n' ' ')"
done
echo "== pair R=64: $(MMK_TC_PAIR=1 R=64 timeout 300 $CS --tool synccheck python scripts/sync_probe.py 2>&1 | grep -E 'ERROR SUMMARY|probe done' | tr '\n' ' ')"
