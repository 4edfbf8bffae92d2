# A/B of prebuilt libraries: every kernel of the rank-128 C4 iteration
cp paper_1003_3272_b200/libmmk.so /tmp/libmmk_orig.so
for rep in 1 2; do for v in "$@"; do
  cp scripts/_variants/libmmk_$v.so paper_1003_3272_b200/libmmk.so; touch paper_1003_3272_b200/libmmk.so
  echo "$v: $(ALL=1 TAG=$v R=128 timeout 300 python scripts/vstep_time.py 2>&1 | grep -E 'gram' | awk '{print $3, $5}' | tr '\n' ' ')"
done; done
cp /tmp/libmmk_orig.so paper_1003_3272_b200/libmmk.so
