# A/B of rank-128 ring depths (scripts/tc_variants.sh builds), V step time at C4 shape
cp paper_1003_3272_b200/libmmk.so /tmp/libmmk_orig.so
for rep in 1 2 3; do for v in "$@"; do
  cp scripts/_variants/libmmk_$v.so paper_1003_3272_b200/libmmk.so; touch paper_1003_3272_b200/libmmk.so
  TAG=$v R=128 timeout 300 python scripts/vstep_time.py 2>&1 | grep -E 'vstep_tc'
done; done
cp /tmp/libmmk_orig.so paper_1003_3272_b200/libmmk.so
