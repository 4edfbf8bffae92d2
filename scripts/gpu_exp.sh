# A/B of V-step variants (scripts/tc_variants.sh builds) in both forms; no result checks
cp paper_1003_3272_b200/libmmk.so /tmp/libmmk_orig.so
for rep in 1 2; do
for name in ${VARS:-base e1 e2 e3}; do
  cp scripts/_variants/libmmk_$name.so paper_1003_3272_b200/libmmk.so
  for v in 0 1; do MMK_TC_PAIR=$v TAG=$name timeout 300 python scripts/vstep_time.py 2>&1 | grep vstep; done
done
done
cp /tmp/libmmk_orig.so paper_1003_3272_b200/libmmk.so
