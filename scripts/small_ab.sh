# A/B of two prebuilt libraries on the paper-shape workloads (fused engine us/iteration)
cp paper_1003_3272_b200/libmmk.so /tmp/libmmk_orig.so
for rep in 1 2 3; do for v in "$@"; do
  cp scripts/_variants/libmmk_$v.so paper_1003_3272_b200/libmmk.so; touch paper_1003_3272_b200/libmmk.so
  echo "$v: $(timeout 300 python scripts/suite_probe.py 2>&1 | grep fused | tr '\n' ' ')"
done; done
cp /tmp/libmmk_orig.so paper_1003_3272_b200/libmmk.so
