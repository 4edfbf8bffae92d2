# pipeline trace of the V step (CTA 0) for the pair and single-CTA forms
cp paper_1003_3272_b200/libmmk.so /tmp/libmmk_orig.so
cp scripts/_variants/libmmk_trace.so paper_1003_3272_b200/libmmk.so
for v in ${MODES:-1 0}; do echo "== PAIR=$v"; MMK_TC_PAIR=$v timeout 300 python scripts/tc_trace.py 2>&1 | tail -14; done
cp /tmp/libmmk_orig.so paper_1003_3272_b200/libmmk.so
