timeout 300 python -m pytest tests/test_nnmf_tc_gpu.py tests/test_nnmf_c4_gpu.py -x -q 2>&1 | tail -1
cp paper_1003_3272_b200/libmmk.so /tmp/libmmk_orig.so
cp scripts/_variants/libmmk_q1.so paper_1003_3272_b200/libmmk.so
timeout 300 python -m pytest tests/test_nnmf_tc_gpu.py tests/test_nnmf_c4_gpu.py -x -q 2>&1 | tail -1
cp /tmp/libmmk_orig.so paper_1003_3272_b200/libmmk.so
for rep in 1 2 3; do for name in base q1; do
  cp scripts/_variants/libmmk_$name.so paper_1003_3272_b200/libmmk.so
  MMK_TC_PAIR=0 TAG=$name timeout 300 python scripts/vstep_time.py 2>&1 | grep vstep
done; done
cp /tmp/libmmk_orig.so paper_1003_3272_b200/libmmk.so
