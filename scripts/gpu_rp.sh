cp scripts/_variants/libmmk_rp.so paper_1003_3272_b200/libmmk.so
timeout 900 python -m pytest tests/test_nnmf_tc_gpu.py tests/test_nnmf_c4_gpu.py -x -q 2>&1 | tail -3
python scripts/tc_det2.py 131072 16384 20
bash scripts/tc_variants.sh run base rp
