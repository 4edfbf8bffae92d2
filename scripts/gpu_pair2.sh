timeout 200 python -m pytest tests/test_nnmf_tc_gpu.py -x -q -k "test_tc_iteration_matches_fp64 or deterministic or run_parity" 2>&1 | tail -2
for v in 1 0 1 0; do MMK_TC_PAIR=$v TAG=cur timeout 300 python scripts/vstep_time.py 2>&1 | grep vstep; done
bash scripts/gpu_trace.sh
