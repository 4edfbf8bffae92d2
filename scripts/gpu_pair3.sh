timeout 300 python -m pytest tests/test_nnmf_tc_gpu.py -x -q 2>&1 | tail -2
VARS="base x5" bash scripts/gpu_exp.sh
MODES=0 bash scripts/gpu_trace.sh
