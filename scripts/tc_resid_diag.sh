python scripts/tc_resid_diag.py
python - <<'PY'
import os, sys
os.environ["MMK_TC_EXP"] = "4"
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_nnmf_tc_gpu as T
x, v, w = T.well_fit(1024, 2048, 3072)
print("F' kernel (no correction)", T.one_iter(x, v, w, force_simt=False)[2])
PY
