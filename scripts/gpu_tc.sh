python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for k in 1 2; do python scripts/suite_probe.py 2>&1 | grep fused; done
MMK_SMALL_ENGINE=0 python scripts/suite_probe.py 2>&1 | grep "fused"
