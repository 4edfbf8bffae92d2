python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
python scripts/suite_probe.py 2>&1 | grep -A4 pet
