python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_sharded_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -25
