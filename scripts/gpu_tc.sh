python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 600 python bench.py --workload pet-large --steps 50 --warmup 3 --no-suite --cpu-seconds 5 2>&1 | tail -c 2500
