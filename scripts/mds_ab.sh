# A/B of prebuilt libraries on the C5 MDS bench line (mds_tri kernel time, it/s)
cp paper_1003_3272_b200/libmmk.so /tmp/libmmk_orig.so
for rep in 1 2 3; do for v in "$@"; do
  cp scripts/_variants/libmmk_$v.so paper_1003_3272_b200/libmmk.so; touch paper_1003_3272_b200/libmmk.so
  timeout 300 python bench.py --workload mds-large --steps 20 --warmup 5 --no-suite --no-e2e --cpu-seconds 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['kernels']['mds_tri']['avg_ms'],4), d['roofline']['frac'] and round(d['roofline']['frac'],3), d['clocks']['reasons'])"
done; done
cp /tmp/libmmk_orig.so paper_1003_3272_b200/libmmk.so
