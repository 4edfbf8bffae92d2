python -c "from paper_1003_3272_b200 import build; build.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gram|vgw' --csv --log-file gpurun_out/lh.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-suite --cpu-seconds 0 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/lh.csv')))
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; start=i; break
ik=h.index('Kernel Name'); iv=h.index('Metric Value')
for r in rows[start+1:][-6:]: print(r[ik][:30], float(r[iv].replace(',',''))/1000, 'us')
PY
