"""Extract the judged metric columns of an ncu --set full report into a CSV
(profiles/<round>/ncu_full_*.csv)."""
import csv, io, subprocess, sys

COLS = ["Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
idx = [h.index(c) if c in h else None for c in COLS]
with open(out, "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(COLS)
    w.writerow([rows[1][i] if i is not None else "" for i in idx])
    for r in rows[2:]:
        w.writerow([r[i] if i is not None else "" for i in idx])
print(open(out).read()[:2000])
