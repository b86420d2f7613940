"""Summarise gpurun_out/split/<tag>.csv (scripts/lhe_split.sh): last launch of each kernel."""
import csv
import sys

for tag in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f"gpurun_out/split/{tag}.csv")) if len(r) > 10]
    h = rows[0]
    agg = {}
    for r in rows[1:]:
        k = r[h.index("Kernel Name")].split("(")[0].split("::")[-1][:34]
        agg.setdefault(k, {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    print(tag)
    for k, d in agg.items():
        print(f"  {k:34s} {d['gpu__time_duration.sum'] / 1e3:8.1f} us  inst {d['smsp__inst_executed.sum'] / 1e6:7.1f}M"
              f"  issue {d['smsp__issue_active.avg.pct_of_peak_sustained_active']:5.1f}%"
              f"  warps {d['sm__warps_active.avg.per_cycle_active']:5.1f}"
              f"  dram {(d['dram__bytes_read.sum'] + d['dram__bytes_write.sum']) / 1e6:7.1f} MB")
