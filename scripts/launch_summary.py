"""Per-kernel average duration from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

agg = defaultdict(list)
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"][:90]].append(float(d["Metric Value"].replace(",", "")))
for k, v in agg.items():
    print(f"{sum(v) / len(v) / 1e3:10.1f} us  x{len(v):<4d} {k}")
