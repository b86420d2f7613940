"""Top source lines (instructions executed, stall samples) of an ncu report:
python scripts/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
out, cur, h = [], None, None
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if h and len(r) == len(h) and r[0]:
        try:
            n = int(r[h.index("Instructions Executed")] or 0)
            st = int(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        if n or st:
            out.append((n, st, cur.split("/")[-1], r[0], r[1].strip()[:96]))
tot = sum(o[0] for o in out)
ts = sum(o[1] for o in out)
print(f"warp instructions {tot}, stall samples {ts}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0] / tot * 100:5.1f}% {o[1] / ts * 100:5.1f}%  {o[2]}:{o[3]}  {o[4]}")
