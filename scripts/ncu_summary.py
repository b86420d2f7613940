#!/usr/bin/env python
"""Summarise an ncu --set full capture into the numbers the bench/roofline cite.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--algo-bytes N] > profiles/<round>/<name>.md

Reads the raw page (`ncu -i ... --page raw --csv`) and prints, per profiled
launch: duration, DRAM bytes read/written (the `traffic` figure), achieved
DRAM throughput, pipe utilisation (FMA / ALU / XU=MUFU), issue activity,
occupancy, registers, and the warp-stall breakdown.
"""

import argparse
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--algo-bytes", type=float, default=None, help="algorithmic bytes per launch")
    args = ap.parse_args()
    hdr, units, rows = raw_rows(args.rep)
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows:
        name = r[col["Kernel Name"]] if "Kernel Name" in col else "?"
        print(f"### {name}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key, label in KEYS:
            if key in col:
                print(f"| {label} (`{key}`) | {r[col[key]]} | {units[col[key]]} |")
        rd = to_float(r[col["dram__bytes_read.sum"]]) if "dram__bytes_read.sum" in col else None
        wr = to_float(r[col["dram__bytes_write.sum"]]) if "dram__bytes_write.sum" in col else None
        if rd is not None and wr is not None:
            scales = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            # ncu picks the unit per metric (e.g. Gbyte read, Mbyte written)
            traffic = (rd * scales.get(units[col["dram__bytes_read.sum"]], 1)
                       + wr * scales.get(units[col["dram__bytes_write.sum"]], 1))
            print(f"| traffic = read + write | {traffic:.6g} | byte |")
            if args.algo_bytes:
                print(f"| traffic / algorithmic bytes | {traffic / args.algo_bytes:.4f} | |")
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                v = to_float(r[i])
                if v:
                    stalls.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in stalls) or 1.0
        print("\nwarp-state samples: " + ", ".join(f"{n} {v / tot:.1%}" for v, n in sorted(stalls, reverse=True)[:10]))
        print()


if __name__ == "__main__":
    main()
