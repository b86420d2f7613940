#!/bin/bash
# per-kernel device time / instructions / issue of the local tone map on 16 C3
# frames (ncu, one pass): bash scripts/lhe_split.sh <tag> [env...]
tag=$1; shift
mkdir -p gpurun_out/split
env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.per_cycle_active --clock-control none -k regex:lhe_ --csv python scripts/ab_tone.py --op local --images 16 --iters 1 --rounds 1 --configs "" > gpurun_out/split/$tag.csv 2>gpurun_out/split/$tag.err
