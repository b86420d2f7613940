#!/bin/bash
# One GPU evidence pass: smoke, pytest -m gpu, the bench line per workload (+ the
# reference arm and a torchrun launch), the ncu launch list of the default bench
# command and full captures of the hot kernels, into gpurun_out/<tag>/.
# Usage (from the repo root, under gpurun):  bash scripts/gpu_round.sh [tag] [--no-tests]
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/nvsmi.txt 2>&1
if [ "$2" != "--no-tests" ]; then
  timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke=$?"
  timeout 1500 python -m pytest tests -m gpu -q -rfs -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu=$?"
  tail -1 $OUT/pytest_gpu.log
fi
timeout 600 python bench.py --steps 20 --warmup 3 > $OUT/bench_driver20.json 2> $OUT/bench_driver20.err; echo "bench_driver20=$?"
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench_default=$?"
timeout 600 python bench.py --op tone --steps 20 --warmup 3 > $OUT/bench_tone.json 2> $OUT/bench_tone.err; echo "bench_tone=$?"
for W in C2 C4 C1; do
  timeout 600 python bench.py --workload $W --steps 50 --warmup 5 --cpu-seconds 5 > $OUT/bench_$W.json 2> $OUT/bench_$W.err; echo "bench_$W=$?"
done
timeout 1200 python bench.py --workload C5 --steps 5 --warmup 3 --cpu-seconds 5 > $OUT/bench_C5.json 2> $OUT/bench_C5.err; echo "bench_C5=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "bench_ref=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu --no-methods > $OUT/bench_torchrun.json 2> $OUT/bench_torchrun.err; echo "bench_torchrun=$?"
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-methods --no-sustained"
$B > $OUT/ncu_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches_c3.csv $B > $OUT/ncu_launch.log 2>&1
echo "ncu_launches=$?"
$B > $OUT/ncu_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"ldg_stream_kernel" -s 3 -c 1 -o $OUT/prof_c3_decolor $B > $OUT/ncu_full_decolor.log 2>&1
echo "ncu_full_decolor=$?"
T="python bench.py --op tone --steps 5 --warmup 3 --no-e2e --no-cpu --no-methods --no-sustained"
$T > $OUT/ncu_plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"ldg_stream_kernel" -s 3 -c 1 -o $OUT/prof_c3_tone $T > $OUT/ncu_full_tone.log 2>&1
echo "ncu_full_tone=$?"
H="python bench.py --workload C4 --steps 2 --warmup 3 --no-e2e --no-cpu --no-sustained"
$H > $OUT/ncu_plain4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"hdr_tm_kernel" -s 3 -c 1 -o $OUT/prof_c4_hdr $H > $OUT/ncu_full_hdr.log 2>&1
echo "ncu_full_hdr=$?"
# local tone map (C3 frames): per-kernel split and full captures of its two per-pixel kernels
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.per_cycle_active \
  --clock-control none -k regex:lhe_ --csv python scripts/ab_tone.py --op local --images 16 --iters 1 --rounds 1 --configs "" \
  > $OUT/lhe_split.csv 2> $OUT/lhe_split.err; echo "lhe_split=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lhe_hist16|lhe_apply16" -c 2 -o $OUT/prof_c3_lhe \
  python scripts/ab_tone.py --op local --images 16 --iters 1 --rounds 1 --configs "" > $OUT/ncu_full_lhe.log 2>&1
echo "ncu_full_lhe=$?"
timeout 600 python scripts/ab_tone.py --op local --images 64 --iters 10 --rounds 3 --sleep 2 --configs "" > $OUT/ab_local.log 2>&1
timeout 600 python scripts/ab_tone.py --op tone_exact --images 256 --iters 20 --rounds 3 --sleep 2 --configs "" > $OUT/ab_tone_exact.log 2>&1
echo "ab=$?"
timeout 300 python scripts/hdr_trace.py --images 32 --runs 3 > $OUT/hdr_trace.log 2>&1
timeout 600 python scripts/ab_tone.py --op hdr --images 32 --iters 20 --rounds 3 --sleep 1 --configs "PF=4;TM=0;SCHED=grouped" > $OUT/ab_hdr.log 2>&1
echo "hdr_extra=$?"
