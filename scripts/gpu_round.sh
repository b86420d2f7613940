#!/bin/bash
# One GPU pass: smoke, parity tests, the bench line per workload (+ reference arm
# and a torchrun launch), and the ncu evidence (launch list + one full capture of
# the hot kernel) for the C3 bench command.
# Usage (from the repo root, under gpurun):  bash scripts/gpu_round.sh [tag]
TAG=${1:-r01e}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "smoke=$?"
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest_gpu=$?"
tail -1 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_default_$TAG.json 2> $OUT/bench_default_$TAG.err; echo "bench_default=$?"
for W in C2 C4 C1; do
  timeout 600 python bench.py --workload $W --steps 50 --warmup 5 --cpu-seconds 5 > $OUT/bench_${W}_$TAG.json 2> $OUT/bench_${W}_$TAG.err; echo "bench_$W=$?"
done
timeout 900 python bench.py --workload C5 --steps 5 --warmup 3 --cpu-seconds 5 > $OUT/bench_C5_$TAG.json 2> $OUT/bench_C5_$TAG.err; echo "bench_C5=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "bench_ref=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu > $OUT/bench_torchrun_$TAG.json 2> $OUT/bench_torchrun_$TAG.err; echo "bench_torchrun=$?"
B="python bench.py --workload C3 --steps 5 --warmup 3 --no-e2e --no-cpu"
$B > $OUT/ncu_plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $B > $OUT/ncu_launch_$TAG.log 2>&1
echo "ncu_launches=$?"
$B > $OUT/ncu_plain2_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o $OUT/prof_c3_$TAG $B > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu_full=$?"
T="python scripts/bench_methods.py --mpix 512 --iters 3 --methods tone_rgb,local"
$T > $OUT/methods_plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"tone_rgb_fast|lhe_(hist|apply)_u8g" -s 3 -c 3 -o $OUT/prof_tone_lhe_$TAG $T > $OUT/ncu_tone_lhe_$TAG.log 2>&1
echo "ncu_tone_lhe=$?"
