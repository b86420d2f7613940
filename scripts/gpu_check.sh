set -o pipefail
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
B2="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$B2 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/prof_u8 $B2 > gpurun_out/ncu_full.log 2>&1; echo full=$?
