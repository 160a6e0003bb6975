#!/bin/bash
# gpurun: full bench (default args), shift bench, launch list of a short bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
timeout 600 python bench.py --workload shift --steps 20 --warmup 3 > gpurun_out/bench_shift.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shift.log
timeout 300 python bench.py --batch 512 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_b512.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --batch 512 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
