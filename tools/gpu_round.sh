#!/bin/bash
# gpurun: full bench (default args), launch list of a short bench, ncu --set full of the top kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
timeout 300 python bench.py --batch 512 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_b512.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --batch 512 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_keyswitch|k_blind" -s 0 -c 4 \
   -o gpurun_out/prof_step python bench.py --batch 296 --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_step.log 2>&1
echo done
