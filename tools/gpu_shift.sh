#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --batch 296 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_bs.log 2>&1; echo "rc=$?" >> gpurun_out/bench_bs.log
timeout 600 python bench.py --workload shift --batch 64 --steps 2 --warmup 3 > gpurun_out/bench_shift64.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shift64.log
timeout 900 python bench.py --workload shift --steps 3 --warmup 3 > gpurun_out/bench_shift.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shift.log
