#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "shift or pack" --durations=5 > gpurun_out/pytest_shift.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shift.log
timeout 900 python bench.py --workload shift --steps 3 --warmup 3 > gpurun_out/bench_shift.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shift.log
