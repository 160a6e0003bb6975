#!/bin/bash
# gpurun: shift-based bootstrap (NEXT #4) parity + BR regression timing + a small shiftboot bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "shift or blind_rotate or bootstrap_tiny" > gpurun_out/pytest_shiftboot.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shiftboot.log
timeout 300 python tools/prof_br.py --acc 296 --reps 2 > gpurun_out/prof_br_plain.log 2>&1
timeout 900 python bench.py --workload shiftboot --batch 256 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/bench_shiftboot.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shiftboot.log
