#!/bin/bash
# gpurun: full GPU suite, then the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
