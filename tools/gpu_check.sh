#!/bin/bash
# One gpurun call: GPU tests, integer-pipe microbenchmark, short bench runs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1; nproc >> gpurun_out/gpu.txt
timeout 120 ./tools/intbench > gpurun_out/intbench.json 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --batch 256 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b256.log 2>&1; echo "rc=$?" >> gpurun_out/bench_b256.log
