#!/bin/bash
# One gpurun call: GPU tests (not slow), then a short bench and one BR timing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --batch ${BENCH_B:-1024} --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
