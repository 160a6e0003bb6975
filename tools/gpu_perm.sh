#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "permute or shift or pack" --durations=6 -m "not slow" > gpurun_out/pytest_perm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_perm.log
