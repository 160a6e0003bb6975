#!/bin/bash
# gpurun: BR timing only (plus the BR parity tests) -- quick A/B of kernel variants.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "blind_rotate or bootstrap_tiny or noiseless" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 300 python tools/prof_br.py --acc 296 --reps 2 > gpurun_out/prof_br_plain.log 2>&1
