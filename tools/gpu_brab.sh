#!/bin/bash
# gpurun: BR kernel variant check -- parity subset + BR timing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m "not slow" -k "blind_rotate or bootstrap_tiny or noiseless or fhew or tfhe or multi or bootstrap_shift or empty or generic" > gpurun_out/pytest_brab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_brab.log
timeout 300 python tools/prof_br.py --acc 296 --reps 3 > gpurun_out/prof_br_ab.log 2>&1
