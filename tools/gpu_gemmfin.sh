#!/bin/bash
# gpurun: GEMM-epilogue changes -- parity of shift / permute / key switches, then their benches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "shift or permute or keyswitch or bootstrap_tiny or fhew or multi or tfhe or empty" > gpurun_out/pytest_gemmfin.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemmfin.log
timeout 600 python bench.py --workload shift --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_shift.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shift.log
timeout 900 python bench.py --workload permute --batch 64 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_permute.log 2>&1; echo "rc=$?" >> gpurun_out/bench_permute.log
