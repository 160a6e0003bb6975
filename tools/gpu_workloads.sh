#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "large or multi or tfhe" -m "not slow" > gpurun_out/pytest_wl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wl.log
for w in bootstrap multilut tfhe permute; do
  B=4096; [ $w = permute ] && B=64
  timeout 900 python bench.py --workload $w --batch $B --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$w.log
done
