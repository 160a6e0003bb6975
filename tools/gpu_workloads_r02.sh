#!/bin/bash
# gpurun: every bench workload once (evidence for profiles/r02), each under its own timeout
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() { tag=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/wl_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/wl_$tag.log; }
run multilut --workload multilut --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run tfhe --workload tfhe --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run shift --workload shift --steps 10 --warmup 3 --no-cpu-baseline
run permute --workload permute --batch 64 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run box --box --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run fhew --config fhew --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run tiny --config tiny --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run shiftboot --workload shiftboot --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline
for f in gpurun_out/wl_*.log; do echo "$f: $(tail -2 $f | head -1 | cut -c1-160)"; done
