#!/bin/bash
# gpurun: round-2 closing evidence on one box -- the short workloads with the configuration-aware
# labels (Box-scale and the shift-based bootstrap are unchanged: profiles/r02/workloads), then the
# GPU suite with the larger oracle samples (FDFB_PARITY_FULL=1)
cd "$(dirname "$0")/.."
O=gpurun_out/final2; mkdir -p $O
run() { tag=$1; shift; timeout 600 python bench.py "$@" > $O/wl_$tag.log 2>&1; echo "rc=$?" >> $O/wl_$tag.log; }
run fhew --config fhew --steps 50 --warmup 5 --e2e-steps 5 --no-cpu-baseline
run fhew4096 --config fhew --batch 4096 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run tiny --config tiny --steps 300 --warmup 5 --e2e-steps 5 --no-cpu-baseline
run tfhe --workload tfhe --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run multilut --workload multilut --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline
run permute --workload permute --batch 64 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline
FDFB_PARITY_FULL=1 timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu_full_parity.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_full_parity.log
echo done
