#!/bin/bash
# gpurun: the GPU suite with the larger oracle samples (FDFB_PARITY_FULL=1: 16 Large bootstraps,
# all five Config-4 Shift items) -- evidence run, ~20 min; the default suite is tools/gpu_head_r02.sh
cd "$(dirname "$0")/.."
O=gpurun_out/fullparity; mkdir -p $O
FDFB_PARITY_FULL=1 timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu_full_parity.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_full_parity.log
echo done
