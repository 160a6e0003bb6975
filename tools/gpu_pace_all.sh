#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/pace
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pacing or edge_moduli" > gpurun_out/pace/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pace/pytest.log
bash tools/gpu_pace.sh
