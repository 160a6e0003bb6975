#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/noise_large.py --logL-boot 11 --batches 26 > gpurun_out/noise_L11.log 2>&1
timeout 300 python tools/noise_large.py --logL-boot 8 --batches 3 > gpurun_out/noise_L8.log 2>&1
timeout 300 python tools/noise_large.py --logL-boot 14 --batches 3 > gpurun_out/noise_L14.log 2>&1
