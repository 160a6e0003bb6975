#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/prof_br.py --acc 296 --reps 2 > gpurun_out/prof_br_plain.log 2>&1
