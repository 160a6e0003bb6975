#!/bin/bash
# gpurun: ncu --set full of one blind-rotation launch (296 accumulators = 2 CTAs per SM).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/prof_br.py --acc 296 > gpurun_out/prof_br_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate -s 1 -c 1 \
   -o gpurun_out/prof_br_${TAG:-x} python tools/prof_br.py --acc 296 > gpurun_out/ncu_br.log 2>&1
echo done
