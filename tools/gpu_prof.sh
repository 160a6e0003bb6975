#!/bin/bash
# gpurun: full-size bench, launch list, ncu --set full of the blind-rotation kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
timeout 300 python bench.py --batch 256 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_b256.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --batch 256 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_br.py --acc 148 > gpurun_out/prof_br_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate -s 1 -c 1 \
   -o gpurun_out/prof_br python tools/prof_br.py --acc 148 > gpurun_out/ncu_br.log 2>&1
echo done
