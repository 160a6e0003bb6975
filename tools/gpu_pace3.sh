#!/bin/bash
# gpurun: bounded-wait pacing x two-part bootstrap
cd "$(dirname "$0")/.."
O=gpurun_out/pace3; mkdir -p $O
for P in 0 32,160,8 32,160,2 0; do
  echo "== $P"; FDFB_BR_PACE=$P timeout 200 python tools/prof_br.py --acc 2960 --reps 2 2>&1 | tail -1
done > $O/prof.log 2>&1
for cfg in "1 0 1" "1 32,160,8 1" "1 32,160,2 1" "1 32,160,8 0" "1 32,160,32 1" "1 0 1"; do
  set -- $cfg
  echo "== split=$1 pace=$2 pace_split=$3"; FDFB_BOOT_SPLIT=$1 FDFB_BR_PACE=$2 FDFB_BR_PACE_SPLIT=$3 timeout 400 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
done > $O/bench.log 2>&1
echo done
