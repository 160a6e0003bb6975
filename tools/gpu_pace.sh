#!/bin/bash
# gpurun: key-stream pacing A/B (FDFB_BR_PACE): BR time and DRAM bytes of a 10-round launch,
# then short bench steps.  Results are bit-identical by construction (pacing changes no arithmetic).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/pace
mkdir -p $O
for P in 0 32,160 16,96 64,320 0; do
  echo "== $P"; FDFB_BR_PACE=$P timeout 200 python tools/prof_br.py --acc 2960 --reps 2 2>&1 | tail -2
done > $O/prof.log 2>&1
for P in 0 32,160; do
  FDFB_BR_PACE=$P timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file $O/ncu_$P.csv python tools/prof_br.py --acc 2960 --reps 1 > $O/ncu_$P.log 2>&1
done
for P in 0 32,160 0 32,160; do
  echo "== $P"; FDFB_BR_PACE=$P timeout 400 python bench.py --steps 4 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1
done > $O/bench.log 2>&1
echo done
