#!/bin/bash
# gpurun: middle-round bounded pacing (the new default) vs unpaced, pacing tests, DRAM bytes of a default step
cd "$(dirname "$0")/.."
O=gpurun_out/pace4; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pacing" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for P in 0 32,160,8 0 32,160,8; do
  echo "== $P"; FDFB_BR_PACE=$P timeout 200 python tools/prof_br.py --acc 2960 --reps 2 2>&1 | tail -1
done > $O/prof.log 2>&1
for P in 0 32,160,8 0 32,160,8; do
  echo "== pace=$P"; FDFB_BR_PACE=$P timeout 400 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
done > $O/bench.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file $O/traffic_default.csv python tools/traffic_step.py > $O/traffic.log 2>&1
echo done
