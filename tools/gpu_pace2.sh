#!/bin/bash
# gpurun: pacing x two-part bootstrap matrix (bench lines), the edge-moduli test, DRAM bytes of a paced step
cd "$(dirname "$0")/.."
O=gpurun_out/pace2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "edge_moduli" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for cfg in "1 0" "0 0" "0 32,160" "1 128,256" "0 16,64"; do
  set -- $cfg
  echo "== split=$1 pace=$2"; FDFB_BOOT_SPLIT=$1 FDFB_BR_PACE=$2 timeout 400 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-260
done > $O/bench.log 2>&1
FDFB_BOOT_SPLIT=0 FDFB_BR_PACE=32,160 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file $O/traffic_split0_pace.csv python tools/traffic_step.py > $O/traffic.log 2>&1
echo done
