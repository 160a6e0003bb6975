#!/bin/bash
# gpurun: Shift-path evidence: launch list of the shift bench and ncu --set full of its three kernels
cd "$(dirname "$0")/.."
O=gpurun_out/shift; mkdir -p $O
timeout 600 python bench.py --workload shift --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --workload shift --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_shift_bits|k_imma|k_shift_gemm_finish' -c 3 \
   -o $O/shift_full python tools/traffic_step.py --workload shift > $O/ncu_full.log 2>&1
echo done
