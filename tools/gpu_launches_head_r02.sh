#!/bin/bash
# gpurun: ncu launch lists (gpu__time_duration.sum, --clock-control none) of the default bench command and of
# the FHEW-like bench on HEAD; each command first runs without ncu (exit code recorded)
cd "$(dirname "$0")/.."
O=gpurun_out/launches_head; mkdir -p $O
timeout 600 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/bench_plain.log 2>&1; echo "rc=$?" >> $O/bench_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default_head.csv \
   python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
python tools/launch_summary.py $O/launches_default_head.csv > $O/launches_default_head_summary.txt 2>&1
timeout 300 python bench.py --config fhew --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/bench_fhew_plain.log 2>&1; echo "rc=$?" >> $O/bench_fhew_plain.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_fhew_head.csv \
   python bench.py --config fhew --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch_fhew.log 2>&1; echo "rc=$?" >> $O/ncu_launch_fhew.log
python tools/launch_summary.py $O/launches_fhew_head.csv > $O/launches_fhew_head_summary.txt 2>&1
echo done
