#!/bin/bash
# gpurun: round-2 evidence -- NCCL/sharded tests, every workload, Shift-path ncu, default launch list, BR ncu full.
# ncu reports stay in /tmp on the box; only their text summaries come back (gpurun_out <= 64 MiB).
cd "$(dirname "$0")/.."
O=gpurun_out/ev; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sharded.py -q > $O/pytest_sharded.log 2>&1; echo "rc=$?" >> $O/pytest_sharded.log
bash tools/gpu_workloads_r02.sh > $O/workloads_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_shift.csv \
   python bench.py --workload shift --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch_shift.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_shift_bits|k_imma|k_shift_gemm_finish' -c 3 \
   -o /tmp/shift_full python tools/traffic_step.py --workload shift > $O/ncu_shift.log 2>&1
python tools/ncu_summary.py /tmp/shift_full.ncu-rep > $O/ncu_shift_full.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv \
   python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 300 python tools/prof_br.py --acc 888 > $O/prof_br_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate -s 1 -c 1 \
   -o /tmp/prof_br_paced python tools/prof_br.py --acc 888 > $O/ncu_br.log 2>&1
python tools/ncu_summary.py /tmp/prof_br_paced.ncu-rep > $O/ncu_br_full.txt 2>&1
python tools/ncu_lines.py /tmp/prof_br_paced.ncu-rep _Z16k_blind_rotate_pILi2048ELi3ELb0EEv9DevParams9RnsParamsPKjPmiiiS3_PKmiS4_jjjj 60 > $O/ncu_br_lines.txt 2>&1
du -sh gpurun_out
echo done
