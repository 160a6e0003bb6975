#!/bin/bash
# gpurun: end-of-round evidence -- full GPU suite, smoke, every bench workload, launch list, ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
for w in multilut tfhe; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$w.log
done
timeout 900 python bench.py --workload shiftboot --batch 1024 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/bench_shiftboot1024.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shiftboot1024.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_b512.csv \
  python bench.py --batch 512 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launches.log
TAG=final tools/gpu_ncu_br.sh
