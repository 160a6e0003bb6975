#!/bin/bash
# gpurun: verify HEAD -- default GPU suite (timed), smoke, default bench line, reference arm, Shift bench
cd "$(dirname "$0")/.."
O=gpurun_out/head2; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu_all.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_full.log 2>&1; echo "rc=$?" >> $O/bench_full.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
timeout 600 python bench.py --workload shift > $O/bench_shift.log 2>&1; echo "rc=$?" >> $O/bench_shift.log
echo done
