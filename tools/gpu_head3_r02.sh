#!/bin/bash
# gpurun: verify HEAD after the pacing rule (brK that fits L2 runs unpaced) -- default GPU suite, smoke,
# default bench, FHEW-like benches
cd "$(dirname "$0")/.."
O=gpurun_out/head3; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu_all.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_full.log 2>&1; echo "rc=$?" >> $O/bench_full.log
timeout 300 python bench.py --config fhew --steps 50 --warmup 5 --e2e-steps 5 --no-cpu-baseline > $O/bench_fhew.log 2>&1; echo "rc=$?" >> $O/bench_fhew.log
timeout 300 python bench.py --config fhew --batch 4096 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/bench_fhew4096.log 2>&1; echo "rc=$?" >> $O/bench_fhew4096.log
echo done
