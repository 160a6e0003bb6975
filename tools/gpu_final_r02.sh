#!/bin/bash
# gpurun: round-2 final check -- full GPU suite, smoke, default bench line, butterfly microbenchmark
cd "$(dirname "$0")/.."
O=gpurun_out/final; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu_all.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_full.log 2>&1; echo "rc=$?" >> $O/bench_full.log
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/bfbench tools/bfbench.cu && timeout 120 /tmp/bfbench > $O/bfbench.jsonl 2>&1
echo done
