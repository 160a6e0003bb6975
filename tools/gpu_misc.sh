#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k host_buffers > gpurun_out/pytest_host.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_host.log
FDFB_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --dist-backend gloo --batch 148 --steps 1 --warmup 3 --e2e-steps 1 > gpurun_out/bench_2rank.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2rank.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 3 --cpu-seconds 4 > gpurun_out/bench_ref2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref2.log
