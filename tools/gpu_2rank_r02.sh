#!/bin/bash
# gpurun: functional run of bench.py's multi-rank path on the one GPU (FDFB_SHARE_DEVICE=1 maps both
# ranks to device 0; gloo carries the key broadcast and the max-over-ranks reduction; NCCL refuses two
# ranks on one device).  Not a measurement: the ranks time-slice the GPU.
cd "$(dirname "$0")/.."
O=gpurun_out/tworank; mkdir -p $O
FDFB_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29541 bench.py --gpus 2 --steps 1 --warmup 1 --e2e-steps 1 --batch 1024 --dist-backend gloo --no-cpu-baseline \
  > $O/bench_2rank_shared_device_functional.log 2>&1; echo "rc=$?" >> $O/bench_2rank_shared_device_functional.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $O/bench_ref_2rank.log 2>&1; echo "rc=$?" >> $O/bench_ref_2rank.log
echo done
