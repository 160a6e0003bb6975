"""Rank process for tests/test_gpu_sharded.py: the Box-scale path of bench.py on a shared GPU
(FDFB_SHARE_DEVICE, gloo on the host): rank 0 generates the keys and broadcasts them, every rank
encrypts and bootstraps its contiguous shard with global object indices, and the shards are
gathered; rank 0 saves the gathered inputs and outputs (numpy) for the single-rank comparison.
FDFB_TEST_BACKEND=nccl runs the same path over NCCL with device tensors (one rank per GPU, so on
the one-GPU box a world of 1: the NCCL calls of bench.py's multi-GPU path, executed for real)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2109_02731_b200 import Context  # noqa: E402
from paper_2109_02731_b200.dist import broadcast_keys, gather_outputs, max_over_ranks, shard_range  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    name, total, out_path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    backend = os.environ.get("FDFB_TEST_BACKEND", "gloo")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.load_config(name)
        ctx = Context(cfg, 0)
        seed = cfg["seeds"]["keys"]
        if rank == 0:
            keys = ctx.keygen(seed, which=0x0F)
        else:
            keys = {"s": torch.empty(ctx.n, dtype=torch.int8, device=dev),
                    "S": torch.empty(ctx.N, dtype=torch.int8, device=dev),
                    "brk": ctx._bytes(ctx.sizes["brk"]), "bpk": ctx._bytes(ctx.sizes["bpk"]),
                    "ksk": ctx._bytes(ctx.sizes["ksk"]), "pack": None}
        torch.cuda.synchronize()
        if backend == "nccl":
            broadcast_keys(keys)                                                 # device tensors, NCCL
        else:
            host = {k: (None if v is None else v.cpu()) for k, v in keys.items()}   # gloo: host staging
            broadcast_keys(host)
            keys = {k: (None if v is None else v.to(dev)) for k, v in host.items()}
        start, count = shard_range(total, world, rank)
        msgs = synth.messages(cfg, total)[start:start + count]
        ct = ctx.lwe_encrypt(cfg["seeds"]["err"], keys["s"], torch.from_numpy(msgs.copy()).to(dev),
                             first_index=start)
        out = ctx.bootstrap_batch(keys, ctx.setup_lut(synth.lut(cfg)), ct)
        torch.cuda.synchronize()
        if backend == "nccl":
            full_in, full_out = gather_outputs(ct, total).cpu(), gather_outputs(out, total).cpu()
        else:
            full_in, full_out = gather_outputs(ct.cpu(), total), gather_outputs(out.cpu(), total)
        assert max_over_ranks(float(rank), device=dev if backend == "nccl" else None) == world - 1
        if rank == 0:
            np.savez(out_path, ct=full_in.numpy(), out=full_out.numpy())
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
