"""Rank process for tests/test_dist.py (gloo, CPU): key broadcast, shard, gather, max."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2109_02731_b200.dist import broadcast_keys, gather_outputs, max_over_ranks, shard_range  # noqa: E402


def main():
    rank, world, total = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(sys.argv[1])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(5)
        ref = {"s": torch.randint(-1, 2, (64,), dtype=torch.int8, generator=g),
               "S": torch.randint(-1, 2, (256,), dtype=torch.int8, generator=g),
               "brk": torch.randint(0, 256, (4096,), dtype=torch.uint8, generator=g),
               "bpk": torch.randint(0, 256, (1000,), dtype=torch.uint8, generator=g),
               "ksk": torch.randint(0, 256, (777,), dtype=torch.uint8, generator=g), "pack": None}
        keys = {k: (None if v is None else (v.clone() if rank == 0 else torch.zeros_like(v))) for k, v in ref.items()}
        broadcast_keys(keys)
        ok_keys = all((keys[k] is None and ref[k] is None) or torch.equal(keys[k], ref[k]) for k in ref)
        start, count = shard_range(total, world, rank)          # this rank's ciphertexts
        idx = torch.arange(start, start + count, dtype=torch.int64)
        local = torch.stack([idx * 3 + 1, idx ^ 0x5A5A], dim=1).to(torch.uint64)
        full = gather_outputs(local, total)
        allidx = torch.arange(total, dtype=torch.int64)
        want = torch.stack([allidx * 3 + 1, allidx ^ 0x5A5A], dim=1).to(torch.uint64)
        print(json.dumps({"rank": rank, "keys": ok_keys, "gather": bool(torch.equal(full, want)),
                          "max": max_over_ranks(10.0 + rank)}), flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
