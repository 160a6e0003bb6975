"""Multi-GPU plumbing for the batched bootstrap.

Ciphertexts are independent (the paper parallelises over activations,
PAPER.md:2866-2867), so a batch shards into contiguous per-rank slices with no
data-path collective.  The only communication is the one-time key broadcast from
rank 0 (NCCL over NVLink on the GPU box; any torch.distributed backend works, the
tests use gloo on CPU) and, optionally, an untimed gather of the outputs.
"""
import torch
import torch.distributed as dist

KEY_ORDER = ("s", "S", "brk", "bpk", "ksk", "pack")


def shard_range(total: int, world: int, rank: int):
    """Contiguous shard [start, start+count) of `total` items for `rank`; the first
    total % world ranks get one extra item, so shards differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def broadcast_keys(keys: dict, src: int = 0, group=None) -> dict:
    """Broadcast every present key tensor from `src` in a fixed order (in place).
    Non-source ranks must pass tensors of the right size and dtype (e.g. from
    Context.sizes); None entries are skipped identically on every rank."""
    for name in KEY_ORDER:
        t = keys.get(name)
        if t is not None:
            dist.broadcast(t, src=src, group=group)
    return keys


def gather_outputs(local: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather the per-rank output shards (shard_range layout) into one tensor."""
    world = dist.get_world_size(group)
    if local.dtype == torch.uint64:                 # transport 64-bit words as int64 (bit pattern kept)
        return gather_outputs(local.view(torch.int64), total, group).view(torch.uint64)
    counts = [shard_range(total, world, r)[1] for r in range(world)]
    cap = max(counts)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (device times are reported as the max over ranks)."""
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
