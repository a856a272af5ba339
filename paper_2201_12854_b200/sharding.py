"""Batch sharding for the multi-GPU forward.

Every (sequence, head) of the MCA forward is independent, so N
GPUs split the global batch into contiguous shards with no collective in the
hot path. Rank g encodes sequences [start, start + count) with
``b_offset = start``: stream ids use the global sequence index, so the sharded
outputs are bitwise the unsharded ones. The only communication is an optional
all_gather of the outputs (or their checksums) for validation, outside timing.
"""
from __future__ import annotations


def shard_range(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """(start, count) of rank's contiguous shard; the first global_batch % world
    ranks take one extra sequence."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if global_batch < 0:
        raise ValueError("global_batch < 0")
    base, extra = divmod(global_batch, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def gather_shards(local, global_batch: int, rank: int, world: int, group=None):
    """all_gather variable-size batch shards ([count, ...] tensors) into the
    global [global_batch, ...] tensor on every rank (validation only)."""
    import torch
    import torch.distributed as dist

    counts = [shard_range(global_batch, r, world)[1] for r in range(world)]
    cmax = max(counts) if counts else 0
    pad = torch.zeros((cmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)
