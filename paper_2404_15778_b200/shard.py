"""Sequence sharding across GPUs.

Batches shard by sequence: each rank holds a full main+draft replica and an
independent slot range; per-sequence RNG keys use the *global* sequence id
(ref:sampling.py:61-66, ref:engine.py:259-260), so a sequence's output does
not depend on which rank runs it.  There is no collective on the hot path —
only the start/stop barriers, the max-over-ranks time / sum-over-ranks token
reductions and one final gather of the generated tokens.
"""

from __future__ import annotations


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, end) of global sequences owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def global_sequence_ids(n_total: int, world: int, rank: int) -> list[int]:
    a, b = shard_range(n_total, world, rank)
    return list(range(a, b))


def reduce_run(dist, device, dev_s: float, host_s: float, tokens: int) -> tuple[float, float, int]:
    """(max device time, max host time, total tokens) over ranks."""
    import torch
    t = torch.tensor([dev_s, host_s], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n = torch.tensor([tokens], dtype=torch.int64, device=device)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t[0]), float(t[1]), int(n[0])


def gather_tokens(dist, world: int, sequence_ids: list[int], tokens: list[list[int]]):
    """Final gather: {global sequence id: tokens} on every rank."""
    mine = dict(zip(sequence_ids, tokens))
    out = [None] * world
    dist.all_gather_object(out, mine)
    merged = {}
    for part in out:
        merged.update(part)
    return merged
