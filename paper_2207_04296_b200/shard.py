"""Batch sharding across ranks.

Single operators run on one GPU ("replicas only": `bench.py --gpus N` runs N
independent replicas). Batched workloads shard on the batch dimension with no
exchange in the hot path: rank r of W takes samples [r*B/W, (r+1)*B/W); weights
are replicated. Every output element keeps its reduction order, so the
concatenation of the shards equals the unsharded result bit-for-bit.
"""
from __future__ import annotations

from dataclasses import replace


def batch_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_spec(spec, rank: int, world: int):
    """(sub-spec for this rank's samples, (lo, hi)) for any spec with a batch `n`."""
    lo, hi = batch_range(spec.n, rank, world)
    return replace(spec, n=max(hi - lo, 0)), (lo, hi)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Timing rule: a multi-rank time is the max over ranks."""
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
