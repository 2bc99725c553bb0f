"""Point sharding across ranks (one process per GPU) — SURVEY §8e.

Points are independent, so a batch of N points is split into contiguous
slices of ceil(N / G) points, one per rank; the compiled program is replicated
(each rank compiles the same polynomial; kernels are cached per process). No
collective touches the data path. The optional result gather (`gather=True`)
concatenates the slices on every rank with one all_gather over padded,
equal-size buffers (NCCL over NVLink on GPUs, gloo in CPU tests).
"""
from __future__ import annotations

from typing import Callable, Sequence


def shard_bounds(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of `rank`'s contiguous slice; slices tile [0, n_total)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-n_total // world) if n_total else 0
    start = min(n_total, rank * per)
    return start, min(n_total, start + per)


def evaluate_sharded(evaluate: Callable, coords: Sequence, n_total: int, world: int, rank: int,
                     gather: bool = False, group=None):
    """Evaluates this rank's slice of `coords` (per-variable arrays or tensors
    holding the whole batch, or already-sliced shards when their length is the
    shard length) with `evaluate(shard_coords) -> tensor`. With gather=True
    returns the full n_total results on every rank (torch.distributed)."""
    start, stop = shard_bounds(n_total, world, rank)
    local = [c[start:stop] if len(c) == n_total else c for c in coords]
    out = evaluate(local)
    if not gather or world == 1:
        return out
    import torch
    import torch.distributed as dist
    per = -(-n_total // world)
    buf = torch.zeros(per, dtype=out.dtype, device=out.device)
    buf[: stop - start] = out
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    pieces = []
    for r in range(world):
        s, e = shard_bounds(n_total, world, r)
        pieces.append(parts[r][: e - s])
    return torch.cat(pieces)


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Timing reduction: the slowest rank defines the step time."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
