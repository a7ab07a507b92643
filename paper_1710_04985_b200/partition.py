"""Batch partitioner: independent right-hand
sides (or independent factors) are spread over the ranks of one node; every
rank holds a full replica of the analyzed factor.  There is no collective on
the solve path -- a single triangular system does not shard (each level
depends on the previous one), so only the batch is partitioned.

Host integer logic only; torch.distributed is used by the callers for
barriers and for gathering timings/results outside the timed region.
"""
from __future__ import annotations


def block_range(total: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of ``total`` items owned by ``rank``.
    The first ``total % world_size`` ranks get one extra item."""
    if world_size < 1 or not 0 <= rank < world_size or total < 0:
        raise ValueError("bad partition arguments")
    base, extra = divmod(total, world_size)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


def factor_assignment(weights, world_size: int) -> list[list[int]]:
    """Independent factors (NEXT-4) over the ranks: longest-processing-time
    greedy on the per-factor weights (e.g. nnz): factors in decreasing weight
    (ties by index) go to the least-loaded rank (ties: lowest rank).
    Deterministic; every factor is owned by exactly one rank; the maximum load
    is at most the mean load plus the largest weight."""
    if world_size < 1:
        raise ValueError("bad partition arguments")
    order = sorted(range(len(weights)), key=lambda i: (-weights[i], i))
    load = [0.0] * world_size
    owned: list[list[int]] = [[] for _ in range(world_size)]
    for i in order:
        r = min(range(world_size), key=lambda q: (load[q], q))
        owned[r].append(i)
        load[r] += float(weights[i])
    return [sorted(o) for o in owned]


def all_ranges(total: int, world_size: int) -> list[tuple[int, int]]:
    return [block_range(total, world_size, r) for r in range(world_size)]


def gather_columns(local, total: int, group=None):
    """Reassemble the (n, total) result from each rank's (n, cols_r) block
    (outside any timed region).  Works with the gloo and nccl backends."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    ranges = all_ranges(total, ws)
    width = max(b - a for a, b in ranges)
    n = local.shape[0]
    pad = local.new_zeros((n, width))
    pad[:, :local.shape[1]] = local
    bufs = [torch.empty_like(pad) for _ in range(ws)]
    dist.all_gather(bufs, pad.contiguous(), group=group)
    return torch.cat([bufs[r][:, :ranges[r][1] - ranges[r][0]] for r in range(ws)], dim=1)
