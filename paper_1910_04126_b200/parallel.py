"""Multi-GPU plumbing for the query path.

Docs are replicated (the ≤ 0.3 GB layout fits every GPU) and the query batch is sharded across
ranks, one process per GPU: the path partitions into independent problems, so there is no
data-path collective; the only communication is the max-over-ranks reduction of the timings.
Doc sharding with an all-gather of (key, id) top-m lists is SURVEY §8(e)'s next step.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(nq_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous query range [a, b) of `rank`; ranges are disjoint, cover [0, nq_total) and differ
    in size by at most one."""
    base, extra = divmod(nq_total, world)
    a = rank * base + min(rank, extra)
    b = a + base + (1 if rank < extra else 0)
    return a, b


def shard_queries(q_off, q_ids, q_w, rank: int, world: int):
    """The rank's queries as a CSR batch with offsets rebased to 0."""
    q_off = np.asarray(q_off, np.int64)
    a, b = shard_bounds(len(q_off) - 1, rank, world)
    lo, hi = int(q_off[a]), int(q_off[b])
    return (q_off[a:b + 1] - lo).astype(np.int64), np.asarray(q_ids)[lo:hi], np.asarray(q_w)[lo:hi], (a, b)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity without a process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
