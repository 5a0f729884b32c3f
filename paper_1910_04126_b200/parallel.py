"""Multi-GPU plumbing for the query path.

Two layouts, one process per GPU:

* query sharding (the bench default, weak scaling): docs are replicated (the ≤ 0.3 GB layout fits
  every GPU) and each rank answers a contiguous slice of the query batch — the path partitions
  into independent problems, so there is no data-path collective; only the timings are reduced.
* doc sharding: each rank holds a contiguous doc range [base, base + n_local) and
  the replicated index.  Per batch: local Quadtree + local top-m as (value, global id) →
  all-gather → merge to the global top-m by (value, id) — identical on every rank → each rank
  scores with the Flowtree the merged candidates it owns (+inf elsewhere) → MIN all-reduce →
  top-k.  Quadtree values are exact and the Flowtree value of a pair does not depend on which
  other pairs share its launch, so the answer is bit-identical to `ft_knn` on the whole
  collection.  The selection, Quadtree and Flowtree work runs in the library's kernels
  (`ft_topk`, `ft_quadtree_estimate`, `ft_flowtree_estimate_lists`); torch.distributed moves
  the candidate lists (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_bounds(nq_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous range [a, b) of `rank`; ranges are disjoint, cover [0, nq_total) and differ in
    size by at most one."""
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


def shard_docs(doc_off, ids, w, rank: int, world: int):
    """The rank's contiguous doc range as a CSR collection rebased to 0, and its first global id."""
    doc_off = np.asarray(doc_off, np.int64)
    a, b = shard_bounds(len(doc_off) - 1, rank, world)
    lo, hi = int(doc_off[a]), int(doc_off[b])
    return (doc_off[a:b + 1] - lo).astype(np.int64), np.asarray(ids)[lo:hi], np.asarray(w)[lo:hi], a


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity without a process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class LibShard:
    """A rank's share of the doc-sharded k-NN on its GPU, through the library."""

    def __init__(self, ft, dataset, base: int):
        self.ft, self.ds, self.base = ft, dataset, int(base)
        self.n_local = dataset.n

    def local_topm(self, q_off, q_ids, q_w, m: int):
        import torch
        nq = len(q_off) - 1
        vals = torch.empty((nq, self.n_local), dtype=torch.float64, device="cuda")
        self.ds.quadtree(q_off, q_ids, q_w, out=vals)
        return self.ft.ft_topk(vals, min(m, self.n_local) if self.n_local else m, id_base=self.base)

    def topk(self, vals, ids, k: int):
        return self.ft.ft_topk(vals.contiguous(), k, ids=ids.contiguous())

    def score_owned(self, q_off, q_ids, q_w, cand_ids):
        import torch
        local = cand_ids - self.base
        local = torch.where((local >= 0) & (local < self.n_local), local, torch.full_like(local, -1))
        return self.ft.ft_flowtree_estimate_lists(self.ds.h, q_off, q_ids, q_w, local.contiguous())


def knn_doc_sharded(shard, q_off, q_ids, q_w, k: int, m: int, dist):
    """Doc-sharded Quadtree-prefiltered Flowtree k-NN; every rank returns the same
    (ids [nq, k], values [nq, k]), equal to `ft_knn(k, m)` over the union of the shards."""
    import torch
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    ids_l, vals_l = shard.local_topm(q_off, q_ids, q_w, m)
    if ids_l.shape[1] < m:                                 # a shard smaller than m: pad (-1, +inf)
        pad = m - ids_l.shape[1]
        ids_l = torch.cat([ids_l, torch.full((ids_l.shape[0], pad), -1, dtype=ids_l.dtype, device=ids_l.device)], 1)
        vals_l = torch.cat([vals_l, torch.full((vals_l.shape[0], pad), float("inf"), dtype=vals_l.dtype,
                                               device=vals_l.device)], 1)
    if world > 1:
        ids_g = [torch.empty_like(ids_l) for _ in range(world)]
        vals_g = [torch.empty_like(vals_l) for _ in range(world)]
        dist.all_gather(ids_g, ids_l)
        dist.all_gather(vals_g, vals_l)
        ids_all, vals_all = torch.cat(ids_g, 1), torch.cat(vals_g, 1)
    else:
        ids_all, vals_all = ids_l, vals_l
    cand_ids, _ = shard.topk(vals_all, ids_all, m)        # the global top-m, identical on every rank
    fv = shard.score_owned(q_off, q_ids, q_w, cand_ids)   # +inf for candidates another rank owns
    if world > 1:
        dist.all_reduce(fv, op=dist.ReduceOp.MIN)
    return shard.topk(fv, cand_ids, k)
