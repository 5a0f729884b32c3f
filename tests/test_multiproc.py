"""World-size-2 gloo test of the multi-GPU plumbing (paper_1910_04126_b200/parallel.py) on CPU.

The query path shards by query (no data-path collective): each rank answers a
disjoint contiguous slice of the batch and the timings are max-reduced.  With no GPU here, the
per-rank compute is the CPU oracle; the test checks the sharding covers the batch exactly once,
the per-rank answers concatenate to the single-process answers, and the reduction is a max.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_1910_04126_b200 import parallel, workloads
    wl = workloads.make("tiny", n_queries=7)
    q_off, q_ids, q_w, (a, b) = parallel.shard_queries(wl.q_off, wl.q_ids, wl.q_w, rank, world)
    T = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    res = []
    for q in range(len(q_off) - 1):
        ids, vals = T.knn(wl.doc_off, wl.ids, wl.w, q_ids[q_off[q]:q_off[q + 1]], q_w[q_off[q]:q_off[q + 1]],
                          wl.k, 30)
        res.append((a + q, ids.tolist(), vals.tolist()))
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    t = parallel.max_over_ranks(10.0 * (rank + 1), dist)
    if rank == 0:
        np.save(result_path, np.array([gathered, t], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover_once():
    from paper_1910_04126_b200 import parallel
    for nq in (1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                a, b = parallel.shard_bounds(nq, r, world)
                seen.extend(range(a, b))
                assert b - a in (nq // world, nq // world + 1)
            assert seen == list(range(nq))


def test_two_rank_gloo_sharded_knn(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    gathered, tmax = np.load(out, allow_pickle=True)
    assert tmax == 20.0
    flat = sorted(x for part in gathered for x in part)
    assert [x[0] for x in flat] == list(range(7))
    import oracle
    from paper_1910_04126_b200 import workloads
    wl = workloads.make("tiny", n_queries=7)
    T = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    for q, ids, vals in flat:
        ref_ids, ref_vals = T.knn(wl.doc_off, wl.ids, wl.w, *wl.query(q), wl.k, 30)
        assert ids == ref_ids.tolist() and vals == ref_vals.tolist()
