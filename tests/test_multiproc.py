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


class OracleShard:
    """The doc-sharded protocol's per-rank compute on the CPU oracle (numpy selection with the
    library's ordering: value, then id as uint32 so padding −1 sorts last)."""

    def __init__(self, T, doc_off, ids, w, base):
        self.T, self.doc_off, self.ids, self.w, self.base = T, doc_off, ids, w, base
        self.n_local = len(doc_off) - 1

    @staticmethod
    def _sel(vals, ids, k):
        import torch
        vals, ids = vals.numpy(), ids.numpy()
        out_i = np.full((vals.shape[0], k), -1, np.int64)
        out_v = np.full((vals.shape[0], k), np.inf)
        for r in range(vals.shape[0]):
            order = np.lexsort((ids[r].astype(np.uint32), vals[r]))[:k]
            out_i[r, :len(order)] = ids[r][order]
            out_v[r, :len(order)] = vals[r][order]
        return torch.from_numpy(out_i), torch.from_numpy(out_v)

    def local_topm(self, q_off, q_ids, q_w, m):
        import torch
        nq = len(q_off) - 1
        vals = np.array([[self.T.qt(self.ids[self.doc_off[d]:self.doc_off[d + 1]], self.w[self.doc_off[d]:self.doc_off[d + 1]],
                                    q_ids[q_off[q]:q_off[q + 1]], q_w[q_off[q]:q_off[q + 1]])[1]
                          for d in range(self.n_local)] for q in range(nq)])
        gid = np.broadcast_to(np.arange(self.n_local, dtype=np.int64) + self.base, vals.shape).copy()
        return self._sel(torch.from_numpy(vals), torch.from_numpy(gid), min(m, self.n_local))

    def topk(self, vals, ids, k):
        return self._sel(vals, ids, k)

    def score_owned(self, q_off, q_ids, q_w, cand_ids):
        import torch
        c = cand_ids.numpy()
        out = np.full(c.shape, np.inf)
        for q in range(c.shape[0]):
            for j, g in enumerate(c[q]):
                d = int(g) - self.base
                if 0 <= d < self.n_local:
                    out[q, j] = self.T.ft(self.ids[self.doc_off[d]:self.doc_off[d + 1]],
                                          self.w[self.doc_off[d]:self.doc_off[d + 1]],
                                          q_ids[q_off[q]:q_off[q + 1]], q_w[q_off[q]:q_off[q + 1]])
        return torch.from_numpy(out)


def _doc_worker(rank, world, port, result_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_1910_04126_b200 import parallel, workloads
    wl = workloads.make("tiny", n_queries=6)
    T = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    d_off, d_ids, d_w, base = parallel.shard_docs(wl.doc_off, wl.ids, wl.w, rank, world)
    shard = OracleShard(T, d_off, d_ids, d_w, base)
    ids, vals = parallel.knn_doc_sharded(shard, wl.q_off, wl.q_ids, wl.q_w, wl.k, 30, dist)
    if rank == 0:
        np.save(result_path, np.array([ids.numpy(), vals.numpy()], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_doc_sharded_knn(tmp_path):
    """Doc sharding: local top-m → all-gather → merge → owned Flowtree → MIN
    all-reduce → top-k equals the single-process Quadtree-prefiltered k-NN exactly."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "res_docs.npy")
    mp.spawn(_doc_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    ids, vals = np.load(out, allow_pickle=True)
    import oracle
    from paper_1910_04126_b200 import workloads
    wl = workloads.make("tiny", n_queries=6)
    T = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    for q in range(wl.nq):
        ref_ids, ref_vals = T.knn(wl.doc_off, wl.ids, wl.w, *wl.query(q), wl.k, 30)
        assert ids[q].tolist() == ref_ids.tolist() and vals[q].tolist() == ref_vals.tolist()


def test_shard_docs_cover_once():
    from paper_1910_04126_b200 import parallel, workloads
    wl = workloads.make("tiny")
    got_ids = []
    for r in range(3):
        off, ids, w, base = parallel.shard_docs(wl.doc_off, wl.ids, wl.w, r, 3)
        assert off[0] == 0 and off[-1] == len(ids) and base == parallel.shard_bounds(wl.n, r, 3)[0]
        got_ids.append(ids)
    assert np.array_equal(np.concatenate(got_ids), wl.ids)


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


class _HostCollectives:
    """torch.distributed over gloo with the library's CUDA tensors staged through host memory (the
    protocol's collectives; on a multi-GPU node they run on NCCL device buffers instead)."""

    def __init__(self, dist):
        self.d = dist
        self.ReduceOp = dist.ReduceOp

    def is_initialized(self):
        return self.d.is_initialized()

    def get_world_size(self):
        return self.d.get_world_size()

    def all_gather(self, outs, t):
        host = [o.cpu() for o in outs]
        self.d.all_gather(host, t.cpu())
        for o, h in zip(outs, host):
            o.copy_(h)

    def all_reduce(self, t, op):
        h = t.cpu()
        self.d.all_reduce(h, op=op)
        t.copy_(h)


def _lib_doc_worker(rank, world, port, result_path, name, n_docs, nq, m):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1910_04126_b200 import flowtree as ft, parallel, workloads
    wl = workloads.make(name, n_docs=n_docs, n_queries=nq) if name != "tiny" else workloads.make("tiny")
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    d_off, d_ids, d_w, base = parallel.shard_docs(wl.doc_off, wl.ids, wl.w, rank, world)
    ds = ft.Dataset(ix, d_off, d_ids, d_w)
    ids, vals = parallel.knn_doc_sharded(parallel.LibShard(ft, ds, base), wl.q_off, wl.q_ids, wl.q_w, wl.k, m,
                                         _HostCollectives(dist))
    if rank == 0:
        np.save(result_path, np.array([ids.cpu().numpy(), vals.cpu().numpy()], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name,n_docs,nq,m", [("reviews", 3000, 6, 200), ("tiny", None, None, 30)])
def test_two_process_library_doc_sharded_knn(tmp_path, name, n_docs, nq, m):
    """Doc sharding with the LIBRARY on each rank — Quadtree + ft_topk local top-m,
    all-gather, merge, the owned candidates' Flowtree through the distance table (d = 300), MIN
    all-reduce, top-k — in two processes (world size 2, gloo; one GPU shared, the ranks' kernels
    never wait on one another): bit-identical to a single ft_knn over the whole collection."""
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "res_lib.npy")
    mp.spawn(_lib_doc_worker, args=(2, _free_port(), out, name, n_docs, nq, m), nprocs=2, join=True)
    ids, vals = np.load(out, allow_pickle=True)
    from paper_1910_04126_b200 import flowtree as ft, workloads
    wl = workloads.make(name, n_docs=n_docs, n_queries=nq) if name != "tiny" else workloads.make("tiny")
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
    ref_ids, ref_vals = ds.knn(wl.q_off, wl.q_ids, wl.q_w, wl.k, m)
    assert np.array_equal(ids, ref_ids) and np.array_equal(vals, ref_vals)
