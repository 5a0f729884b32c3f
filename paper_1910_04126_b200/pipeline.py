"""The paper's three-stage nearest-neighbour pipeline on the library: Quadtree → Flowtree → Exact W1
(§4.4 :402-431; Table 5 :935-937 — "Quadtree, Flowtree, Exact: 424, 9, 1"; SURVEY §8(f)
row 1).

Stage 1 keeps the c1 docs with the smallest Quadtree estimate, stage 2 the c2 of those with the
smallest Flowtree estimate (both inside `ft_knn(k=c2, prefilter_m=c1)`), stage 3 computes the exact
W1 of the c2 survivors (`ft_exact_w1_lists`, the transportation simplex) and returns the k smallest
by (W1, doc id) (`ft_topk`).  Every stage runs in the library's kernels; this module only chains
the calls on device tensors.
"""
from __future__ import annotations


def knn_qt_ft_exact(ft, ds, q_off, q_ids, q_w, c1: int = 424, c2: int = 9, k: int = 1, stream=None):
    """(ids [nq, k], exact W1 [nq, k]) as device tensors; padding −1 / +inf."""
    import torch
    nq = len(q_off) - 1
    ids_ft = torch.empty((nq, c2), dtype=torch.int64, device="cuda")
    val_ft = torch.empty((nq, c2), dtype=torch.float64, device="cuda")
    ds.knn(q_off, q_ids, q_w, c2, c1, out_ids=ids_ft, out_val=val_ft, stream=stream)
    w1 = ft.ft_exact_w1_lists(ds.h, q_off, q_ids, q_w, ids_ft, stream=stream)
    return ft.ft_topk(w1, k, ids=ids_ft, stream=stream)
