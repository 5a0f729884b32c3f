"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the tiny config (every stage, exhaustive and prefiltered k-NN, flow export) and a 2,000-doc
reviews subset that runs the d = 300 path — k_vocab, the tcgen05 distance table k_dist_i8, the
lane-per-pair Flowtree k_ftd with its warp-kernel hand-over, the selection kernels and the
exact-W1 simplex.   python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

for name, nd, nq, m in (("tiny", None, None, 30), ("reviews", 2000, 8, 200), ("image", 300, 2, 0)):
    wl = workloads.make(name, n_docs=nd, n_queries=nq)
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
    ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    ids, vals = ds.knn(wl.q_off, wl.q_ids, wl.q_w, wl.k, m)
    ds.knn(wl.q_off, wl.q_ids, wl.q_w, wl.k, 0)
    b, bw = wl.query(0)
    ds.flow(b, bw, 1)
    if name == "reviews":
        d_ids = torch.from_numpy(np.asarray(ids[:, :2], np.int64)).cuda()
        ft.ft_exact_w1_lists(ds.h, wl.q_off, wl.q_ids, wl.q_w, d_ids)
        ft.ft_set_option(ft.FT_OPT_WARP_ONLY, 1)
        ds.knn(wl.q_off, wl.q_ids, wl.q_w, wl.k, m)
        ft.ft_set_option(ft.FT_OPT_WARP_ONLY, 0)
    torch.cuda.synchronize()
    ds.close()
    ix.close()
print("sanitize workload ok")
