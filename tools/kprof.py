"""Run single stages of the hot path on the reviews-like config (for ncu captures).

  python tools/kprof.py qt|ft|knn|exact [--queries N]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("what", choices=["qt", "ft", "knn", "exact"])
p.add_argument("--queries", type=int, default=1000)
p.add_argument("--config", default="reviews")
p.add_argument("--reps", type=int, default=2)
a = p.parse_args()
wl = workloads.make(a.config, n_queries=a.queries)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
dev = torch.device("cuda:0")
qi = torch.from_numpy(wl.q_ids).to(dev)
qw = torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32)
st = torch.cuda.current_stream()
for _ in range(a.reps):
    if a.what == "qt":
        out = torch.empty((wl.nq, wl.n), dtype=torch.float64, device=dev)
        ds.quadtree(wl.q_off, qi, qw, out=out, stream=st)
    elif a.what == "ft":
        out = torch.empty((wl.nq, wl.n), dtype=torch.float64, device=dev)
        ds.flowtree(wl.q_off, qi, qw, out=out, stream=st)
    elif a.what == "exact":
        from paper_1910_04126_b200 import pipeline
        pipeline.knn_qt_ft_exact(ft, ds, wl.q_off, qi, qw, 424, 9, 1, stream=st)
    else:
        oi = torch.empty((wl.nq, wl.k), dtype=torch.int64, device=dev)
        ov = torch.empty((wl.nq, wl.k), dtype=torch.float64, device=dev)
        ds.knn(wl.q_off, qi, qw, wl.k, wl.prefilter_m, out_ids=oi, out_val=ov, stream=st)
ds.synchronize(st)
print("ok", a.what)
