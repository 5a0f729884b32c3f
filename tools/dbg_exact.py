"""Time the exact-W1 stage on its own (1000 queries x 9 docs of a workload) and, with
FT_OPT_DEBUG bit 2, print the per-CTA cycle split (cost matrix / pointer jumping / pricing / cycle)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_1910_04126_b200 import flowtree as ft, workloads

name = sys.argv[1] if len(sys.argv) > 1 else "reviews"
nd = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
wl = workloads.make(name, n_docs=nd, n_queries=1000)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
rng = np.random.default_rng(0)
docs = torch.from_numpy(rng.integers(0, ds.n, (wl.nq, 9))).cuda()
for dbg in (False, True):
    if dbg:
        ft.ft_set_option(ft.FT_OPT_DEBUG, 2)
    for _ in range(2):
        out = ft.ft_exact_w1_lists(ds.h, wl.q_off, wl.q_ids, wl.q_w, docs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = ft.ft_exact_w1_lists(ds.h, wl.q_off, wl.q_ids, wl.q_w, docs)
    e1.record()
    torch.cuda.synchronize()
    print(name, "dbg" if dbg else "", f"{e0.elapsed_time(e1):.2f} ms for {docs.numel()} pairs",
          "nan", int(torch.isnan(out).sum()), flush=True)
