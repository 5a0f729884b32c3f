import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1910_04126_b200 import flowtree as ft, workloads
for name, nd, nq in [("text", 1100, 5), ("reviews", 2000, 33)]:
    wl = workloads.make(name, n_docs=nd, n_queries=nq)
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
    a = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    os.environ["FT_GENERAL_ONLY"] = "1"
    b = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    del os.environ["FT_GENERAL_ONLY"]
    rel = np.abs(a - b) / np.abs(b)
    print(name, "max rel", np.nanmax(rel), "frac bad", np.mean(rel > 1e-5), "nan", np.isnan(a).sum())
    print(" per query frac bad", np.round(np.mean(rel > 1e-5, axis=1), 3))
    bad = np.argwhere(rel > 1e-5)[:5]
    for q, d in bad:
        print("  q", q, "d", d, a[q, d], b[q, d], "sq", wl.q_off[q+1]-wl.q_off[q], "sd", wl.doc_off[d+1]-wl.doc_off[d])
