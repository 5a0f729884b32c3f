"""Selection statistics of the Quadtree rows (reviews): how many keys the sample threshold of
k_select_fast gathers per row, how many rows fall back to the radix kernel, and the select time."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads

wl = workloads.make("reviews", n_queries=1000)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
vals = torch.empty((wl.nq, ds.n), dtype=torch.float64, device="cuda")
ds.quadtree(wl.q_off, wl.q_ids, wl.q_w, out=vals)
v = vals.cpu().numpy()
L, S, k = ds.n, 4096, 1000
ex = k * S / L
ti = min(S - 1, int(ex + 4 * np.sqrt(ex) + 8))
cnts, distinct = [], []
for r in range(0, wl.nq, 10):
    samp = np.sort(v[r, (np.arange(S) * L) // S])
    t = samp[ti]
    cnts.append(int((v[r] <= t).sum()))
    distinct.append(len(np.unique(v[r])))
cnts = np.array(cnts)
print("gathered per row: median", np.median(cnts), "p90", np.percentile(cnts, 90), "max", cnts.max(),
      "rows > 8192:", int((cnts > 8192).sum()), "of", len(cnts), "| distinct values per row median", np.median(distinct))
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ids, val = ft.ft_topk(vals, k)
    e1.record(); e1.synchronize()
    print("ft_topk 1000 x 100k -> 1000:", round(e0.elapsed_time(e1), 3), "ms")
