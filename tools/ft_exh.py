"""Exhaustive Flowtree stage time (all n docs for a query batch; the distance table timed apart)
and the ft_knn batch stage times, per config.   python tools/ft_exh.py [config] [queries]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reviews"
nqx = int(sys.argv[2]) if len(sys.argv) > 2 else 64
wl = workloads.make(name, n_queries=max(nqx, 8))
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
dev = torch.device("cuda:0")
qi = torch.from_numpy(wl.q_ids).to(dev)
qw = torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32)
st = torch.cuda.current_stream()
qoff = wl.q_off[: nqx + 1]
out = torch.empty((nqx, wl.n), dtype=torch.float64, device=dev)
f = lambda: ds.flowtree(qoff, qi, qw, out=out, stream=st)
f()
torch.cuda.synchronize()
ft.ft_profile_enable(ds.h, True)
ft.ft_profile_reset(ds.h)
n = 3
for _ in range(n):
    f()
ds.synchronize(st)
p = {k: v[0] / n for k, v in ft.profile_dict(ds.h).items() if v[1]}
ft.ft_profile_enable(ds.h, False)
fte = p.get("flowtree", float("nan"))
print(f"{name}: exhaustive {nqx} x {wl.n}: Flowtree {fte:.3f} ms ({nqx * wl.n / fte / 1e6:.3f} Gpairs/s), "
      f"table {p.get('dist_table', 0):.3f} ms", flush=True)
