"""Distance-table role clocks (FT_OPT_DEBUG bit 1) and stage time on a config's k-NN batch.
python tools/dist_dbg.py [config] [queries]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reviews"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
wl = workloads.make(name, n_queries=nq)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
qi = torch.from_numpy(wl.q_ids).cuda()
qw = torch.from_numpy(wl.q_w.view(np.int32)).cuda().view(torch.uint32)
oi = torch.empty((wl.nq, wl.k), dtype=torch.int64, device="cuda")
ov = torch.empty((wl.nq, wl.k), dtype=torch.float64, device="cuda")
m = wl.prefilter_m or 0
for dbg in (0, 1):
    ft.ft_set_option(ft.FT_OPT_DEBUG, dbg)
    ds.knn(wl.q_off, qi, qw, wl.k, m, out_ids=oi, out_val=ov)
    ft.ft_profile_enable(ds.h, True)
    ft.ft_profile_reset(ds.h)
    for _ in range(3):
        ds.knn(wl.q_off, qi, qw, wl.k, m, out_ids=oi, out_val=ov)
    ds.synchronize()
    p = ft.profile_dict(ds.h)
    ft.ft_profile_enable(ds.h, False)
    print("debug" if dbg else "plain", {k: round(v[0] / 3, 3) for k, v in p.items()}, flush=True)
