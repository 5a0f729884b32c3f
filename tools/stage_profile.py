"""Per-stage device times of one ft_knn call on a config (library stage events):
python tools/stage_profile.py text [queries]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "text"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
wl = workloads.make(name, n_queries=nq)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
qi = torch.from_numpy(wl.q_ids).cuda()
qw = torch.from_numpy(wl.q_w.view(np.int32)).cuda().view(torch.uint32)
oi = torch.empty((wl.nq, wl.k), dtype=torch.int64, device="cuda")
ov = torch.empty((wl.nq, wl.k), dtype=torch.float64, device="cuda")
ds.knn(wl.q_off, qi, qw, wl.k, wl.prefilter_m, out_ids=oi, out_val=ov)
ft.ft_profile_enable(ds.h, True)
ft.ft_profile_reset(ds.h)
ds.knn(wl.q_off, qi, qw, wl.k, wl.prefilter_m, out_ids=oi, out_val=ov)
ds.synchronize()
print(name, {k: round(v[0], 3) for k, v in ft.profile_dict(ds.h).items()})
