"""ft_knn batch stage times under different values of one library option (ft_set_option).
  python tools/opt_sweep.py config OPTION v1 v2 ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

name, opt = sys.argv[1], sys.argv[2]
vals = [int(v) for v in sys.argv[3:]]
wl = workloads.make(name, n_queries=1000 if name != "stress" else 256)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
dev = torch.device("cuda:0")
qi = torch.from_numpy(wl.q_ids).to(dev)
qw = torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32)
st = torch.cuda.current_stream()
oi = torch.empty((wl.nq, wl.k), dtype=torch.int64, device=dev)
ov = torch.empty((wl.nq, wl.k), dtype=torch.float64, device=dev)
for v in vals:
    ft.ft_set_option(getattr(ft, opt), v)
    f = lambda: ds.knn(wl.q_off, qi, qw, wl.k, wl.prefilter_m, out_ids=oi, out_val=ov, stream=st)
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    ft.ft_profile_enable(ds.h, True)
    ft.ft_profile_reset(ds.h)
    n = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    e1.synchronize()
    ds.synchronize(st)
    p = {k: x[0] / n for k, x in ft.profile_dict(ds.h).items() if x[1]}
    ft.ft_profile_enable(ds.h, False)
    print(f"{name} {opt}={v}: {e0.elapsed_time(e1) / n:.3f} ms/batch  " + " ".join(f"{k}={x:.3f}" for k, x in p.items()),
          flush=True)
ft.ft_set_option(getattr(ft, opt), 0)
