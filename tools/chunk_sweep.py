"""ft_knn batch time and per-stage times vs the distance-table query chunk (FT_OPT_TABLE_CHUNK):
small chunks keep a chunk's tables L2-resident between the table kernel and the Flowtree kernel.

  python tools/chunk_sweep.py [config] [chunk ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reviews"
chunks = [int(c) for c in sys.argv[2:]] or [0, 256, 128, 64, 32, 16]
wl = workloads.make(name, n_queries=1000 if name != "stress" else 256)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
dev = torch.device("cuda:0")
qi = torch.from_numpy(wl.q_ids).to(dev)
qw = torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32)
st = torch.cuda.current_stream()
oi = torch.empty((wl.nq, wl.k), dtype=torch.int64, device=dev)
ov = torch.empty((wl.nq, wl.k), dtype=torch.float64, device=dev)
ref = None
for c in chunks:
    ft.ft_set_option(ft.FT_OPT_TABLE_CHUNK, c)
    f = lambda: ds.knn(wl.q_off, qi, qw, wl.k, wl.prefilter_m, out_ids=oi, out_val=ov, stream=st)
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    ft.ft_profile_enable(ds.h, True)
    ft.ft_profile_reset(ds.h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    e1.synchronize()
    ds.synchronize(st)
    p = {k: v[0] / n for k, v in ft.profile_dict(ds.h).items() if v[1]}
    ft.ft_profile_enable(ds.h, False)
    ids = oi.cpu().numpy()
    if ref is None:
        ref = ids
    print(f"{name} chunk={c}: {e0.elapsed_time(e1) / n:.3f} ms/batch  " + " ".join(f"{k}={v:.3f}" for k, v in p.items())
          + f"  ids==ref {np.array_equal(ids, ref)}", flush=True)
ft.ft_set_option(ft.FT_OPT_TABLE_CHUNK, 0)
