"""Flowtree-stage times of the kernel variants (reviews-like unless given):
python tools/ft_kernels.py [config] [knn_queries] [exhaustive_queries]
default = lane-per-pair k_ftd (+ warp kernel list mode); FT_OPT_WARP_ONLY = warp kernel for every
pair."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reviews"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
nqx = int(sys.argv[3]) if len(sys.argv) > 3 else 64
wl = workloads.make(name, n_queries=nq)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
qi = torch.from_numpy(wl.q_ids).cuda()
qw = torch.from_numpy(wl.q_w.view(np.int32)).cuda().view(torch.uint32)
oi = torch.empty((wl.nq, wl.k), dtype=torch.int64, device="cuda")
ov = torch.empty((wl.nq, wl.k), dtype=torch.float64, device="cuda")
sub = wl.subset_queries(nqx)
si = torch.from_numpy(sub.q_ids).cuda()
sw = torch.from_numpy(sub.q_w.view(np.int32)).cuda().view(torch.uint32)
out = torch.empty((sub.nq, wl.n), dtype=torch.float64, device="cuda")
res = {}
only = sys.argv[4].split(",") if len(sys.argv) > 4 else None
for var, warp_only in (("ftd", 0), ("warp", 1)):
    if only and var not in only:
        continue
    ft.ft_set_option(ft.FT_OPT_WARP_ONLY, warp_only)
    m = wl.prefilter_m if wl.prefilter_m else 0
    ds.knn(wl.q_off, qi, qw, wl.k, m, out_ids=oi, out_val=ov)
    ft.ft_profile_enable(ds.h, True)
    ft.ft_profile_reset(ds.h)
    for _ in range(3):
        ds.knn(wl.q_off, qi, qw, wl.k, m, out_ids=oi, out_val=ov)
    ds.synchronize()
    p = ft.profile_dict(ds.h)
    knn_ft = p["flowtree"][0] / 3 if "flowtree" in p else None
    ids_v = oi.cpu().numpy().copy()
    ds.flowtree(sub.q_off, si, sw, out=out)
    ft.ft_profile_reset(ds.h)
    for _ in range(3):
        ds.flowtree(sub.q_off, si, sw, out=out)
    ds.synchronize()
    p = ft.profile_dict(ds.h)
    ft.ft_profile_enable(ds.h, False)
    ex = p["flowtree"][0] / 3
    res[var] = (knn_ft, ex, out.cpu().numpy().copy(), ids_v)
    print(f"{name} {var}: knn flowtree stage {knn_ft:.3f} ms ({wl.nq} q); exhaustive {ex:.3f} ms "
          f"({sub.nq} q x {wl.n} docs = {sub.nq * wl.n / ex / 1e6:.3f} G pairs/s); dist {p.get('dist_table', (0,))[0]/3:.3f} ms",
          flush=True)
a = res["ftd"][2]
for v in [v for v in ("warp",) if v in res]:
    b = res[v][2]
    print(v, "max rel diff vs ftd", float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))),
          "knn ids equal", bool(np.array_equal(res[v][3], res["ftd"][3])))
