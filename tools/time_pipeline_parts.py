import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1910_04126_b200 import flowtree as ft, workloads, pipeline
wl = workloads.make("reviews", n_queries=1000)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
qi = torch.from_numpy(wl.q_ids).cuda(); qw = torch.from_numpy(wl.q_w.view(np.int32)).cuda().view(torch.uint32)
def tm(f, n=3):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); e1.synchronize(); return e0.elapsed_time(e1) / n
ids = torch.empty((1000, 9), dtype=torch.int64, device="cuda"); vals = torch.empty((1000, 9), dtype=torch.float64, device="cuda")
print("knn(9,424)", tm(lambda: ds.knn(wl.q_off, qi, qw, 9, 424, out_ids=ids, out_val=vals)))
print("exact", tm(lambda: ft.ft_exact_w1_lists(ds.h, wl.q_off, qi, qw, ids)))
print("pipeline", tm(lambda: pipeline.knn_qt_ft_exact(ft, ds, wl.q_off, qi, qw, 424, 9, 1)))
i2 = torch.empty((1000, 10), dtype=torch.int64, device="cuda"); v2 = torch.empty((1000, 10), dtype=torch.float64, device="cuda")
print("knn(10,1000)", tm(lambda: ds.knn(wl.q_off, qi, qw, 10, 1000, out_ids=i2, out_val=v2)))
for c in ("3", "48"):
    ft.ft_set_option(ft.FT_OPT_TABLE_BUDGET_MB, int(c) * 1024)
    print("budget", c, "knn(9,424)", tm(lambda: ds.knn(wl.q_off, qi, qw, 9, 424, out_ids=ids, out_val=vals)))
