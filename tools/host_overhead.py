import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1910_04126_b200 import flowtree as ft, workloads
wl = workloads.make("reviews", n_queries=1000)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
qi = torch.from_numpy(wl.q_ids).cuda(); qw = torch.from_numpy(wl.q_w.view(np.int32)).cuda().view(torch.uint32)
oi = torch.empty((wl.nq, wl.k), dtype=torch.int64, device="cuda"); ov = torch.empty((wl.nq, wl.k), dtype=torch.float64, device="cuda")
qi_pin = torch.from_numpy(wl.q_ids.copy()).pin_memory(); qw_pin = torch.from_numpy(wl.q_w.view(np.int32).copy()).pin_memory().view(torch.uint32)
oi_pin = torch.empty((wl.nq, wl.k), dtype=torch.int64).pin_memory(); ov_pin = torch.empty((wl.nq, wl.k), dtype=torch.float64).pin_memory()
st = torch.cuda.current_stream()
for mode in ("dev", "host"):
    for r in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        if mode == "dev": ds.knn(wl.q_off, qi, qw, wl.k, wl.prefilter_m, out_ids=oi, out_val=ov, stream=st)
        else: ds.knn(wl.q_off, qi_pin, qw_pin, wl.k, wl.prefilter_m, out_ids=oi_pin, out_val=ov_pin, stream=st)
        t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
        print(mode, r, "call %.2f ms, +sync %.2f ms" % ((t1 - t0) * 1e3, (t2 - t0) * 1e3), flush=True)
# the bench's e2e loop (L2 flush between steps), per step: device-event time and host wall time
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for r in range(12):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    ds.knn(wl.q_off, qi_pin, qw_pin, wl.k, wl.prefilter_m, out_ids=oi_pin, out_val=ov_pin, stream=st)
    e1.record(st)
    e1.synchronize()
    print("e2e step %d: events %.2f ms, wall %.2f ms" % (r, e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3), flush=True)
