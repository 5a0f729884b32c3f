"""Time the k-NN stages of a config under several library variants (tools/variants.py builds) and
check that every variant returns the same answer as the first.
python tools/variant_bench.py reviews 1000 base e16 ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_1910_04126_b200 import flowtree as ft, workloads
cfg, _, trunc = CFG.partition(":q")
wl = workloads.make(cfg, n_queries=NQ)
if trunc:   # "reviews:q48": every query cut to its first 48 items (supports ≤ 48)
    T = int(trunc)
    qs = [wl.query(j) for j in range(wl.nq)]
    qs = [(i[:T], x[:T]) for i, x in qs]
    q_off = np.zeros(len(qs) + 1, np.int64); q_off[1:] = np.cumsum([len(i) for i, _ in qs])
    import dataclasses
    wl = dataclasses.replace(wl, q_off=q_off, q_ids=np.concatenate([i for i, _ in qs]).astype(np.int32),
                             q_w=np.concatenate([x for _, x in qs]).astype(np.uint32))
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
qi = torch.from_numpy(wl.q_ids).cuda(); qw = torch.from_numpy(wl.q_w.view(np.int32)).cuda().view(torch.uint32)
oi = torch.empty((wl.nq, wl.k), dtype=torch.int64, device="cuda"); ov = torch.empty((wl.nq, wl.k), dtype=torch.float64, device="cuda")
m = wl.prefilter_m or 0
ds.knn(wl.q_off, qi, qw, wl.k, m, out_ids=oi, out_val=ov); ds.synchronize()
ft.ft_profile_enable(ds.h, True); ft.ft_profile_reset(ds.h)
R = 5
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(R): ds.knn(wl.q_off, qi, qw, wl.k, m, out_ids=oi, out_val=ov)
e1.record(); ds.synchronize(); e1.synchronize()
p = {k: round(v[0] / R, 3) for k, v in ft.profile_dict(ds.h).items()}
np.save(OUT + "_i.npy", oi.cpu().numpy()); np.save(OUT + "_v.npy", ov.cpu().numpy())
print(json.dumps({"ms": round(e0.elapsed_time(e1) / R, 3), "stages": p}))
'''


def main():
    cfg, nq, names = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
    ref = None
    for name in names:
        lib = os.path.join(ROOT, "paper_1910_04126_b200", "libflowtree_b200.so") if name == "main" else \
            os.path.join(ROOT, "build", "variants", name, "libflowtree_b200.so")
        out = f"/tmp/vb_{cfg.replace(':', '_')}_{name}"
        code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfg)).replace("NQ", str(nq)).replace("OUT", repr(out))
        env = dict(os.environ, FT_LIB=lib)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        if p.returncode != 0:
            print(name, "FAILED", p.stderr[-1500:], flush=True)
            continue
        import numpy as np
        i, v = np.load(out + "_i.npy"), np.load(out + "_v.npy")
        same = ""
        if ref is None:
            ref = (i, v)
        else:
            same = f"ids_equal={bool((i == ref[0]).all())} vals_equal={bool((v == ref[1]).all())}"
        print(name, p.stdout.strip().splitlines()[-1], same, flush=True)


if __name__ == "__main__":
    main()
