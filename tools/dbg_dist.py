"""Distance-table accuracy probe: single-point docs and queries expose the table directly."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402

wl = workloads.make("reviews", n_docs=64, n_queries=2)
rng = np.random.default_rng(3)
N = wl.X.shape[0]
xs = rng.choice(N, 3000, replace=False).astype(np.int32)
ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
ds = ft.Dataset(ix, np.arange(len(xs) + 1, dtype=np.int64), xs, np.ones(len(xs), np.uint32))
ys = rng.choice(N, 40, replace=False).astype(np.int32)
got = ds.flowtree(np.arange(len(ys) + 1, dtype=np.int64), ys, np.ones(len(ys), np.uint32))
Xd = wl.X.astype(np.float64)
ref = np.sqrt(((Xd[ys][:, None, :] - Xd[xs][None, :, :]) ** 2).sum(-1))
same = ys[:, None] == xs[None, :]
rel = np.abs(got - ref) / np.where(same, 1, ref)
rel[same] = 0
print("max rel", rel.max(), "median", np.median(rel), "p99", np.quantile(rel, 0.99))
qi, di = np.unravel_index(np.argmax(rel), rel.shape)
print("worst pair", qi, di, "got", got[qi, di], "ref", ref[qi, di])
mu = Xd.mean(0)
print("||mu||", np.linalg.norm(mu), "typical ||x-mu||^2", ((Xd[xs[:5]] - mu) ** 2).sum(1))
# emulate 1xTF32 and 3xTF32 errors for the worst pair
def tf32(v):
    b = v.astype(np.float32).view(np.uint32)
    return ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)
x = (Xd[xs[di]] - mu).astype(np.float32).astype(np.float64)
y = (Xd[ys[qi]] - mu).astype(np.float32).astype(np.float64)
xh, yh = tf32(x), tf32(y)
xl, yl = x - xh, y - yh
for name, dot in [("exact", x @ y), ("1xtf32", xh @ yh), ("3xtf32", xh @ yh + xh @ tf32(yl) + tf32(xl) @ yh)]:
    d2 = (x @ x) + (y @ y) - 2 * dot
    print(name, np.sqrt(max(d2, 0)), "rel", abs(np.sqrt(max(d2, 0)) - ref[qi, di]) / ref[qi, di])
# per-row / per-column error structure
print("rel by query (max):", np.round(rel.max(1)[:10], 7))
print("rel by doc (max) first 10:", np.round(rel.max(0)[:10], 7))
