"""The random sphere model of PAPER.md §3.2 (:206-223) and its Figure 2 experiment (§4.1, :241-256)
— SURVEY §8(f) row 2 — run on the library.

Instance (SPEC.md synth-model): N ground points iid uniform on S^{d-1}; a planted
support x_1..x_s (s distinct ground points, uniform weights); the query ν is uniform over y_1..y_s,
y_k uniform on the sphere within chordal distance ε of x_k.  The query points are appended to the
ground set, so the quadtree is built over N + s points.

Success is measured two ways:
  * criteria (Theorem 5's proof; SPEC.md `trial_success`): H_k = the smallest
    quadtree cell holding both x_k and y_k; Quadtree succeeds iff every H_k holds no other point,
    Flowtree iff no H_k holds another planted x_j or query point y_j (the SPEC's conservative
    strengthening: it can only lower the Flowtree rate);
  * search: the planted doc against competitor docs that swap one x_k for another ground point of
    H_k (the near-misses that can fool the tree) plus random s-subsets, ranked by the library's
    Quadtree and Flowtree estimates of the one query; success = the planted doc is the unique
    minimum.

The quadtree, its paths and the estimates all come from the CUDA library through the C ABI; this
module draws inputs (numpy PCG64, no method arithmetic) and reads the outputs.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class Instance:
    X: np.ndarray          # [(N + s) x d] float32: ground points, then the query points
    N: int
    s: int
    eps: float
    planted: np.ndarray    # [s] ground ids x_1..x_s
    query: np.ndarray      # [s] ids y_1..y_s (= N .. N+s-1)


def _cap_point(rng, x: np.ndarray, eps: float) -> np.ndarray:
    """Uniform point of S^{d-1} within chordal distance eps of the unit vector x: the polar angle
    θ ≤ θmax = 2 asin(eps/2) has density ∝ sin^{d-2} θ (rejection against the uniform proposal),
    the direction in the tangent space at x is uniform."""
    d = x.shape[0]
    tmax = 2.0 * np.arcsin(min(eps, 2.0) / 2.0)
    while True:
        t = rng.uniform(0.0, tmax)
        if d == 2 or rng.uniform() <= (np.sin(t) / np.sin(tmax)) ** (d - 2):
            break
    g = rng.standard_normal(d)
    g -= (g @ x) * x
    u = g / np.linalg.norm(g)
    y = np.cos(t) * x + np.sin(t) * u
    return y / np.linalg.norm(y)


def generate_instance(N: int, d: int, s: int, eps: float, seed: int) -> Instance:
    """SPEC.md synth-model `generate_instance`, deterministic under `seed`."""
    if not (N >= s >= 1 and 0 < eps < 2 and d >= 2):
        raise ValueError("need N >= s >= 1, 0 < eps < 2, d >= 2")
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((N, d))
    G /= np.linalg.norm(G, axis=1, keepdims=True)
    planted = rng.choice(N, size=s, replace=False).astype(np.int32)
    Y = np.stack([_cap_point(rng, G[i], eps) for i in planted])
    X = np.concatenate([G, Y]).astype(np.float32)
    return Instance(X=X, N=N, s=s, eps=eps, planted=planted, query=np.arange(N, N + s, dtype=np.int32))


def _lca_cells(paths: np.ndarray, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Deepest common node of the root-to-leaf paths of points a[k] and b[k]."""
    pa, pb = paths[a], paths[b]
    same = (pa == pb) & (pa >= 0)
    depth = same.shape[1] - 1 - np.argmax(same[:, ::-1], axis=1)      # last common depth
    return pa[np.arange(len(a)), depth], depth


def trial_success(inst: Instance, paths: np.ndarray, node_count: np.ndarray) -> tuple[bool, bool]:
    """Theorem 5's criteria on the quadtree built over ground ∪ query (SPEC.md `trial_success`)."""
    cells, depth = _lca_cells(paths, inst.planted, inst.query)
    qt_ok = bool(np.all(node_count[cells] == 2))
    # H_k holds another x_j or y_j iff that point's path passes through H_k at depth(H_k)
    pts = np.concatenate([inst.planted, inst.query])
    owner = np.concatenate([np.arange(inst.s), np.arange(inst.s)])
    at = paths[pts][:, depth]                     # [2s x s]: node of point p at depth(H_k)
    inside = at == cells[None, :]
    inside &= owner[:, None] != np.arange(inst.s)[None, :]
    ft_ok = not bool(inside.any())
    return qt_ok, ft_ok


def competitors(inst: Instance, paths: np.ndarray, n_random: int, seed: int):
    """Docs for the search test: the planted support first, then every swap of one x_k for another
    ground point of H_k, then `n_random` random s-subsets of the ground ids (CSR, weights 1)."""
    rng = np.random.default_rng(seed)
    cells, depth = _lca_cells(paths, inst.planted, inst.query)
    docs = [np.sort(inst.planted)]
    ground_paths = paths[: inst.N]
    pset = set(inst.planted.tolist())
    for k in range(inst.s):
        members = np.nonzero(ground_paths[:, depth[k]] == cells[k])[0]
        for z in members:
            if int(z) in pset:
                continue
            sw = inst.planted.copy()
            sw[k] = z
            docs.append(np.sort(sw))
    for _ in range(n_random):
        docs.append(np.sort(rng.choice(inst.N, size=inst.s, replace=False)))
    ids = np.concatenate(docs).astype(np.int32)
    off = np.zeros(len(docs) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in docs])
    return off, ids, np.ones(len(ids), np.uint32)


def search_success(ft, inst: Instance, seed: int, max_depth: int, n_random: int = 200):
    """(quadtree_ok, flowtree_ok, n_docs) from the library's estimates over the competitor docs."""
    ix = ft.Index(inst.X, seed=seed, max_depth=max_depth)
    off, ids, w = competitors(inst, ix.paths(), n_random, seed + 1)
    ds = ft.Dataset(ix, off, ids, w)
    q_off = np.array([0, inst.s], np.int64)
    q_ids = np.sort(inst.query).astype(np.int32)
    q_w = np.ones(inst.s, np.uint32)
    qt = ds.quadtree(q_off, q_ids, q_w)[0]
    fl = ds.flowtree(q_off, q_ids, q_w)[0]
    unique_min = lambda v: bool(np.all(v[1:] > v[0]))
    return unique_min(qt), unique_min(fl), len(off) - 1


def sweep(ft, d: int, s: int, eps: float, N_values, trials: int, seed: int, max_depth: int = 32,
          n_random: int = 200, search_trials: int = 0):
    """Figure 2: per N, the fraction of trials each method succeeds."""
    rows = []
    for N in N_values:
        qt_c = ft_c = qt_s = ft_s = 0
        for t in range(trials):
            tseed = (seed * 1_000_003 + N * 7919 + t) % (2**63)
            inst = generate_instance(N, d, s, eps, tseed)
            ix = ft.Index(inst.X, seed=tseed, max_depth=max_depth)
            _, count = ix.nodes()
            a, b = trial_success(inst, ix.paths(), count)
            qt_c += a
            ft_c += b
            ix.close()
            if t < search_trials:
                a, b, _ = search_success(ft, inst, tseed, max_depth, n_random)
                qt_s += a
                ft_s += b
        row = {"N": N, "quadtree_rate": qt_c / trials, "flowtree_rate": ft_c / trials}
        if search_trials:
            row.update(quadtree_search_rate=qt_s / search_trials, flowtree_search_rate=ft_s / search_trials)
        rows.append(row)
    return rows


if __name__ == "__main__":
    import argparse
    import json

    from paper_1910_04126_b200 import flowtree as ft_lib

    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--d", type=int, default=10)
    p.add_argument("--s", type=int, default=10)
    p.add_argument("--eps", type=float, default=0.25)
    p.add_argument("--N", default="100,300,1000,3000,10000")
    p.add_argument("--trials", type=int, default=100)
    p.add_argument("--search-trials", type=int, default=20)
    p.add_argument("--seed", type=int, default=2019)
    a = p.parse_args()
    for r in sweep(ft_lib, a.d, a.s, a.eps, [int(x) for x in a.N.split(",")], a.trials, a.seed,
                   search_trials=a.search_trials):
        print(json.dumps(r))
