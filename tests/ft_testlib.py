"""Test-only reference computations used to PIN the oracle to something other than itself
(DESIGN.md §4).  None of these retype the oracle's formulas: each computes the quantity by a
different route (an LP, an exhaustive enumeration, a recursive partitioner, a CDF integral)."""
from __future__ import annotations

import itertools
import json
import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------------------------
# exact W1 (Eq. (1)) as a transportation LP
# --------------------------------------------------------------------------------------------
def transport_lp(cost: np.ndarray, a: np.ndarray, b: np.ndarray) -> float:
    """min <τ, cost> s.t. τ 1 = a, τ^T 1 = b, τ >= 0 (scipy HiGHS)."""
    from scipy.optimize import linprog
    p, q = cost.shape
    A_eq = np.zeros((p + q, p * q))
    for i in range(p):
        A_eq[i, i * q:(i + 1) * q] = 1.0
    for j in range(q):
        A_eq[p + j, j::q] = 1.0
    res = linprog(cost.ravel(), A_eq=A_eq, b_eq=np.concatenate([a, b]), bounds=(0, None), method="highs",
                  options={"primal_feasibility_tolerance": 1e-10, "dual_feasibility_tolerance": 1e-10})
    assert res.status == 0, res.message
    return float(res.fun)


def euclid_cost(X, xs, ys):
    Xd = np.asarray(X, np.float64)
    A = Xd[np.asarray(xs)]
    B = Xd[np.asarray(ys)]
    return np.sqrt(((A[:, None, :] - B[None, :, :]) ** 2).sum(-1))


def exact_w1(X, mu_ids, mu_w, nu_ids, nu_w) -> float:
    a = np.asarray(mu_w, np.float64); a = a / a.sum()
    b = np.asarray(nu_w, np.float64); b = b / b.sum()
    return transport_lp(euclid_cost(X, mu_ids, nu_ids), a, b)


def birkhoff_w1(X, mu_ids, nu_ids) -> float:
    """Uniform, equal-size supports: by Birkhoff–von Neumann the LP optimum is attained at a
    permutation, so W1 = min over all s! permutations of the mean matched distance."""
    C = euclid_cost(X, mu_ids, nu_ids)
    s = len(mu_ids)
    perms = np.array(list(itertools.permutations(range(s))), dtype=np.int64)
    costs = C[np.arange(s)[None, :], perms].sum(1)
    return float(costs.min()) / s


def w1_1d_cdf(xs, a, ys, b) -> float:
    """1-D closed form W1 = ∫ |F_μ − F_ν| (points on the line)."""
    pts = sorted(set(map(float, xs)) | set(map(float, ys)))
    a = np.asarray(a, np.float64) / np.sum(a)
    b = np.asarray(b, np.float64) / np.sum(b)
    tot = 0.0
    for lo, hi in zip(pts[:-1], pts[1:]):
        Fa = sum(w for x, w in zip(xs, a) if x <= lo)
        Fb = sum(w for y, w in zip(ys, b) if y <= lo)
        tot += abs(Fa - Fb) * (hi - lo)
    return tot


# --------------------------------------------------------------------------------------------
# tree metric t(x, y) from a built tree (total edge weight on the leaf-leaf path,
# edge between level ℓ+1 and ℓ weighing 2^ℓ)
# --------------------------------------------------------------------------------------------
def tree_metric(paths: np.ndarray, l_root: int, xs, ys) -> np.ndarray:
    out = np.zeros((len(xs), len(ys)))
    for i, x in enumerate(xs):
        px = [v for v in paths[x] if v >= 0]
        for j, y in enumerate(ys):
            py = [v for v in paths[y] if v >= 0]
            lca = 0
            while lca + 1 < min(len(px), len(py)) and px[lca + 1] == py[lca + 1]:
                lca += 1
            t = 0.0
            for depth in range(lca + 1, len(px)):
                t += 2.0 ** (l_root - depth)
            for depth in range(lca + 1, len(py)):
                t += 2.0 ** (l_root - depth)
            out[i, j] = t
    return out


def tree_w1_lp(paths, l_root, mu_ids, mu_w, nu_ids, nu_w) -> float:
    a = np.asarray(mu_w, np.float64); a = a / a.sum()
    b = np.asarray(nu_w, np.float64); b = b / b.sum()
    return transport_lp(tree_metric(paths, l_root, mu_ids, nu_ids), a, b)


# --------------------------------------------------------------------------------------------
# independent brute-force recursive partitioner (SPEC.md:112 idea): geometric cells of side
# 2Φ/2^k anchored at the shifted root corner, computed per depth (not by shifting one integer)
# --------------------------------------------------------------------------------------------
def brute_tree(X, sigma, D):
    Xd = np.asarray(X, np.float64)
    if Xd.ndim == 1:
        Xd = Xd[:, None]
    N, d = Xd.shape
    mn = Xd.min(0)
    phi = float((Xd.max(0) - mn).max())
    t = Xd - mn                      # translate to [0, Φ]^d
    lower = np.asarray(sigma, np.float64) - phi   # root H = [-Φ, Φ]^d + σ

    def cells(pts, k):
        side = 2.0 * phi / (2.0 ** k)
        c = np.floor((t[pts] - lower) / side).astype(np.int64)
        return np.minimum(c, 2 ** k - 1)   # half-open cells, top face closed

    # recursive partition -> nested (points, children) with the bit-vector of each child
    def part(pts, k):
        node = {"pts": list(pts), "children": []}
        if len(pts) == 1 or k == D or phi == 0.0:
            return node
        c = cells(np.asarray(pts), k + 1)
        groups = {}
        for p, row in zip(pts, c):
            groups.setdefault(tuple(int(v) for v in row), []).append(p)
        for key in groups:
            bits = tuple(v & 1 for v in key)
            node["children"].append((bits, part(groups[key], k + 1)))
        node["children"].sort(key=lambda bc: bc[0])
        return node

    root = part(list(range(N)), 0)
    # BFS numbering: depth by depth, parents in id order, children by bit-vector
    ids, depth_of, parent_of = {}, [], []
    frontier = [(root, -1)]
    k = 0
    nid = 0
    leaf_of = {}
    paths_nodes = {}
    while frontier:
        nxt = []
        for node, par in frontier:
            ids[id(node)] = nid
            depth_of.append(k); parent_of.append(par)
            for p in node["pts"]:
                paths_nodes.setdefault(p, []).append(nid)
            if not node["children"]:
                for p in node["pts"]:
                    leaf_of[p] = nid
            for _, ch in node["children"]:
                nxt.append((ch, nid))
            nid += 1
        frontier = nxt
        k += 1
    d_star = max(len(v) for v in paths_nodes.values()) - 1
    paths = -np.ones((N, d_star + 1), np.int32)
    for p, lst in paths_nodes.items():
        paths[p, :len(lst)] = lst
    return dict(phi=phi, d_star=d_star, n_nodes=nid, paths=paths, depth=np.array(depth_of),
                parent=np.array(parent_of))


def l_root_of(phi: float) -> int:
    """ceil(log2 Φ) + 1 by exact integer search over powers of two."""
    e = 0
    while 2.0 ** e < phi:
        e += 1
    while e > -1100 and 2.0 ** (e - 1) >= phi:
        e -= 1
    return e + 1
