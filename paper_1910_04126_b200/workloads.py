"""Seeded synthetic workloads for the Flowtree hot path (BASELINE.json ``configs``).

This module holds input generators only — none of the method's arithmetic — and is the one
module shared by the CUDA path's tests/bench and by the CPU oracle.  The real
datasets of the paper (20news, Amazon reviews, MNIST with GloVe-50; Table 1)
are not available; these configs stand in for them with their shapes:

  tiny     unit scale (all 400 pairs checked)
  text     20news  (n 11,314, avg s 115.9)  -> n=10,000, s~U{20..150}, d=300
  reviews  Amazon  (n 10,000, avg s 57.44)  -> n=100,000, s~U{10..90}, d=300
  image    MNIST   (n 60,000, avg s 150.07, 28x28 grid)
  stress   scale   n=1,000,000, s~U{10..64}, 256-query batch

Recipes: a mixture point is mean + 0.3·N(0, I_d) with 64 component means
drawn N(0, I_d) and the component uniform; Zipf(1.1) is pmf ∝ r^-1.1 over ranks 1..N with rank
r -> vocab id r-1, drawn without replacement by rejecting repeats; the generator is numpy
``default_rng(seed)`` (PCG64).
"""
from __future__ import annotations

import dataclasses
import hashlib
import math

import numpy as np


@dataclasses.dataclass
class Workload:
    name: str
    X: np.ndarray          # float32 [N, d]
    doc_off: np.ndarray    # int64 [n+1]
    ids: np.ndarray        # int32 [nnz], sorted within each doc
    w: np.ndarray          # uint32 [nnz]
    q_off: np.ndarray      # int64 [nq+1]
    q_ids: np.ndarray      # int32
    q_w: np.ndarray        # uint32
    k: int
    prefilter_m: int       # 0 = exhaustive Flowtree
    max_depth: int         # depth cap D passed to the builder
    tree_seed: int

    @property
    def n(self) -> int:
        return len(self.doc_off) - 1

    @property
    def nq(self) -> int:
        return len(self.q_off) - 1

    def doc(self, i):
        a, b = int(self.doc_off[i]), int(self.doc_off[i + 1])
        return self.ids[a:b], self.w[a:b]

    def query(self, j):
        a, b = int(self.q_off[j]), int(self.q_off[j + 1])
        return self.q_ids[a:b], self.q_w[a:b]

    def fingerprint(self) -> str:
        h = hashlib.sha256()
        for a in (self.X, self.doc_off, self.ids, self.w, self.q_off, self.q_ids, self.q_w):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()[:16]

    def subset_queries(self, nq: int) -> "Workload":
        nq = min(nq, self.nq)
        e = int(self.q_off[nq])
        return dataclasses.replace(self, q_off=self.q_off[:nq + 1].copy(), q_ids=self.q_ids[:e].copy(),
                                   q_w=self.q_w[:e].copy())


CONFIGS = {
    # name: (data seed, tree seed)
    "tiny": (1, 101),
    "text": (2, 102),
    "reviews": (3, 103),
    "image": (4, 104),
    "stress": (5, 105),
}


def mixture_points(rng, N: int, d: int, n_comp: int = 64, sigma: float = 0.3) -> np.ndarray:
    means = rng.standard_normal((n_comp, d))
    comp = rng.integers(0, n_comp, size=N)
    X = means[comp] + sigma * rng.standard_normal((N, d))
    return X.astype(np.float32)


def zipf_cdf(N: int, a: float = 1.1) -> np.ndarray:
    r = np.arange(1, N + 1, dtype=np.float64)
    p = r ** (-a)
    c = np.cumsum(p)
    c /= c[-1]
    c[-1] = 1.0
    return c


def _first_unique(draws: np.ndarray, sizes: np.ndarray):
    """Per row: the first sizes[row] distinct values of the row in draw order (or None rows)."""
    order = np.argsort(draws, axis=1, kind="stable")
    sd = np.take_along_axis(draws, order, 1)
    first_sorted = np.ones_like(sd, dtype=bool)
    first_sorted[:, 1:] = sd[:, 1:] != sd[:, :-1]
    first = np.empty_like(first_sorted)
    np.put_along_axis(first, order, first_sorted, 1)
    cnt = np.cumsum(first, axis=1)
    ok = cnt[:, -1] >= sizes
    take = first & (cnt <= sizes[:, None])
    return ok, take


def sets_without_replacement(rng, sizes: np.ndarray, sampler, chunk: int = 32768):
    """Draw, for each i, a set of sizes[i] distinct ids by rejecting repeats of iid draws from
    ``sampler(rng, shape)``.  Returns (offsets int64[n+1], ids int32[sum], ids sorted per set)."""
    n = len(sizes)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(sizes)
    out = np.empty(int(off[-1]), np.int32)
    for c0 in range(0, n, chunk):
        rows = np.arange(c0, min(n, c0 + chunk))
        K = int(sizes[rows].max()) * 3 + 8
        while rows.size:
            draws = sampler(rng, (rows.size, K))
            ok, take = _first_unique(draws, sizes[rows])
            for r_local in np.nonzero(ok)[0]:
                r = rows[r_local]
                out[off[r]:off[r + 1]] = np.sort(draws[r_local][take[r_local]])
            rows = rows[~ok]
            K *= 2
    return off, out


def _zipf_sampler(cdf):
    def f(rng, shape):
        return np.minimum(np.searchsorted(cdf, rng.random(shape), side="right"), len(cdf) - 1)
    return f


def _uniform_sampler(N):
    def f(rng, shape):
        return rng.integers(0, N, size=shape)
    return f


def aspect_ratio_depth(X: np.ndarray) -> int:
    """tiny config: D = ceil(log2(aspect ratio)) + 1, aspect ratio = max / min non-zero pairwise
    Euclidean distance over X (FP64 brute force).  A workload parameter, not method arithmetic."""
    Xd = X.astype(np.float64)
    sq = (Xd * Xd).sum(1)
    best_max, best_min = 0.0, math.inf
    for i in range(0, len(Xd), 256):
        blk = Xd[i:i + 256]
        diff = blk[:, None, :] - Xd[None, :, :]
        dist = np.sqrt((diff * diff).sum(-1))
        best_max = max(best_max, float(dist.max()))
        nz = dist[dist > 0]
        if nz.size:
            best_min = min(best_min, float(nz.min()))
    del sq
    return int(math.ceil(math.log2(best_max / best_min))) + 1


def _text_like(name, seed, N, d, n, s_lo, s_hi, nq, k, prefilter_m, tree_seed, n_docs=None, n_queries=None):
    rng = np.random.default_rng(seed)
    X = mixture_points(rng, N, d)
    cdf = zipf_cdf(N)
    n = n if n_docs is None else n_docs
    nq = nq if n_queries is None else n_queries
    sizes = rng.integers(s_lo, s_hi + 1, size=n)
    doc_off, ids = sets_without_replacement(rng, sizes, _zipf_sampler(cdf))
    qsizes = rng.integers(s_lo, s_hi + 1, size=nq)
    q_off, q_ids = sets_without_replacement(rng, qsizes, _zipf_sampler(cdf))
    return Workload(name, X, doc_off, ids, np.ones(len(ids), np.uint32), q_off, q_ids,
                    np.ones(len(q_ids), np.uint32), k, prefilter_m, 32, tree_seed)


def _image_docs(rng, n):
    g = np.arange(28, dtype=np.float64)
    pi, pj = np.meshgrid(g, g, indexing="ij")
    P = np.stack([pi.ravel(), pj.ravel()], 1)                  # id = 28 i + j
    ids_all, w_all, sizes = [], [], np.zeros(n, np.int64)
    chunk = 4096
    for c0 in range(0, n, chunk):
        m = min(chunk, n - c0)
        nb = rng.integers(1, 4, size=m)                          # b ~ U{1,2,3}
        cen = rng.uniform(4.0, 23.0, size=(m, 3, 2))             # centres ~ U[4,23]^2
        sig = rng.uniform(2.0, 4.0, size=(m, 3))                 # sigma_b ~ U[2,4]
        s = rng.integers(130, 171, size=m)                       # s ~ U{130..170}
        I = np.zeros((m, 784))
        for b in range(3):
            d2 = ((P[None, :, :] - cen[:, b, None, :]) ** 2).sum(-1)
            blob = np.exp(-d2 / (2.0 * sig[:, b, None] ** 2))
            I += np.where((b < nb)[:, None], blob, 0.0)
        # top s pixels by intensity, ties by id: sort by (-I, id)
        order = np.lexsort((np.broadcast_to(np.arange(784), (m, 784)), -I), axis=-1)
        for r in range(m):
            sup = np.sort(order[r, :s[r]])
            Ir = I[r, sup]
            wr = np.clip(np.rint(255.0 * Ir / I[r].max()), 1, 255).astype(np.uint32)
            ids_all.append(sup.astype(np.int32)); w_all.append(wr)
        sizes[c0:c0 + m] = s
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(sizes)
    return off, np.concatenate(ids_all), np.concatenate(w_all), P.astype(np.float32)


def make(name: str, n_docs: int | None = None, n_queries: int | None = None) -> Workload:
    """Build a config from BASELINE.json by name, optionally with fewer docs/queries (parity
    cases use the same law at reduced n)."""
    seed, tree_seed = CONFIGS[name]
    if name == "tiny":
        rng = np.random.default_rng(seed)
        X = rng.standard_normal((1000, 8)).astype(np.float32)
        n = 100 if n_docs is None else n_docs
        nq = 4 if n_queries is None else n_queries
        doc_off, ids = sets_without_replacement(rng, np.full(n, 8), _uniform_sampler(1000))
        q_off, q_ids = sets_without_replacement(rng, np.full(nq, 8), _uniform_sampler(1000))
        D = aspect_ratio_depth(X)
        return Workload(name, X, doc_off, ids, np.ones(len(ids), np.uint32), q_off, q_ids,
                        np.ones(len(q_ids), np.uint32), 5, 0, D, tree_seed)
    if name == "text":
        return _text_like(name, seed, 50_000, 300, 10_000, 20, 150, 1000, 10, 0, tree_seed, n_docs, n_queries)
    if name == "reviews":
        return _text_like(name, seed, 100_000, 300, 100_000, 10, 90, 1000, 10, 1000, tree_seed, n_docs, n_queries)
    if name == "stress":
        return _text_like(name, seed, 100_000, 300, 1_000_000, 10, 64, 256, 10, 2000, tree_seed, n_docs, n_queries)
    if name == "image":
        rng = np.random.default_rng(seed)
        n = 60_000 if n_docs is None else n_docs
        nq = 1000 if n_queries is None else n_queries
        doc_off, ids, w, X = _image_docs(rng, n)
        q_off, q_ids, q_w, _ = _image_docs(rng, nq)
        return Workload(name, X, doc_off, ids, w, q_off, q_ids, q_w, 10, 0, 32, tree_seed)
    raise KeyError(name)
