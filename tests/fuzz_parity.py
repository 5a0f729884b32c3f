"""Randomised parity sweep on the GPU box: many small seeded configurations (dimension, ground-set
size, support sizes, weights, duplicated points, depth caps, batch sizes, k, prefilter m), each
checked against the CPU oracle — node paths and Quadtree values bit-exact, Flowtree values within
1e-5 (oracle 0 ⇒ exactly 0), k-NN ids rank by rank up to the tie band.  Test infrastructure (it
calls oracle/, so it lives under tests/); prints one line per case and a summary, exits non-zero if any case mismatched.

    python tests/fuzz_parity.py [--seconds 600] [--seed0 0]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1910_04126_b200 import flowtree as ft, workloads  # noqa: E402
from __graft_entry__ import _ids_exact_up_to_ties  # noqa: E402

FT_TOL = 1e-5
DIMS = [1, 2, 3, 8, 16, 31, 32, 33, 40, 64, 65, 100, 128, 300, 301]


def make_case(seed, gen=2):
    """gen 1: the first sweep's size lists (kept so that its seeds reproduce); gen 2 adds larger
    ground sets, doc counts, batches and supports beyond the lane-per-pair kernel's 254."""
    rng = np.random.default_rng(1_000_003 * seed + 17)
    if gen == 3:
        return make_image_like(seed, rng)
    if gen == 4:
        # paper-shaped medium cases: d = 300 mixtures, Zipf ids, odd doc counts and batch sizes
        # (ragged tiles, odd chunk pairs, several table chunks), prefiltered or exhaustive
        N = int(rng.choice([5000, 50000]))
        n = int(rng.choice([4999, 20001, 50000]))
        nq = int(rng.choice([63, 100, 257, 500]))
        s_lo, s_hi = [(10, 90), (10, 150), (1, 40)][int(rng.integers(0, 3))]
        X = workloads.mixture_points(rng, N, int(rng.choice([300, 128, 65])))
        sampler = workloads._zipf_sampler(workloads.zipf_cdf(N))
        doc_off, ids = workloads.sets_without_replacement(rng, rng.integers(s_lo, s_hi + 1, size=n), sampler)
        q_off, q_ids = workloads.sets_without_replacement(rng, rng.integers(s_lo, s_hi + 1, size=nq), sampler)
        m = int(rng.choice([100, 1000, 2000] + ([0] if n < 5000 else [])))
        return workloads.Workload(f"paper{seed}", X, doc_off, ids, np.ones(len(ids), np.uint32), q_off, q_ids,
                                  np.ones(len(q_ids), np.uint32), 10, m, 32, 6000 + seed)
    big = gen >= 2
    d = int(rng.choice(DIMS))
    N = int(rng.choice([2, 3, 17, 100, 784, 1000, 5000] + ([40000] if big else [])))
    n = int(rng.choice([1, 2, 33, 257, 1000, 3000] + ([20000] if big else [])))
    nq = int(rng.choice([1, 2, 31, 33, 65, 100] + ([300] if big else [])))
    kind = rng.integers(0, 3)
    if kind == 0:
        X = workloads.mixture_points(rng, N, d, n_comp=int(rng.integers(1, 9)))
    elif kind == 1:
        X = rng.uniform(-1.0, 1.0, size=(N, d)).astype(np.float32)
    else:
        X = rng.integers(0, 28, size=(N, d)).astype(np.float32)   # grid points, many coincide for small d
    if N >= 4 and rng.random() < 0.3:                              # exact duplicates under distinct ids
        src = rng.integers(0, N, size=max(1, N // 10))
        dst = rng.integers(0, N, size=len(src))
        X[dst] = X[src]
    s_hi = int(min(N, rng.choice([1, 2, 5, 40, 90, 150, 255] + ([254, 400] if big else []))))
    s_lo = int(rng.integers(1, s_hi + 1))
    zipf = rng.random() < 0.5 and s_hi * 20 <= N      # rejection sampling: Zipf sets must stay far below N
    sampler = workloads._zipf_sampler(workloads.zipf_cdf(N)) if zipf else workloads._uniform_sampler(N)

    def sets(count):
        sizes = rng.integers(s_lo, s_hi + 1, size=count)
        off, ids = workloads.sets_without_replacement(rng, sizes, sampler)
        wk = rng.integers(0, 3)
        if wk == 0:
            w = np.ones(len(ids), np.uint32)
        elif wk == 1:
            w = rng.integers(1, 8, size=len(ids)).astype(np.uint32)
        else:
            cap = int(rng.choice([255, 4000, 65535]))              # total mass per distribution <= cap
            w = rng.integers(1, max(1, cap // max(1, s_hi)) + 1, size=len(ids)).astype(np.uint32)
        return off, ids, w

    doc_off, ids, w = sets(n)
    q_off, q_ids, q_w = sets(nq)
    k = int(min(n, rng.choice([1, 3, 10, 20])))
    m = int(rng.choice([0, k, min(n, 2 * k + 5), min(n, 100), n]))
    if m and m < k:
        m = k
    depth = int(rng.choice([1, 2, 4, 8, 32, 32, 32]))
    return workloads.Workload(f"fuzz{seed}", X, doc_off, ids, w, q_off, q_ids, q_w, k, m, depth, 7000 + seed)


def make_image_like(seed, rng):
    """gen 3: image-like cases — a small dense grid in the plane or in R^3 (every cell of the deep
    tree is shared by many docs, so nearly every pair matches inside common multi-point cells: the
    warp kernel's per-depth northwest corners), large supports with non-uniform integer masses."""
    d = int(rng.choice([2, 2, 3]))
    side = int(rng.choice([8, 16, 28]))
    g = np.stack(np.meshgrid(*[np.arange(side)] * d, indexing="ij"), -1).reshape(-1, d).astype(np.float32)
    if len(g) > 4096:
        g = g[rng.choice(len(g), 4096, replace=False)]
    N = len(g)
    n = int(rng.choice([33, 257, 1000]))
    nq = int(rng.choice([1, 5, 33, 70]))
    s_hi = int(min(N, rng.choice([20, 150, 254, 300])))
    s_lo = int(rng.integers(1, s_hi + 1))
    sampler = workloads._uniform_sampler(N)

    def sets(count):
        off, ids = workloads.sets_without_replacement(rng, rng.integers(s_lo, s_hi + 1, size=count), sampler)
        w = rng.integers(1, max(2, 65535 // s_hi // int(rng.choice([1, 16, 200]))), size=len(ids)).astype(np.uint32)
        return off, ids, w

    doc_off, ids, w = sets(n)
    q_off, q_ids, q_w = sets(nq)
    k = int(min(n, rng.choice([1, 10])))
    m = int(rng.choice([0, min(n, 50)]))
    if m and m < k:
        m = k
    depth = int(rng.choice([2, 4, 6, 8, 32]))
    return workloads.Workload(f"img{seed}", g, doc_off, ids, w, q_off, q_ids, q_w, k, m, depth, 9000 + seed)


def make_custom(seed, d, N, n, nq, s_lo, s_hi, depth, k, m, kind="uniform"):
    """A directed case at the documented limits (see DIRECTED)."""
    rng = np.random.default_rng(77_000 + seed)
    X = (workloads.mixture_points(rng, N, d) if kind == "mixture"
         else rng.uniform(-1.0, 1.0, size=(N, d)).astype(np.float32))
    sampler = workloads._uniform_sampler(N)
    doc_off, ids = workloads.sets_without_replacement(rng, rng.integers(s_lo, s_hi + 1, size=n), sampler)
    q_off, q_ids = workloads.sets_without_replacement(rng, rng.integers(s_lo, s_hi + 1, size=nq), sampler)
    return workloads.Workload(f"directed{seed}", X, doc_off, ids, np.ones(len(ids), np.uint32), q_off, q_ids,
                              np.ones(len(q_ids), np.uint32), k, m, depth, 8000 + seed)


# the size limits include/flowtree.h documents: support 2048 (support x depth <= 8192), supports of
# 1000 through the distance table (11 column groups per query), N beyond the 2^19-id vocab bitmap
# (hash lookups; with and without a table), k = prefilter_m = 8192
DIRECTED = [
    dict(d=8, N=50000, n=40, nq=3, s_lo=1500, s_hi=2048, depth=4, k=5, m=0),
    dict(d=300, N=5000, n=60, nq=3, s_lo=700, s_hi=1000, depth=32, k=5, m=0, kind="mixture"),
    dict(d=4, N=600000, n=2000, nq=10, s_lo=5, s_hi=20, depth=32, k=10, m=100),
    dict(d=40, N=600000, n=500, nq=5, s_lo=5, s_hi=30, depth=32, k=10, m=0, kind="mixture"),
    dict(d=16, N=3000, n=9000, nq=2, s_lo=1, s_hi=4, depth=32, k=8192, m=8192),
    dict(d=300, N=2000, n=300, nq=70, s_lo=200, s_hi=254, depth=32, k=10, m=0, kind="mixture"),
]


def check_case(wl, rng):
    T = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    assert np.array_equal(ix.paths(), T.paths), "node paths"
    smax = int(max(np.diff(wl.doc_off).max(), np.diff(wl.q_off).max()))
    try:
        ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
        qt = np.asarray(ds.quadtree(wl.q_off, wl.q_ids, wl.q_w))
    except ft.FlowtreeError as e:
        if "FT_ERANGE" in str(e) and smax * max(1, ix.d_star) > 8192:
            ix.close()
            return "support x depth > 8192 rejected"      # the documented size limit (flowtree.h)
        if "FT_EOVERFLOW" not in str(e):
            raise
        # a Quadtree numerator >= 2^53 (heavy masses on a deep tree) fails the whole call: the oracle
        # must report the same overflow for at least one pair of the batch
        pairs = [(q, dd) for q in range(wl.nq) for dd in range(wl.n)]
        if len(pairs) > 400000:     # (seed 20313 of the second sweep: exactly 1 of 100,000 pairs overflows)
            pairs = [pairs[i] for i in rng.choice(len(pairs), size=400000, replace=False)]
        for q, dd in pairs:
            try:
                T.qt(*wl.doc(dd), *wl.query(q))
            except oracle.OracleError as oe:
                assert oe.code == 3, f"oracle error {oe.code}"
                ds.close()
                ix.close()
                return "both overflow"
        raise AssertionError("GPU reports FT_EOVERFLOW, the oracle does not on the sampled pairs")
    fl = np.asarray(ds.flowtree(wl.q_off, wl.q_ids, wl.q_w))
    npairs = min(200, wl.nq * wl.n)
    pq = rng.integers(0, wl.nq, size=npairs)
    pd = rng.integers(0, wl.n, size=npairs)
    for q, dd in zip(pq, pd):
        b, bw = wl.query(int(q))
        a, aw = wl.doc(int(dd))
        ref_qt = T.qt(a, aw, b, bw)[1]
        assert qt[q, dd] == ref_qt, f"Quadtree ({q},{dd}): {qt[q, dd]!r} vs {ref_qt!r}"
        ref = T.ft(a, aw, b, bw)
        g = float(fl[q, dd])
        if ref == 0.0:
            assert g == 0.0, f"Flowtree ({q},{dd}): oracle 0, gpu {g!r}"
        else:
            assert abs(g - ref) <= FT_TOL * abs(ref), f"Flowtree ({q},{dd}): {g!r} vs {ref!r}"
    # flows of a few pairs, triple by triple in canonical order (the warp kernel's export)
    for q, dd in list(zip(pq, pd))[:3]:
        b, bw = wl.query(int(q))
        g = ds.flow(b, bw, int(dd))
        o = T.flow(*wl.doc(int(dd)), b, bw)
        for key in ("src", "dst", "mass", "node"):
            assert np.array_equal(g[key], o[key].astype(g[key].dtype)), f"flow ({q},{dd}) {key}"
    # a doc subset with repeats (one list for the batch) and per-query candidate lists with -1 padding
    sub = rng.integers(0, wl.n, size=int(rng.integers(1, 70))).astype(np.int64)
    qs = np.asarray(ds.quadtree(wl.q_off, wl.q_ids, wl.q_w, docs=sub))
    fs = np.asarray(ds.flowtree(wl.q_off, wl.q_ids, wl.q_w, docs=sub))
    assert np.array_equal(qs, qt[:, sub]), "Quadtree over a doc subset differs from the all-docs values"
    np.testing.assert_allclose(fs, fl[:, sub], rtol=2e-6, atol=0, err_msg="Flowtree over a doc subset")
    L = int(rng.integers(1, 40))
    cand = rng.integers(-1, wl.n, size=(wl.nq, L)).astype(np.int64)
    dev = torch.device("cuda:0")
    out = torch.empty(cand.shape, dtype=torch.float64, device=dev)
    ft.ft_flowtree_estimate_lists(ds.h, wl.q_off, torch.from_numpy(wl.q_ids).to(dev),
                                  torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32),
                                  torch.from_numpy(cand).to(dev), out)
    ds.synchronize(torch.cuda.current_stream())
    o = out.cpu().numpy()
    pad = cand < 0
    assert np.all(np.isinf(o[pad])), "padding candidates must score +inf"
    ref = np.take_along_axis(fl, np.where(pad, 0, cand), 1)
    np.testing.assert_allclose(o[~pad], ref[~pad], rtol=2e-6, atol=0, err_msg="Flowtree over candidate lists")
    # exact W1 (transportation simplex) on small supports against the oracle's LP
    if smax <= 40:
        nqe = min(4, wl.nq)
        ed = rng.integers(0, wl.n, size=(wl.nq, 3)).astype(np.int64)
        ex = ft.ft_exact_w1_lists(ds.h, wl.q_off, wl.q_ids, wl.q_w, torch.from_numpy(ed).to(dev)).cpu().numpy()
        for q in range(nqe):
            b, bw = wl.query(q)
            for jx in range(3):
                a_, aw_ = wl.doc(int(ed[q, jx]))
                ref_w1 = oracle.exact_w1(wl.X, a_, aw_, b, bw)
                g = float(ex[q, jx])
                assert abs(g - ref_w1) <= 1e-6 * ref_w1 + 1e-12 * (ref_w1 == 0.0) or (ref_w1 == 0.0 and g == 0.0), \
                    f"exact W1 ({q},{int(ed[q, jx])}): {g!r} vs {ref_w1!r}"
                assert g <= float(fl[q, ed[q, jx]]) * (1 + 1e-6) + 1e-12, "exact W1 above Flowtree"
    # ft_topk on a tie-heavy random matrix against numpy's (value, id) order
    R, Lk = int(rng.integers(1, 6)), int(rng.choice([1, 7, 300, 5000, 40000]))
    kk = int(min(Lk, rng.choice([1, 5, 64, 1000])))
    tv = rng.integers(0, int(rng.choice([2, 50, 100000])), size=(R, Lk)).astype(np.float64)
    oi, ov = ft.ft_topk(torch.from_numpy(tv).to(dev), kk, id_base=5)
    torch.cuda.synchronize()
    for r in range(R):
        o_ = np.lexsort((np.arange(Lk), tv[r]))[:kk]
        assert np.array_equal(oi[r].cpu().numpy(), 5 + o_) and np.array_equal(ov[r].cpu().numpy(), tv[r][o_]), "ft_topk"
    ids, vals = ds.knn(wl.q_off, wl.q_ids, wl.q_w, wl.k, wl.prefilter_m)
    ids, vals = np.asarray(ids), np.asarray(vals)
    for q in rng.choice(wl.nq, size=min(4, wl.nq), replace=False):
        b, bw = wl.query(int(q))
        ref_ids, ref_val = T.knn(wl.doc_off, wl.ids, wl.w, b, bw, wl.k, wl.prefilter_m)
        _ids_exact_up_to_ties(T, wl, b, bw, ids[q], vals[q], ref_ids, ref_val)
    ds.close()
    ix.close()
    return "ok"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600.0)
    ap.add_argument("--seed0", type=int, default=0)
    ap.add_argument("--max-cases", type=int, default=100000)
    ap.add_argument("--poison", action="store_true",
                    help="before each case fill and release 1 GiB of device memory with a non-zero pattern, so "
                         "a kernel that reads scratch it never wrote sees garbage instead of a fresh process's zeros")
    ap.add_argument("--opt", action="append", default=[], help="library option NAME=VALUE (e.g. FT_OPT_WARP_ONLY=1)")
    ap.add_argument("--random-opts", action="store_true",
                    help="per case, switch a random subset of the library's alternative code paths on (hash lookups, "
                         "warp kernel only, radix selection, unfused prefilter, single-chunk Quadtree scan, query-major "
                         "tables, small table chunks): every path must agree with the oracle")
    ap.add_argument("--directed", action="store_true", help="run the DIRECTED limit cases instead of the random sweep")
    ap.add_argument("--gen", type=int, default=2, help="case generator version (1: the first sweep's size lists)")
    ap.add_argument("--only", type=int, default=None, help="run this one seed (to reproduce a failure)")
    a = ap.parse_args()
    import torch
    assert torch.cuda.is_available(), "fuzz_parity needs a GPU"
    for o in a.opt:
        name, val = o.split("=")
        ft.ft_set_option(getattr(ft, name), int(val))
    t0 = time.time()
    done = 0
    fails = 0
    seed = a.seed0
    if a.only is not None:
        seed, a.max_cases = a.only, 1
    if a.directed:
        a.max_cases, seed, a.seconds = len(DIRECTED), 0, 1e9
    while time.time() - t0 < a.seconds and done + fails < a.max_cases:
        wl = make_custom(seed, **DIRECTED[seed]) if a.directed else make_case(seed, a.gen)
        optdesc = ""
        if a.random_opts:
            orng = np.random.default_rng(555 + seed)
            for o in range(ft.FT_NUM_OPTIONS):
                ft.ft_set_option(o, 0)
            for name, val in (("FT_OPT_VOCAB_HASH", 1), ("FT_OPT_WARP_ONLY", 1), ("FT_OPT_QT_HASH", 1),
                              ("FT_OPT_SELECT_RADIX", 1), ("FT_OPT_PREFILTER_UNFUSED", 1), ("FT_OPT_QT_PAIR_OFF", 1),
                              ("FT_OPT_DIST_QMAJOR", 1), ("FT_OPT_TABLE_CHUNK", int(orng.integers(1, 40))),
                              ("FT_OPT_EXACT_START_NW", 1), ("FT_OPT_QT_WAVES", int(orng.integers(1, 17)))):
                if orng.random() < 0.3:
                    ft.ft_set_option(getattr(ft, name), val)
                    optdesc += f" {name[7:]}={val}"
        if a.poison:
            pat = [-1, 0x7F7F7F7F, 0x00FFFF00, 12345678][seed % 4]
            for _ in range(2):
                t = torch.full((128 << 20,), pat, dtype=torch.int32, device="cuda")
                torch.cuda.synchronize()
                del t
                torch.cuda.empty_cache()
        desc = (f"seed {seed}: d={wl.X.shape[1]} N={wl.X.shape[0]} n={wl.n} nq={wl.nq} nnz={len(wl.ids)} "
                f"k={wl.k} m={wl.prefilter_m} D={wl.max_depth} wmax={int(wl.w.max())}{optdesc}")
        try:
            res = check_case(wl, np.random.default_rng(seed))
        except Exception as e:  # noqa: BLE001
            print(f"FAIL {desc}: {type(e).__name__}: {e}", flush=True)
            fails += 1
            if fails >= 10 or "CUDA" in str(e).upper():
                raise SystemExit(1)
            seed += 1
            continue
        print(f"ok   {desc}" + ("" if res == "ok" else f"  [{res}]"), flush=True)
        done += 1
        seed += 1
    print(f"fuzz_parity: {done} cases ok, {fails} failed in {time.time() - t0:.0f} s (seeds {a.seed0}..{seed - 1})")
    if fails:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
