"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars: node paths, Quadtree values, flows and prefilter ids bit-exact; Flowtree
values within 1e-5 relative (oracle 0 ⇒ GPU exactly 0); final top-k ids exact up to the tie band
(oracle values within 2·tol of a rank boundary may permute among themselves).
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

import oracle
import ft_testlib as H
from conftest import get_workload

pytestmark = pytest.mark.gpu

FT_TOL = 1e-5


@pytest.fixture(scope="module")
def ft():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_04126_b200 import build
    build.build()
    from paper_1910_04126_b200 import flowtree
    return flowtree


@pytest.fixture
def opt(ft):
    """Set library options (ft_set_option) for one test; every option is reset to 0 afterwards."""
    def set_(name, value=1):
        ft.ft_set_option(getattr(ft, name), value)
    yield set_
    for o in range(ft.FT_NUM_OPTIONS):
        ft.ft_set_option(o, 0)


_TREES = {}


def oracle_tree(wl):
    key = (wl.name, wl.X.shape, wl.tree_seed, wl.max_depth)
    if key not in _TREES:
        _TREES[key] = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    return _TREES[key]


def pmap(fn, items, workers=16):
    with cf.ThreadPoolExecutor(workers) as ex:
        return list(ex.map(fn, items))


def assert_ft_close(gpu, ref, what=""):
    gpu = np.asarray(gpu, np.float64); ref = np.asarray(ref, np.float64)
    zero = ref == 0.0
    assert np.all(gpu[zero] == 0.0), f"{what}: oracle 0 but GPU nonzero"
    rel = np.abs(gpu - ref) / np.maximum(np.abs(ref), 1e-300)
    bad = np.nonzero(~zero & (rel > FT_TOL))[0]
    assert bad.size == 0, f"{what}: {bad.size} values beyond tol, worst rel {rel[~zero].max():.3e}"


def assert_topk_tieband(gpu_ids, gpu_vals, cand_ids, cand_oracle_vals, k, tol=FT_TOL, what=""):
    """gpu top-k vs oracle ranking of the candidate set, allowing permutations inside tie bands."""
    order = sorted(range(len(cand_ids)), key=lambda i: (cand_oracle_vals[i], cand_ids[i]))
    ref_ids = [int(cand_ids[i]) for i in order][:k]
    ref_vals = [float(cand_oracle_vals[i]) for i in order][:k]
    val_of = {int(c): float(v) for c, v in zip(cand_ids, cand_oracle_vals)}
    kk = min(k, len(cand_ids))
    gids = [int(x) for x in gpu_ids[:kk]]
    assert all(g in val_of for g in gids), f"{what}: id outside the candidate set"
    assert len(set(gids)) == kk
    for r in range(kk):
        a, b = val_of[gids[r]], ref_vals[r]
        assert abs(a - b) <= 2 * tol * max(abs(a), abs(b)), f"{what}: rank {r}: {gids[r]} vs {ref_ids[r]}"
    # exact equality outside any band
    if kk == k and kk < len(cand_ids):
        boundary = ref_vals[-1]
        band = {c for c, v in val_of.items() if abs(v - boundary) <= 2 * tol * abs(boundary)}
        assert set(gids) - band == set(ref_ids) - band, f"{what}: top-k differs outside the tie band"
    for t in range(kk, k):
        assert gpu_ids[t] == -1 and np.isinf(gpu_vals[t])


# ---------------------------------------------------------------------------------------------
# a0 builder
# ---------------------------------------------------------------------------------------------
def _tree_equal(ft, X, seed=0, D=32, sigma=None):
    T = oracle.Tree(X, seed=seed, max_depth=D, sigma=sigma)
    ix = ft.Index(X, seed=seed, max_depth=D, sigma=sigma)
    assert ix.phi == T.phi and ix.l_root == T.l_root and ix.d_star == T.d_star and ix.n_nodes == T.n_nodes
    assert np.array_equal(ix.sigma(), T.sigma)
    assert np.array_equal(ix.paths(), T.paths)
    depth, count = ix.nodes()
    assert np.array_equal(depth, T.node_depth) and np.array_equal(count, T.node_count)
    return ix, T


@pytest.mark.parametrize("fname", ["appendixA_example1.json", "appendixA_example2.json"])
def test_builder_appendix(ft, fname):
    g = H.golden(fname)
    ix, _ = _tree_equal(ft, np.array(g["X"], np.float32), D=g["max_depth"], sigma=g["sigma"])
    assert ix.paths().tolist() == g["paths"]


@pytest.mark.parametrize("case", range(10))
def test_builder_random(ft, case):
    rng = np.random.default_rng(50 + case)
    N, d, D = [(1, 3, 8), (2, 1, 32), (40, 2, 4), (200, 3, 6), (65, 70, 32), (300, 8, 5), (100, 129, 32),
               (50, 1, 52), (30, 2, 1), (500, 2, 32)][case]
    if case in (3, 5):
        X = rng.integers(0, 4, size=(N, d)).astype(np.float32)     # boundaries + duplicates
    else:
        X = rng.standard_normal((N, d)).astype(np.float32)
    if case == 6:
        X[10] = X[20]
    sigma = None
    if case == 3:
        sigma = np.zeros(d)          # u reaches exactly 1: top-cell clamp
    _tree_equal(ft, X, seed=1000 + case, D=D, sigma=sigma)


def test_builder_degenerate(ft):
    _tree_equal(ft, np.ones((7, 4), np.float32), seed=3)          # Φ = 0: a lone root leaf
    _tree_equal(ft, np.zeros((1, 5), np.float32), seed=3)         # N = 1


@pytest.mark.parametrize("name", ["tiny", "image", "text", "reviews"])
def test_builder_configs(ft, name):
    wl = get_workload(name, n_docs=64, n_queries=2)
    T = oracle_tree(wl)
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    assert (ix.phi, ix.l_root, ix.d_star, ix.n_nodes) == (T.phi, T.l_root, T.d_star, T.n_nodes)
    assert np.array_equal(ix.paths(), T.paths)


# ---------------------------------------------------------------------------------------------
# a1-a7 on small configs: every pair
# ---------------------------------------------------------------------------------------------
def _setup(ft, wl):
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
    return ix, ds


def _oracle_all(T, wl, which, pairs):
    def one(p):
        qi, di = p
        a, aw = wl.doc(di)
        b, bw = wl.query(qi)
        return T.qt(a, aw, b, bw) if which == "qt" else T.ft(a, aw, b, bw)
    return pmap(one, pairs)


def test_tiny_all_pairs(ft):
    wl = get_workload("tiny")
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    qt = ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    fl = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    pairs = [(q, d) for q in range(wl.nq) for d in range(wl.n)]
    ref_qt = _oracle_all(T, wl, "qt", pairs)
    ref_ft = _oracle_all(T, wl, "ft", pairs)
    assert np.array_equal(qt.ravel(), np.array([v for _, v in ref_qt]))           # bit-exact
    assert_ft_close(fl.ravel(), ref_ft, "tiny FT")
    for q, d in pairs:                                                               # every flow, bit-exact
        b, bw = wl.query(q)
        g = ds.flow(b, bw, d)
        o = T.flow(*wl.doc(d), b, bw)
        for key in ("src", "dst", "mass", "node"):
            assert np.array_equal(g[key], o[key].astype(g[key].dtype)), (q, d, key)


@pytest.mark.parametrize("name,n_docs,nq", [("image", 1500, 6), ("text", 1100, 5), ("reviews", 2600, 8)])
def test_parity_subsets(ft, name, n_docs, nq):
    """Several CTAs' worth of docs with a ragged tail; exact QT, FT within tol, sampled flows."""
    wl = get_workload(name, n_docs=n_docs, n_queries=nq)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    qt = ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    fl = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    rng = np.random.default_rng(7)
    pairs = [(q, int(d)) for q in range(wl.nq) for d in rng.choice(wl.n, 150, replace=False)]
    pairs += [(q, wl.n - 1) for q in range(wl.nq)]
    ref_qt = _oracle_all(T, wl, "qt", pairs)
    ref_ft = _oracle_all(T, wl, "ft", pairs)
    assert np.array_equal(np.array([qt[q, d] for q, d in pairs]), np.array([v for _, v in ref_qt]))
    assert_ft_close([fl[q, d] for q, d in pairs], ref_ft, f"{name} FT")
    for q, d in pairs[:: max(1, len(pairs) // 40)]:
        b, bw = wl.query(q)
        g = ds.flow(b, bw, d)
        o = T.flow(*wl.doc(d), b, bw)
        assert np.array_equal(g["src"], o["src"]) and np.array_equal(g["dst"], o["dst"])
        assert np.array_equal(g["mass"], o["mass"]) and np.array_equal(g["node"], o["node"])


def test_doc_subset_and_self_queries(ft):
    """docs subset argument; a query equal to a doc gives exactly 0 for both estimates."""
    wl = get_workload("text", n_docs=300, n_queries=2)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    docs = np.array([5, 0, 299, 5, 17], np.int64)
    a, aw = wl.doc(4)
    b, bw = wl.doc(17)
    q_off = np.array([0, len(a), len(a) + len(b)], np.int64)
    q_ids = np.concatenate([a, b]); q_w = np.concatenate([aw, bw])
    qt = ds.quadtree(q_off, q_ids, q_w, docs=docs)
    fl = ds.flowtree(q_off, q_ids, q_w, docs=docs)
    assert fl[1, 4] == 0.0 and qt[1, 4] == 0.0
    for qi, (ids_, w_) in enumerate([(a, aw), (b, bw)]):
        for j, dd in enumerate(docs):
            assert qt[qi, j] == T.qt(*wl.doc(dd), ids_, w_)[1]
            assert_ft_close([fl[qi, j]], [T.ft(*wl.doc(dd), ids_, w_)])


def test_vocab_hash_path_matches_bitmap(ft, opt):
    """The Flowtree kernel looks query vocab up by bitmap (N ≤ 2^19) or hash (larger N); both
    must give identical values and flows (FT_OPT_VOCAB_HASH forces the hash)."""
    wl = get_workload("image", n_docs=300, n_queries=3)
    ix, ds = _setup(ft, wl)
    a = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    f_a = ds.flow(*wl.query(1), 17)
    opt("FT_OPT_VOCAB_HASH")
    b = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    f_b = ds.flow(*wl.query(1), 17)
    assert np.array_equal(a, b)
    for key in f_a:
        assert np.array_equal(f_a[key], f_b[key])


@pytest.mark.parametrize("name,n_docs,nq", [("text", 1500, 37), ("reviews", 2500, 9), ("stress", 3000, 70)])
def test_tile_major_exhaustive_table_bit_identical(ft, opt, name, n_docs, nq):
    """Exhaustive distance tables are built tile-major (every query's rows are all vocab ids, so
    consecutive work items share their A tile and skip its copy); the table entries are the same
    exact-integer distances as the query-major order (FT_OPT_DIST_QMAJOR), so every Flowtree value
    is bit-identical; and a sample against the oracle."""
    wl = get_workload(name, n_docs=n_docs, n_queries=nq)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    a = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    opt("FT_OPT_DIST_QMAJOR")
    b = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    assert np.array_equal(a, b)
    rng = np.random.default_rng(4)
    pairs = [(int(q), int(d)) for q, d in zip(rng.integers(0, wl.nq, 40), rng.integers(0, wl.n, 40))]
    ref = _oracle_all(T, wl, "ft", pairs)
    assert_ft_close([a[q, d] for q, d in pairs], ref, f"{name} tile-major FT")


@pytest.mark.parametrize("name,nq", [("text", 40), ("reviews", 70)])
def test_chunked_flowtree_matches_warp_kernel(ft, opt, name, nq):
    """Exhaustive scoring runs the lane-per-pair kernel k_ftd (pairs sharing an M-node are listed
    for the warp kernel); FT_OPT_WARP_ONLY runs the warp kernel for every pair.  The flows are the
    same triples, so the values agree to FP summation order; ragged chunks (nq not a multiple of
    32) included."""
    wl = get_workload(name, n_docs=2500, n_queries=nq)
    ix, ds = _setup(ft, wl)
    a = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    opt("FT_OPT_WARP_ONLY")
    b = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    assert np.all(np.isfinite(a))
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=0)
    assert np.array_equal(a == 0.0, b == 0.0)


@pytest.mark.parametrize("name,nq,mode", [("text", 40, "lists"), ("reviews", 70, "lists"), ("reviews", 9, "all"),
                                           ("stress", 5, "lists")])
def test_lane_per_pair_flowtree_matches_other_kernels(ft, opt, name, nq, mode):
    """The lane-per-pair kernel (k_ftd: 32 pairs of one query per warp, pairs with a common M-node
    or more than 48 shared ids listed for the warp kernel) against the warp kernel for every pair
    (FT_OPT_WARP_ONLY).  Candidate
    lists (mode "lists") hold repeats and a ragged tail, as the pipeline's top-m rows do."""
    wl = get_workload(name, n_docs=3000, n_queries=nq)
    ix, ds = _setup(ft, wl)
    docs = None
    if mode == "lists":
        rng = np.random.default_rng(5)
        docs = np.concatenate([rng.choice(wl.n, 700, replace=False), [0, wl.n - 1, 0]]).astype(np.int64)
    a = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w, docs=docs)
    opt("FT_OPT_WARP_ONLY")
    b = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w, docs=docs)
    assert np.all(np.isfinite(a))
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=0)
    assert np.array_equal(a == 0.0, b == 0.0)


@pytest.mark.parametrize("name", ["reviews", "stress", "text"])
def test_flow_export_lane_per_pair_kernel_bit_exact(ft, opt, name):
    """The flow of the kernel that scores the d = 300 pairs (k_ftd, lane per pair) exported triple by
    triple and compared bit-exact with the oracle's greedy flow (readings R8, R10):
    self matches at the leaves and the root's northwest corner.  FT_OPT_DEBUG bit 16 makes
    ft_flowtree_flow fail unless k_ftd produced the flow; the few pairs it hands to the warp kernel
    (a matching multi-point cell) are checked through the warp kernel instead."""
    wl = get_workload(name, n_docs=3000, n_queries=6)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    rng = np.random.default_rng(7)
    n_ftd = n_warp = n_self = 0
    for q in range(wl.nq):
        b, bw = wl.query(q)
        for d in rng.choice(wl.n, 25, replace=False):
            o = T.flow(*wl.doc(int(d)), b, bw)
            ft.ft_set_option(ft.FT_OPT_DEBUG, 16)
            try:
                g = ds.flow(b, bw, int(d))
                n_ftd += 1
            except ft.FlowtreeError as e:
                assert e.status == ft.FT_ESTATE, e
                ft.ft_set_option(ft.FT_OPT_DEBUG, 0)
                g = ds.flow(b, bw, int(d))
                n_warp += 1
            for key in ("src", "dst", "mass", "node"):
                assert np.array_equal(g[key], o[key].astype(g[key].dtype)), (q, int(d), key)
            n_self += int(np.sum(o["node"] != 0))
    assert n_ftd >= 0.9 * (n_ftd + n_warp), (n_ftd, n_warp)
    assert n_self > 0                                  # leaf self matches were exercised


@pytest.mark.parametrize("big", [False, True])
def test_flowtree_degenerate_and_maximum_supports(ft, big):
    """Supports at the edges of the lane-per-pair kernel's geometry, through the distance table
    (d = 300): one-point and two-point docs and queries, shared and disjoint ids, non-uniform
    weights; with big=True a 300-point doc and a 256-point query (beyond the kernel's 255-item
    limit, so the warp kernel scores every pair).  All pairs against the oracle, and as candidate
    lists with padding (-1 -> +inf) through the same path."""
    import dataclasses
    base = get_workload("reviews", n_docs=200, n_queries=2)
    rng = np.random.default_rng(17)
    N = base.X.shape[0]
    sizes = [1, 1, 2, 2, 3, 17, 64, 90, 200, 255] + ([300] if big else [])
    docs = [np.sort(rng.choice(N, s_, replace=False)).astype(np.int32) for s_ in sizes]
    docs.append(docs[0].copy())                          # a duplicate one-point doc
    docs.append(np.sort(np.concatenate([docs[2], docs[0]])).astype(np.int32))   # shares ids
    dw = [rng.integers(1, 200, len(d_)).astype(np.uint32) for d_ in docs]
    qs = [docs[0].copy(), docs[2].copy(), np.sort(rng.choice(N, 2, replace=False)).astype(np.int32),
          np.sort(np.unique(np.concatenate([docs[6][:30], rng.choice(N, 60, replace=False)]))).astype(np.int32)]
    if big:
        qs.append(np.sort(rng.choice(N, 256, replace=False)).astype(np.int32))
    qw = [rng.integers(1, 200, len(q_)).astype(np.uint32) for q_ in qs]
    qw[1] = dw[2].copy()                                 # query 1 == doc 2 exactly: FT 0
    wl = dataclasses.replace(
        base, doc_off=np.concatenate([[0], np.cumsum([len(d_) for d_ in docs])]).astype(np.int64),
        ids=np.concatenate(docs), w=np.concatenate(dw),
        q_off=np.concatenate([[0], np.cumsum([len(q_) for q_ in qs])]).astype(np.int64),
        q_ids=np.concatenate(qs), q_w=np.concatenate(qw))
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    got = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    pairs = [(q, d_) for q in range(wl.nq) for d_ in range(wl.n)]
    ref = _oracle_all(T, wl, "ft", pairs)
    assert_ft_close([got[q, d_] for q, d_ in pairs], ref, f"degenerate supports big={big}")
    assert got[1, 2] == 0.0
    import torch
    dev = torch.device("cuda:0")
    cand = np.tile(np.concatenate([np.arange(wl.n), [-1, -1, 3]]), (wl.nq, 1)).astype(np.int64)
    out = torch.empty(cand.shape, dtype=torch.float64, device=dev)
    ft.ft_flowtree_estimate_lists(ds.h, wl.q_off, torch.from_numpy(wl.q_ids).to(dev),
                                  torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32),
                                  torch.from_numpy(cand).to(dev), out)
    ds.synchronize(torch.cuda.current_stream())
    o = out.cpu().numpy()
    assert np.all(np.isinf(o[:, wl.n:wl.n + 2]))
    np.testing.assert_allclose(o[:, :wl.n], got, rtol=1e-6, atol=0)
    np.testing.assert_array_equal(o[:, wl.n + 2], got[:, 3])


@pytest.mark.parametrize("max_depth", [1, 2])
def test_lane_per_pair_flowtree_capped_tree(ft, opt, max_depth):
    """A depth cap that binds (d = 300 mixture, D = 1 or 2) puts many points into multi-point
    leaves and M-nodes: the lane-per-pair kernel must hand every pair whose flow matches at an
    M-node (or at a multi-point leaf holding a shared id) to the warp kernel and score the rest as
    leaves + root.  Against the warp kernel for every pair and, sampled, the oracle."""
    import dataclasses
    wl = dataclasses.replace(get_workload("reviews", n_docs=2000, n_queries=6), max_depth=max_depth)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    rng = np.random.default_rng(3)
    docs = rng.choice(wl.n, 600, replace=False).astype(np.int64)
    a = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w, docs=docs)
    full = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    opt("FT_OPT_WARP_ONLY")
    b = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w, docs=docs)
    fb = ds.flowtree(wl.q_off, wl.q_ids, wl.q_w)
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=0)
    np.testing.assert_allclose(full, fb, rtol=1e-6, atol=0)
    pairs = [(q, int(d)) for q in range(wl.nq) for d in rng.choice(wl.n, 25, replace=False)]
    assert_ft_close([full[q, d] for q, d in pairs], _oracle_all(T, wl, "ft", pairs), f"capped D={max_depth}")


@pytest.mark.parametrize("name", ["image", "text", "reviews"])
def test_qt_dense_matches_hash(ft, opt, name):
    """The Quadtree kernel scans a chunk with the dense bitmap structure when its node union is
    small and with the hash structure otherwise (FT_OPT_QT_HASH forces the hash); both are exact,
    so the values must be bit-identical (the oracle comparison is in the parity tests)."""
    wl = get_workload(name, n_docs=3000, n_queries=40)
    ix, ds = _setup(ft, wl)
    a = ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    opt("FT_OPT_QT_HASH")
    b = ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    assert np.array_equal(a, b)


def test_distance_table_accuracy(ft):
    """FT(δ_x, δ_y) = ||x − y|| (one triple), so single-point docs/queries expose the tensor-core
    distance table directly; compare with FP64 distances.  Error model: the table is
    the exact distance between the points quantised to 24-bit fixed point (unit 2^-e, e the largest
    exponent with max|x − mean|·2^e ≤ 2^23 − 2^16), so |D − ||x − y||| ≤ sqrt(d)·2^-e, plus ≈2^-23
    relative from the FP32 conversion and square root; ids shared by both sides are exactly 0."""
    wl = get_workload("reviews", n_docs=64, n_queries=2)
    rng = np.random.default_rng(3)
    N, d = wl.X.shape
    xs = rng.choice(N, 3000, replace=False).astype(np.int32)
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ds = ft.Dataset(ix, np.arange(len(xs) + 1, dtype=np.int64), xs, np.ones(len(xs), np.uint32))
    ys = np.concatenate([rng.choice(N, 39, replace=False), xs[:1]]).astype(np.int32)   # one shared id
    got = ds.flowtree(np.arange(len(ys) + 1, dtype=np.int64), ys, np.ones(len(ys), np.uint32))
    Xd = wl.X.astype(np.float64)
    ref = np.sqrt(((Xd[ys][:, None, :] - Xd[xs][None, :, :]) ** 2).sum(-1))
    same = ys[:, None] == xs[None, :]
    assert same.any() and np.all(got[same] == 0.0)
    M = np.abs(Xd - Xd.mean(0)).max()
    unit = 2.0 * M / ((1 << 23) - (1 << 16))          # ≥ 2^-e
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(err <= np.sqrt(d) * unit + 3e-7 * ref), (err - 3e-7 * ref).max() / unit
    rel = err[~same] / ref[~same]
    assert np.median(rel) < 5e-8, np.median(rel)
    assert rel.max() < 1e-6, rel.max()


def test_distance_table_near_pairs_and_duplicates(ft):
    """The pairs a Gram-form table gets wrong: nearest neighbours (the same mixture component,
    d² ≈ 50 against ||x̃||² + ||ỹ||² ≈ 600) and duplicated coordinates under distinct ids, in
    one- to three-point supports with non-uniform weights, through the d = 300 table path.  Every
    pair against the oracle at the 1e-5 bar; oracle 0 (identical coordinates) ⇒ GPU exactly 0."""
    base = get_workload("reviews", n_docs=64, n_queries=2)
    X = base.X.copy()
    N = len(X)
    dup_src, dup_dst = np.arange(20), N - 1 - np.arange(20)
    X[dup_dst] = X[dup_src]                                   # distinct ids, identical coordinates
    rng = np.random.default_rng(11)
    Xd = X.astype(np.float64)
    qpts = rng.choice(N - 100, 24, replace=False)
    near = []
    for y in qpts:
        d2 = ((Xd - Xd[y]) ** 2).sum(1)
        d2[y] = np.inf
        near.append(np.argsort(d2)[:12])
    docs, dws = [], []
    for y, nn in zip(qpts, near):
        for x in nn[:5]:
            docs.append([int(x)]); dws.append([1])
        docs.append([int(nn[5]), int(nn[6])]); dws.append([2, 1])
        docs.append([int(nn[7]), int(nn[8]), int(y)]); dws.append([1, 3, 2])
    for a_, b_ in zip(dup_src, dup_dst):
        docs.append([int(b_)]); dws.append([1])
    docs.append([int(v) for v in dup_dst[:3]]); dws.append([1, 1, 1])
    doc_off = np.cumsum([0] + [len(v) for v in docs]).astype(np.int64)
    ids = np.concatenate(docs).astype(np.int32)
    w = np.concatenate(dws).astype(np.uint32)
    queries = [[int(y)] for y in qpts] + [[int(y), int(nn[0])] for y, nn in zip(qpts[:8], near[:8])] + \
              [[int(v)] for v in dup_src[:5]] + [[int(v) for v in dup_src[:3]]]
    qws = [[1]] * 24 + [[2, 1]] * 8 + [[1]] * 5 + [[1, 1, 1]]
    q_off = np.cumsum([0] + [len(v) for v in queries]).astype(np.int64)
    q_ids = np.concatenate(queries).astype(np.int32)
    q_w = np.concatenate(qws).astype(np.uint32)
    ix = ft.Index(X, seed=base.tree_seed, max_depth=base.max_depth)
    ds = ft.Dataset(ix, doc_off, ids, w)
    got = ds.flowtree(q_off, q_ids, q_w)
    T = oracle.Tree(X, seed=base.tree_seed, max_depth=base.max_depth)

    def one(qd):
        qi, di = qd
        return T.ft(ids[doc_off[di]:doc_off[di + 1]], w[doc_off[di]:doc_off[di + 1]],
                    q_ids[q_off[qi]:q_off[qi + 1]], q_w[q_off[qi]:q_off[qi + 1]])
    pairs = [(qi, di) for qi in range(len(queries)) for di in range(len(docs))]
    ref = np.array(pmap(one, pairs)).reshape(len(queries), len(docs))
    assert np.sum(ref == 0.0) >= 6                              # duplicate-coordinate pairs are exact zeros
    assert_ft_close(got.ravel(), ref.ravel(), "near pairs / duplicates")


# ---------------------------------------------------------------------------------------------
# k-NN
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("prefilter_m", [0, 5, 30, 100, 1000])
def test_knn_tiny(ft, prefilter_m):
    wl = get_workload("tiny")
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    k = wl.k
    ids, vals = ds.knn(wl.q_off, wl.q_ids, wl.q_w, k, prefilter_m)
    for q in range(wl.nq):
        b, bw = wl.query(q)
        ftv = [T.ft(*wl.doc(d), b, bw) for d in range(wl.n)]
        if prefilter_m == 0 or prefilter_m >= wl.n:
            cand = list(range(wl.n))
        else:
            qtv = [T.qt(*wl.doc(d), b, bw)[1] for d in range(wl.n)]
            cand = sorted(range(wl.n), key=lambda d: (qtv[d], d))[:prefilter_m]
        assert_topk_tieband(ids[q], vals[q], cand, [ftv[c] for c in cand], k, what=f"q{q}")
        assert_ft_close(vals[q], [ftv[i] for i in ids[q]])


@pytest.mark.parametrize("name,n_docs,nq", [("reviews", 3000, 70), ("stress", 4000, 64), ("image", 800, 65),
                                           ("text", 600, 33)])
def test_quadtree_chunk_pairs_bit_identical(ft, opt, name, n_docs, nq):
    """The Quadtree scan serves 64 queries per record pass (chunk pairs: a u16 per lane packing two
    queries' node masses as bytes) when every query node mass fits a byte; otherwise, or for the odd
    last chunk, chunk by chunk.  Values bit-identical with FT_OPT_QT_PAIR_OFF, and exact against the
    oracle on sampled pairs (image: node masses ≥ 256 take the per-chunk path)."""
    wl = get_workload(name, n_docs=n_docs, n_queries=nq)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    a = ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    opt("FT_OPT_QT_PAIR_OFF")
    b = ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    assert np.array_equal(a, b)
    rng = np.random.default_rng(9)
    pairs = [(int(q), int(d)) for q, d in zip(rng.integers(0, wl.nq, 60), rng.integers(0, wl.n, 60))]
    pairs += [(wl.nq - 1, 0), (32, wl.n - 1), (63 if wl.nq > 63 else 0, 1)]
    ref = _oracle_all(T, wl, "qt", pairs)
    assert np.array_equal(np.array([a[q, d] for q, d in pairs]), np.array([v for _, v in ref]))


@pytest.mark.parametrize("n_docs,radix,unfused", [(5000, False, False), (20000, False, False), (20000, True, False),
                                                   (20000, False, True)])
def test_knn_prefilter_ids_exact(ft, opt, n_docs, radix, unfused):
    """With k = m the returned set is exactly the Quadtree top-m (bit-exact keys, ties by id),
    ordered by (Flowtree value, id) as the oracle ranks it.  n = 5000 < 32·m runs the unfused
    prefilter (values written, whole rows sorted); n = 20000 the fused sample-threshold scan with
    candidate lists (the Quadtree values at d = 300 are heavily tied), or with
    FT_OPT_PREFILTER_UNFUSED the row selection's sample-threshold path; FT_OPT_SELECT_RADIX forces
    the MSD radix kernel."""
    if radix:
        opt("FT_OPT_SELECT_RADIX")
    if unfused:
        opt("FT_OPT_PREFILTER_UNFUSED")
    wl = get_workload("reviews", n_docs=n_docs, n_queries=4)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    m = 300
    ids, vals = ds.knn(wl.q_off, wl.q_ids, wl.q_w, m, m)
    for q in range(wl.nq):
        b, bw = wl.query(q)
        qtv = pmap(lambda d: T.qt(*wl.doc(d), b, bw)[1], range(wl.n))
        top = sorted(range(wl.n), key=lambda d: (qtv[d], d))[:m]
        assert set(ids[q].tolist()) == set(top)                      # the prefilter: exact
        # and the returned order is the Flowtree ranking of that set, (value, id) ascending
        ftv = pmap(lambda d: T.ft(*wl.doc(d), b, bw), top)
        assert_topk_tieband(ids[q], vals[q], top, ftv, m, what=f"prefilter q{q}")
        v = vals[q]
        assert np.all((v[1:] > v[:-1]) | ((v[1:] == v[:-1]) & (ids[q][1:] > ids[q][:-1])))


def test_prefilter_fused_overflow_fallback(ft):
    """Fused prefilter rows whose candidate list overflows: 36,000 copies of one doc plus 2,000
    others (n = 38,000 ≥ 32·m), query 0 = that doc, so 36,000 docs tie at Quadtree value 0 and the
    list (capacity 32,768) overflows — the row is recomputed in full and selected with ties by id.
    Query 1 is an ordinary query (the list path).  Both must equal the oracle's (value, id) top-m."""
    base = get_workload("reviews", n_docs=2001, n_queries=2)
    T = oracle_tree(base)
    src = [0] * 36000 + list(range(1, 2001))
    docs = [base.doc(d) for d in src]
    doc_off = np.zeros(len(src) + 1, np.int64)
    doc_off[1:] = np.cumsum([len(i) for i, _ in docs])
    ids = np.concatenate([i for i, _ in docs]).astype(np.int32)
    w = np.concatenate([x for _, x in docs]).astype(np.uint32)
    d0i, d0w = base.doc(0)
    q1i, q1w = base.query(1)
    q_off = np.array([0, len(d0i), len(d0i) + len(q1i)], np.int64)
    q_ids = np.concatenate([d0i, q1i]).astype(np.int32)
    q_w = np.concatenate([d0w, q1w]).astype(np.uint32)
    ix = ft.Index(base.X, seed=base.tree_seed, max_depth=base.max_depth)
    ds = ft.Dataset(ix, doc_off, ids, w)
    m = 300
    got, vals = ds.knn(q_off, q_ids, q_w, m, m)
    for q, (b, bw) in enumerate([(d0i, d0w), (q1i, q1w)]):
        qd = pmap(lambda d: T.qt(*base.doc(d), b, bw)[1], range(2001))
        top = sorted(range(len(src)), key=lambda i: (qd[src[i]], i))[:m]
        assert set(got[q].tolist()) == set(top), f"query {q}"
    assert set(got[0].tolist()) == set(range(m))        # the tied copies, smallest ids first


def test_prefilter_overflow_fallback_in_a_chunk_pair(ft):
    """The same overflow inside a 64-query chunk pair (40 queries: chunks of 32 + 8 share one CTA
    row; the overflowing query is #35, in the second chunk): the fallback pass re-scans the pair's
    flagged rows only, and the ordinary rows keep their list results."""
    base = get_workload("reviews", n_docs=2001, n_queries=40)
    T = oracle_tree(base)
    src = [0] * 36000 + list(range(1, 2001))
    docs = [base.doc(d) for d in src]
    doc_off = np.zeros(len(src) + 1, np.int64)
    doc_off[1:] = np.cumsum([len(i) for i, _ in docs])
    ids = np.concatenate([i for i, _ in docs]).astype(np.int32)
    w = np.concatenate([x for _, x in docs]).astype(np.uint32)
    qs = [base.query(j) for j in range(40)]
    qs[35] = base.doc(0)
    q_off = np.zeros(41, np.int64)
    q_off[1:] = np.cumsum([len(i) for i, _ in qs])
    q_ids = np.concatenate([i for i, _ in qs]).astype(np.int32)
    q_w = np.concatenate([x for _, x in qs]).astype(np.uint32)
    ix = ft.Index(base.X, seed=base.tree_seed, max_depth=base.max_depth)
    ds = ft.Dataset(ix, doc_off, ids, w)
    m = 300
    got, vals = ds.knn(q_off, q_ids, q_w, m, m)
    for q in (0, 31, 35, 39):
        b, bw = qs[q]
        qd = pmap(lambda d: T.qt(*base.doc(d), b, bw)[1], range(2001))
        top = sorted(range(len(src)), key=lambda i: (qd[src[i]], i))[:m]
        assert set(got[q].tolist()) == set(top), f"query {q}"
    assert set(got[35].tolist()) == set(range(m))


def test_quadtree_large_supports_on_a_deep_tree_run_in_subbatches(ft):
    """32 queries with 150-255-point supports on a deep tree (d = 3, N = 20,000 uniform points:
    D* ~ 15, ~30k nodes) have a worst-case node union beyond the shared-memory hash of one chunk;
    such batches are scored in sub-batches of fewer queries per chunk (40 queries: ten sub-batches
    of 4, found by a randomised sweep — the call used to fail with a launch error).  Quadtree
    values bit-exact on sampled pairs, and the fused prefilter + Flowtree k-NN of sampled queries
    against the oracle pipeline."""
    from paper_1910_04126_b200 import workloads
    from __graft_entry__ import _ids_exact_up_to_ties
    rng = np.random.default_rng(93)
    N, n, nq = 20000, 2000, 40
    X = rng.uniform(-1.0, 1.0, size=(N, 3)).astype(np.float32)
    sampler = workloads._uniform_sampler(N)
    doc_off, ids = workloads.sets_without_replacement(rng, rng.integers(20, 256, size=n), sampler)
    q_off, q_ids = workloads.sets_without_replacement(rng, rng.integers(150, 256, size=nq), sampler)
    wl = workloads.Workload("deep", X, doc_off, ids, rng.integers(1, 8, size=len(ids)).astype(np.uint32), q_off,
                            q_ids, rng.integers(1, 8, size=len(q_ids)).astype(np.uint32), 10, 50, 32, 9093)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    _, _, d_star, M = ft.ft_index_info(ix.h)
    assert min(32 * min(255 * d_star, M), M) * 5 // 4 > 16384, "case no longer needs sub-batches"
    qt = ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    pairs = [(int(q), int(d_)) for q, d_ in zip(rng.integers(0, nq, 300), rng.integers(0, n, 300))]
    pairs += [(q, 0) for q in range(nq)]                       # every sub-batch, ragged tail included
    ref = _oracle_all(T, wl, "qt", pairs)
    for (q, d_), r in zip(pairs, ref):
        assert qt[q, d_] == r[1], (q, d_)
    gids, gvals = ds.knn(wl.q_off, wl.q_ids, wl.q_w, wl.k, wl.prefilter_m)
    for q in (0, 3, 4, 37, 39):
        b, bw = wl.query(q)
        ref_ids, ref_val = T.knn(wl.doc_off, wl.ids, wl.w, b, bw, wl.k, wl.prefilter_m)
        _ids_exact_up_to_ties(T, wl, b, bw, gids[q], gvals[q], ref_ids, ref_val)


def test_knn_padding_and_errors(ft):
    wl = get_workload("tiny", n_docs=7)
    ix, ds = _setup(ft, wl)
    ids, vals = ds.knn(wl.q_off, wl.q_ids, wl.q_w, 10, 0)
    assert np.all(ids[:, 7:] == -1) and np.all(np.isinf(vals[:, 7:]))
    with pytest.raises(ft.FlowtreeError) as e:
        ds.knn(wl.q_off, wl.q_ids, wl.q_w, 10, 5)
    assert e.value.status == ft.FT_EINVAL
    with pytest.raises(ft.FlowtreeError) as e:
        ds.quadtree(np.array([0, 2]), np.array([3, 3], np.int32), np.array([1, 1], np.uint32))
    assert e.value.status == ft.FT_EINVAL                    # duplicate id
    with pytest.raises(ft.FlowtreeError) as e:
        ds.quadtree(np.array([0, 1]), np.array([5000], np.int32), np.array([1], np.uint32))
    assert e.value.status == ft.FT_ERANGE
    with pytest.raises(ft.FlowtreeError) as e:
        ds.flowtree(np.array([0, 1]), np.array([3], np.int32), np.array([70000], np.uint32))
    assert e.value.status == ft.FT_EOVERFLOW
    with pytest.raises(ft.FlowtreeError) as e:
        ds.flowtree(np.array([0, 0]), np.array([], np.int32), np.array([], np.uint32))
    assert e.value.status == ft.FT_EINVAL                    # empty query
    with pytest.raises(ft.FlowtreeError) as e:
        ft.Dataset(ix, np.array([0, 2]), np.array([1, 1], np.int32), np.array([1, 1], np.uint32))
    assert e.value.status == ft.FT_EINVAL and "document 0" in str(e.value)
    with pytest.raises(ft.FlowtreeError) as e:
        ft.Dataset(ix, np.array([0, 1, 2]), np.array([1, 1000], np.int32), np.array([1, 1], np.uint32))
    assert e.value.status == ft.FT_ERANGE and "document 1" in str(e.value)


def test_device_pointers_async_and_sticky_error(ft):
    import torch
    wl = get_workload("tiny")
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    dev = torch.device("cuda:0")
    qi = torch.from_numpy(wl.q_ids).to(dev)
    qw = torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32)
    out = torch.empty((wl.nq, wl.n), dtype=torch.float64, device=dev)
    ds.quadtree(wl.q_off, qi, qw, out=out)
    ds.synchronize(torch.cuda.current_stream())
    host = ds.quadtree(wl.q_off, wl.q_ids, wl.q_w)
    assert np.array_equal(out.cpu().numpy(), host)
    oid = torch.empty((wl.nq, 5), dtype=torch.int64, device=dev)
    ov = torch.empty((wl.nq, 5), dtype=torch.float64, device=dev)
    ds.knn(wl.q_off, qi, qw, 5, 0, out_ids=oid, out_val=ov)
    hid, hv = ds.knn(wl.q_off, wl.q_ids, wl.q_w, 5, 0)
    torch.cuda.synchronize()
    assert np.array_equal(oid.cpu().numpy(), hid) and np.array_equal(ov.cpu().numpy(), hv)
    # a bad vocab id on the device is reported by the next ft_synchronize
    bad = qi.clone(); bad[0] = 10**6
    ds.quadtree(wl.q_off, bad, qw, out=out)
    with pytest.raises(ft.FlowtreeError) as e:
        ds.synchronize(torch.cuda.current_stream())
    assert e.value.status == ft.FT_ERANGE
    assert torch.isnan(out[0]).all()
    ds.synchronize(torch.cuda.current_stream())          # cleared


# ---------------------------------------------------------------------------------------------
# full size (BASELINE configs, the bench's launch configuration), sampled against the oracle
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,nft,nknn", [("reviews", 8, 6), ("text", 8, 4), ("image", 4, 4), ("stress", 4, 4)])
def test_full_size_sampled(ft, name, nft, nknn):
    """Every BASELINE config at its FULL size (reviews n=100k x 1,000 queries; text 10k x 1,000;
    image 60k x 1,000; stress n=1M x 256-query batch), in the launch shape the bench uses:
    Quadtree over all docs for the whole batch, bit-exact on sampled pairs; exhaustive Flowtree
    over all docs for a few queries at the 1e-5 bar on sampled pairs; and the config's k-NN
    (exhaustive, or the Quadtree prefilter for reviews/stress) against the oracle pipeline over
    all n docs for several queries, ids exact up to the R15 tie band."""
    import torch
    wl = get_workload(name)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    dev = torch.device("cuda:0")
    qi = torch.from_numpy(wl.q_ids).to(dev)
    qw = torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32)
    out = torch.empty((wl.nq, wl.n), dtype=torch.float64, device=dev)
    ds.quadtree(wl.q_off, qi, qw, out=out)
    ds.synchronize(torch.cuda.current_stream())
    rng = np.random.default_rng(11)
    qs = np.concatenate([rng.integers(0, wl.nq, 600), [wl.nq - 1, 0]])
    dd = np.concatenate([rng.integers(0, wl.n, 600), [wl.n - 1, 0]])
    got = out[torch.from_numpy(qs).to(dev), torch.from_numpy(dd).to(dev)].cpu().numpy()
    del out
    ref = _oracle_all(T, wl, "qt", list(zip(qs.tolist(), dd.tolist())))
    assert np.array_equal(got, np.array([v for _, v in ref])), f"{name} QT"
    # Flowtree over all docs for nft queries, sampled
    sub = wl.subset_queries(nft)
    fl = ds.flowtree(sub.q_off, sub.q_ids, sub.q_w)
    pairs = [(int(q), int(d)) for q, d in zip(rng.integers(0, sub.nq, 300), rng.integers(0, wl.n, 300))]
    assert_ft_close([fl[q, d] for q, d in pairs], _oracle_all(T, sub, "ft", pairs), f"{name} FT")
    # k-NN with the config's pipeline for nknn queries against the oracle over all n docs
    sub = wl.subset_queries(nknn)
    ids, vals = ds.knn(sub.q_off, sub.q_ids, sub.q_w, wl.k, wl.prefilter_m)
    for q in range(sub.nq):
        b, bw = sub.query(q)
        if wl.prefilter_m:
            qtv = pmap(lambda d: T.qt(*wl.doc(d), b, bw)[1], range(wl.n))
            cand = sorted(range(wl.n), key=lambda d: (qtv[d], d))[:wl.prefilter_m]
        else:
            cand = list(range(wl.n))
        ftv = pmap(lambda d: T.ft(*wl.doc(d), b, bw), cand)
        assert_topk_tieband(ids[q], vals[q], cand, ftv, wl.k, what=f"{name} q{q}")


# ---------------------------------------------------------------------------------------------
# doc-sharded k-NN building blocks on one GPU
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,nd,nq,k,m", [("reviews", 6000, 20, 10, 300), ("tiny", 100, 4, 5, 30)])
def test_doc_sharded_knn_matches_single_dataset(ft, name, nd, nq, k, m):
    """Two doc shards run the protocol's phases (local top-m with global ids, merge with ft_topk,
    owned Flowtree via ft_flowtree_estimate_lists with +inf elsewhere, MIN, top-k): ids and
    values bit-identical to ft_knn on the whole collection."""
    import torch
    from paper_1910_04126_b200 import parallel
    wl = get_workload(name, n_docs=nd, n_queries=nq)
    ix, ds = _setup(ft, wl)
    ref_ids, ref_vals = ds.knn(wl.q_off, wl.q_ids, wl.q_w, k, m)
    shards = []
    for r in range(2):
        off, ids, w, base = parallel.shard_docs(wl.doc_off, wl.ids, wl.w, r, 2)
        shards.append(parallel.LibShard(ft, ft.Dataset(ix, off, ids, w), base))
    loc = [sh.local_topm(wl.q_off, wl.q_ids, wl.q_w, m) for sh in shards]
    ids_all = torch.cat([l[0] for l in loc], 1)
    vals_all = torch.cat([l[1] for l in loc], 1)
    cand, _ = shards[0].topk(vals_all, ids_all, m)
    fv = torch.minimum(*[sh.score_owned(wl.q_off, wl.q_ids, wl.q_w, cand) for sh in shards])
    got_ids, got_vals = shards[0].topk(fv, cand, k)
    torch.cuda.synchronize()
    assert np.array_equal(got_ids.cpu().numpy(), ref_ids)
    assert np.array_equal(got_vals.cpu().numpy(), ref_vals)
    # a single shard through the full protocol (no process group) is ft_knn itself
    one = parallel.LibShard(ft, ds, 0)
    i1, v1 = parallel.knn_doc_sharded(one, wl.q_off, wl.q_ids, wl.q_w, k, m, None)
    assert np.array_equal(i1.cpu().numpy(), ref_ids) and np.array_equal(v1.cpu().numpy(), ref_vals)


def test_topk_entry_point(ft):
    """ft_topk against a numpy (value, id) sort, with ties, NaN and an id base."""
    import torch
    rng = np.random.default_rng(9)
    vals = rng.integers(0, 20, size=(7, 3000)).astype(np.float64)
    vals[0, 5] = np.nan
    ids = rng.permutation(7 * 3000).reshape(7, 3000).astype(np.int64)
    dv, di = torch.from_numpy(vals).cuda(), torch.from_numpy(ids).cuda()
    oi, ov = ft.ft_topk(dv, 40, ids=di)
    oi2, ov2 = ft.ft_topk(dv, 40, id_base=1000)
    torch.cuda.synchronize()
    for r in range(7):
        key = np.where(np.isnan(vals[r]), np.inf, vals[r])
        o = np.lexsort((ids[r], key))[:40]
        assert np.array_equal(oi[r].cpu().numpy(), ids[r][o])
        o2 = np.lexsort((np.arange(3000), key))[:40]
        assert np.array_equal(oi2[r].cpu().numpy(), 1000 + o2)
        assert np.array_equal(ov2[r].cpu().numpy(), vals[r][o2])


@pytest.mark.parametrize("L,k,levels", [(100000, 1500, 400), (100000, 3000, 50), (60000, 1000, 3), (9000, 700, 1000),
                                         (1000000, 2000, 300), (1000000, 2000, 40000)])
def test_topk_large_rows_rank_select(ft, L, k, levels):
    """Rows longer than the 8192-key buffer: sample threshold, gather, then the shared-memory radix
    rank-select of the k-th (value, id) when more than 2048 keys were gathered, or — when ties at
    the threshold overflow the buffer (few distinct values, as the Quadtree keys of a large
    collection) — every key below it plus the first tied keys in row order; all against numpy."""
    import torch
    rng = np.random.default_rng(L + k + levels)
    vals = rng.integers(0, levels, size=(6, L)).astype(np.float64) * 0.5 + 1.0
    vals[1] = rng.standard_normal(L)                        # no ties, negative values
    dv = torch.from_numpy(vals).cuda()
    oi, ov = ft.ft_topk(dv, k)
    oi, ov = oi.cpu().numpy(), ov.cpu().numpy()
    for r in range(6):
        o = np.lexsort((np.arange(L), vals[r]))[:k]
        assert np.array_equal(oi[r], o), r
        assert np.array_equal(ov[r], vals[r][o])


# ---------------------------------------------------------------------------------------------
# exact-W1 stage
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("start", ["greedy", "nw"])
@pytest.mark.parametrize("name,nd,nq,per_q", [("reviews", 3000, 6, 12), ("tiny", 100, 4, 10), ("text", 800, 3, 6),
                                              ("image", 300, 2, 5)])
def test_exact_w1_matches_lp(ft, name, nd, nq, per_q, start, opt):
    """Transportation simplex per (query, doc) against the oracle's exact W1 (LP, FP64 costs):
    within 1e-6 relative (FP32 costs); exact ≤ Flowtree; negative entries score +inf.  Both starting
    bases (mutual-minimum rounds, plain northwest corner) reach the same optimum; image pairs
    (170 + 170 points) take the 512-thread variant."""
    import torch
    if start == "nw":
        opt("FT_OPT_EXACT_START_NW")
    wl = get_workload(name, n_docs=nd, n_queries=nq)
    ix, ds = _setup(ft, wl)
    rng = np.random.default_rng(11)
    docs = np.stack([rng.choice(wl.n, per_q, replace=False) for _ in range(nq)]).astype(np.int64)
    docs[0, -1] = -1
    d_docs = torch.from_numpy(docs).cuda()
    ex = ft.ft_exact_w1_lists(ds.h, wl.q_off, wl.q_ids, wl.q_w, d_docs).cpu().numpy()
    fl = ft.ft_flowtree_estimate_lists(ds.h, wl.q_off, wl.q_ids, wl.q_w, d_docs).cpu().numpy()
    assert np.isinf(ex[0, -1]) and np.isinf(fl[0, -1])
    for q in range(nq):
        b, bw = wl.query(q)
        for j in range(per_q):
            d = int(docs[q, j])
            if d < 0:
                continue
            a, aw = wl.doc(d)
            ref = oracle.exact_w1(wl.X, a, aw, b, bw)
            assert abs(ex[q, j] - ref) <= 1e-6 * max(ref, 1e-12), (q, d, ex[q, j], ref)
            assert ex[q, j] <= fl[q, j] * (1 + 1e-6) + 1e-12
    ds.synchronize()


def test_exact_w1_capacity_and_degenerate(ft):
    """A pair beyond the CTA geometry (300 + 300 points) is NaN with the sticky capacity error;
    one-point sides reduce to the weighted mean distance (closed form); identical measures give 0."""
    import torch
    rng = np.random.default_rng(5)
    X = rng.standard_normal((1000, 4)).astype(np.float32)
    big = np.sort(rng.choice(1000, 300, replace=False)).astype(np.int32)
    doc_off = np.array([0, 300, 301, 304], np.int64)
    ids = np.concatenate([big, [7], [3, 9, 500]]).astype(np.int32)
    w = np.concatenate([rng.integers(1, 50, 300), [4], [1, 2, 3]]).astype(np.uint32)
    ix = ft.Index(X, seed=3, max_depth=24)
    ds = ft.Dataset(ix, doc_off, ids, w)
    # query 0: 300 points (pairs with doc 0 overflow); query 1: 3 points = doc 2
    q_off = np.array([0, 300, 303], np.int64)
    q_ids = np.concatenate([np.sort(rng.choice(1000, 300, replace=False)), [3, 9, 500]]).astype(np.int32)
    q_w = np.concatenate([rng.integers(1, 50, 300), [1, 2, 3]]).astype(np.uint32)
    docs = torch.tensor([[0, 1], [1, 2]], dtype=torch.int64).cuda()
    ex = ft.ft_exact_w1_lists(ds.h, q_off, q_ids, q_w, docs).cpu().numpy()
    assert np.isnan(ex[0, 0])
    Xd = X.astype(np.float64)
    qw = q_w[:300].astype(np.float64)
    want = float((np.linalg.norm(Xd[q_ids[:300]] - Xd[7], axis=1) * qw).sum() / qw.sum())
    assert abs(ex[0, 1] - want) <= 1e-6 * want
    want = float((np.linalg.norm(Xd[[3, 9, 500]] - Xd[7], axis=1) * [1, 2, 3]).sum() / 6)
    assert abs(ex[1, 0] - want) <= 1e-6 * want
    assert ex[1, 1] == 0.0
    with pytest.raises(ft.FlowtreeError):
        ds.synchronize()
    ds.synchronize()


def test_three_stage_pipeline_matches_oracle(ft):
    """Quadtree → Flowtree → Exact (Table 5 "424, 9, 1") against the oracle chain: the
    oracle's QT top-c1 → FT top-c2 (oracle.knn) → exact W1 by LP → smallest; the ids agree unless
    two survivors' W1 lie within the 1e-6 tolerance band."""
    from paper_1910_04126_b200 import pipeline
    wl = get_workload("reviews", n_docs=4000, n_queries=6)
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    ids, w1 = pipeline.knn_qt_ft_exact(ft, ds, wl.q_off, wl.q_ids, wl.q_w, c1=424, c2=9, k=1)
    ids, w1 = ids.cpu().numpy(), w1.cpu().numpy()
    for q in range(wl.nq):
        b, bw = wl.query(q)
        surv, _ = T.knn(wl.doc_off, wl.ids, wl.w, b, bw, 9, 424)
        ex = [oracle.exact_w1(wl.X, *wl.doc(int(d)), b, bw) for d in surv]
        order = sorted(range(len(surv)), key=lambda i: (ex[i], surv[i]))
        best = order[0]
        assert abs(w1[q, 0] - ex[best]) <= 1e-6 * ex[best]
        if ids[q, 0] != surv[best]:
            got = list(surv).index(ids[q, 0])
            assert abs(ex[got] - ex[best]) <= 2e-6 * ex[best]


def test_more_than_65535_queries(ft):
    """Query batches beyond one launch's grid.y (65,535) run in slices: the Flowtree and exact-W1
    values of queries on both sides of the boundary equal the oracle's."""
    import torch
    wl = get_workload("tiny")
    T = oracle_tree(wl)
    ix, ds = _setup(ft, wl)
    rng = np.random.default_rng(21)
    nq = 70000
    q_ids = np.sort(np.stack([rng.choice(wl.X.shape[0], 3, replace=False) for _ in range(nq)]), 1).astype(np.int32)
    q_w = rng.integers(1, 9, size=(nq, 3)).astype(np.uint32)
    q_off = np.arange(nq + 1, dtype=np.int64) * 3
    docs = np.array([0, 7, 42], np.int64)
    fl = ds.flowtree(q_off, q_ids.ravel(), q_w.ravel(), docs=docs)
    dl = torch.from_numpy(np.tile(docs, (nq, 1))).cuda()
    ex = ft.ft_exact_w1_lists(ds.h, q_off, q_ids.ravel(), q_w.ravel(), dl).cpu().numpy()
    for q in (0, 65534, 65535, 65536, nq - 1):
        for j, d in enumerate(docs):
            a, aw = wl.doc(int(d))
            ref = T.ft(a, aw, q_ids[q], q_w[q])
            assert abs(fl[q, j] - ref) <= FT_TOL * ref, (q, d)
            w1 = oracle.exact_w1(wl.X, a, aw, q_ids[q], q_w[q])
            assert abs(ex[q, j] - w1) <= 1e-6 * w1, (q, d)


def test_knn_table_chunking_invariant(ft, opt):
    """The distance tables are built per query chunk (the chunk size follows the free HBM); any
    chunking gives bit-identical k-NN ids and values (FT_OPT_TABLE_CHUNK forces ragged chunks of 3)."""
    wl = get_workload("reviews", n_docs=3000, n_queries=11)
    ix, ds = _setup(ft, wl)
    ids0, v0 = ds.knn(wl.q_off, wl.q_ids, wl.q_w, 10, 300)
    opt("FT_OPT_TABLE_CHUNK", 3)
    ids1, v1 = ds.knn(wl.q_off, wl.q_ids, wl.q_w, 10, 300)
    assert np.array_equal(ids0, ids1) and np.array_equal(v0, v1)


def test_topk_threshold_tie_blocks(ft):
    """The two tie-overflow paths of the sample-threshold selection, forced by construction
    (1M keys, k = 2000, sample threshold inside a tie block larger than the 8192-key buffer):
    block below the threshold already ≥ k (gather the keys strictly below it), and block below < k
    (all of them plus the first tied keys in row order)."""
    import torch
    rng = np.random.default_rng(77)
    L, k = 1000000, 2000
    rows = []
    for below, tie in ((3000, 6000), (500, 9500), (0, 12000)):
        v = 3.0 + rng.random(L)
        pos = rng.permutation(L)
        v[pos[:below]] = 1.0
        v[pos[below:below + tie]] = 2.0
        rows.append(v)
    vals = np.stack(rows)
    oi, ov = ft.ft_topk(torch.from_numpy(vals).cuda(), k)
    oi, ov = oi.cpu().numpy(), ov.cpu().numpy()
    for r in range(len(rows)):
        o = np.lexsort((np.arange(L), vals[r]))[:k]
        assert np.array_equal(oi[r], o), r
        assert np.array_equal(ov[r], vals[r][o])


def test_randomised_parity_sweep(ft):
    """tests/fuzz_parity.py in a fresh process: seeded random small configurations (d 1..301, N 2..5000,
    supports 1..255, unit / small / heavy weights, duplicated points, depth caps, 1..100 queries, k,
    prefilter m) against the oracle — paths and Quadtree values bit-exact, Flowtree within 1e-5, k-NN
    ids up to the tie band, overflow reported by both sides — with device memory poisoned between
    cases so that reads past an array's end see garbage.  The second range is the sequence that
    exposed k_ftd's uniform-weight merge running past the last doc's records (seed 6862)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # --directed: the documented size limits (2048-point supports at support x depth = 8192, 1000-point
    # supports through the distance table, N beyond the vocab bitmap, k = prefilter_m = 8192)
    for args in (["--seed0", "0", "--max-cases", "300"], ["--gen", "1", "--seed0", "6855", "--max-cases", "8"],
                 ["--directed"]):
        p = subprocess.run([sys.executable, os.path.join(root, "tests", "fuzz_parity.py"), "--poison", "--seconds", "150"] + args,
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0 and ", 0 failed" in p.stdout, (args, p.stdout[-3000:], p.stderr[-3000:])


def test_bounds_checked_build_runs_clean(ft):
    """compute-sanitizer is closed on this GPU pool, so the stand-in: the library rebuilt with
    FTI_CHECKED (device-side asserts on every table gather and store, the per-lane queues, the row
    maps and the staged arrays) runs the sanitizer workload (tools/sanitize_run.py: tiny, a 2,000-doc
    reviews subset through the tcgen05 distance table, k_ftd and its warp-kernel hand-over, the
    selection kernels and the exact-W1 simplex, and an image subset) in a fresh process; a failed
    device assert aborts that process."""
    import subprocess
    import sys
    from paper_1910_04126_b200 import build
    lib = build.build(checked=True)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FT_LIB=lib)
    p = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and "sanitize workload ok" in p.stdout, (p.returncode, p.stdout[-2000:], p.stderr[-4000:])
