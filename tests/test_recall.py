"""recall@m / pipeline-tuning harness.

CPU: the ranking arithmetic against brute force (explicit sorts of (value, id) lists), the SPEC
invariants (recall non-decreasing in m; approx = truth ⇒ recall@1 = 1; an exact last stage over
survivors holding the NN ⇒ success), on oracle rows and LP ground truth for the tiny config.
GPU: the library's exact ground truth over all docs equals the oracle's LP argmin; recall from the
library's rows equals recall from the oracle's rows; the CLI path runs end to end.
"""
import numpy as np
import pytest

import oracle
from conftest import get_workload
from paper_1910_04126_b200 import recall as R


def brute_rank(row, t):
    order = sorted(range(len(row)), key=lambda i: (row[i], i))
    return order.index(t)


def test_ranks_of_with_ties():
    rows = np.array([[3.0, 1.0, 1.0, 2.0], [0.5, 0.5, 0.5, 0.1]])
    assert R.ranks_of(rows, [2, 1]).tolist() == [1, 2]
    rng = np.random.default_rng(0)
    rows = rng.integers(0, 5, size=(20, 30)).astype(np.float64)       # many ties
    t = rng.integers(0, 30, 20)
    assert R.ranks_of(rows, t).tolist() == [brute_rank(rows[q], int(t[q])) for q in range(20)]


def test_recall_and_c1_against_brute_force():
    rng = np.random.default_rng(1)
    ranks = rng.integers(0, 50, 300)
    rec = R.recall_at(ranks, range(1, 60))
    vals = [rec[m] for m in range(1, 60)]
    assert all(a <= b for a, b in zip(vals, vals[1:])) and vals[-1] == 1.0
    for p in np.arange(0.90, 0.995, 0.01):
        c = R.c1_for_recall(ranks, p)
        assert np.mean(ranks < c) >= p - 1e-12 and (c == 1 or np.mean(ranks < c - 1) < p - 1e-12)


def test_within_ranks_against_brute_force():
    rng = np.random.default_rng(2)
    nq, n = 12, 40
    qt = rng.integers(0, 6, size=(nq, n)).astype(np.float64)
    fl = rng.integers(0, 6, size=(nq, n)).astype(np.float64)
    t = rng.integers(0, n, nq)
    c1s = [1, 3, 7, 15, 40]
    got = R.within_ranks(qt, fl, t, c1s)
    for q in range(nq):
        top_by_qt = sorted(range(n), key=lambda i: (qt[q, i], i))
        for ci, c1 in enumerate(c1s):
            S = top_by_qt[:c1]
            if int(t[q]) not in S:
                assert got[q, ci] > n
            else:
                byft = sorted(S, key=lambda i: (fl[q, i], i))
                assert got[q, ci] == byft.index(int(t[q]))


@pytest.fixture(scope="module")
def tiny_truth():
    wl = get_workload("tiny")
    T = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    qt = np.zeros((wl.nq, wl.n)); fl = np.zeros((wl.nq, wl.n)); ex = np.zeros((wl.nq, wl.n))
    for q in range(wl.nq):
        b, bw = wl.query(q)
        for d in range(wl.n):
            a, aw = wl.doc(d)
            qt[q, d] = T.qt(a, aw, b, bw)[1]
            fl[q, d] = T.ft(a, aw, b, bw)
            ex[q, d] = oracle.exact_w1(wl.X, a, aw, b, bw)
    nn = np.array([min(range(wl.n), key=lambda d: (ex[q, d], d)) for q in range(wl.nq)])
    return wl, qt, fl, ex, nn


def test_spec_invariants_on_oracle_rows(tiny_truth):
    wl, qt, fl, ex, nn = tiny_truth
    assert R.recall_at(R.ranks_of(ex, nn), [1])[1] == 1.0                  # approx = truth
    for rows in (qt, fl):
        rec = R.recall_at(R.ranks_of(rows, nn), range(1, wl.n + 1))
        v = [rec[m] for m in range(1, wl.n + 1)]
        assert all(a <= b for a, b in zip(v, v[1:])) and v[-1] == 1.0
    # the pipeline predictor: keeping every doc through both stages always succeeds, and the
    # predicted success of each (c1, c2) equals a direct simulation of the pipeline on the rows
    c1s = [1, 5, 20, wl.n]
    within = R.within_ranks(qt, fl, nn, c1s)
    assert R.pipeline_recall(None, within, 3, wl.n, 1, True) == 1.0
    for ci, c1 in enumerate(c1s):
        for c2 in (1, 2, 5, 10):
            hits = 0
            for q in range(wl.nq):
                S = sorted(range(wl.n), key=lambda d: (qt[q, d], d))[:c1]
                S2 = sorted(S, key=lambda d: (fl[q, d], d))[:c2]
                best = min(S2, key=lambda d: (ex[q, d], d))
                hits += best == nn[q]
            assert R.pipeline_recall(None, within, ci, c2, 1, True) == hits / wl.nq


@pytest.mark.gpu
def test_library_ground_truth_and_recall_match_oracle(tiny_truth):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_04126_b200 import build
    build.build()
    from paper_1910_04126_b200 import flowtree as ft
    wl, qt_o, fl_o, ex_o, nn_o = tiny_truth
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
    qt = R.rows(ds, wl.q_off, wl.q_ids, wl.q_w, "qt")
    fl = R.rows(ds, wl.q_off, wl.q_ids, wl.q_w, "ft")
    nn, w1, solved = R.exact_nn(ft, ds, wl.X, wl.doc_off, wl.ids, wl.w, wl.q_off, wl.q_ids, wl.q_w, ft_rows=fl)
    assert nn.tolist() == nn_o.tolist()
    assert np.allclose(w1[:, 0], ex_o[np.arange(wl.nq), nn_o], rtol=1e-6, atol=0)
    assert np.allclose(w1, np.sort(ex_o, axis=1)[:, :10], rtol=1e-6, atol=0)
    assert np.array_equal(qt, qt_o)
    assert R.ranks_of(qt, nn).tolist() == R.ranks_of(qt_o, nn_o).tolist()
    assert np.allclose(fl, fl_o, rtol=1e-5, atol=0)
    # reviews subset: full LP ground truth over 200 docs for 2 queries
    wl = get_workload("reviews", n_docs=200, n_queries=2)
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
    nn, w1, solved = R.exact_nn(ft, ds, wl.X, wl.doc_off, wl.ids, wl.w, wl.q_off, wl.q_ids, wl.q_w)
    for q in range(wl.nq):
        b, bw = wl.query(q)
        ex = [oracle.exact_w1(wl.X, *wl.doc(d), b, bw) for d in range(wl.n)]
        want = min(range(wl.n), key=lambda d: (ex[d], d))
        assert nn[q] == want or abs(ex[nn[q]] - ex[want]) <= 2e-6 * ex[want]
        assert abs(w1[q, 0] - ex[want]) <= 1e-6 * ex[want]


@pytest.mark.gpu
def test_recall_cli_runs_on_tiny():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = R.run_config("tiny", n_tune=2, n_eval=2, log=lambda s: None)
    rq = out["recall_eval"]["quadtree"]
    assert all(0.0 <= v <= 1.0 for v in rq.values())
    for p in out["pipelines"]:
        if p.get("feasible", True):
            assert 0.0 <= p["eval_recall"] <= 1.0
