"""recall@m and pipeline tuning on the synthetic configs, with exact ground truth from the library's
exact-W1 stage (§4.3 :381, §4.4 :402-431, App. B.2 :887-893).

* recall@m: the fraction of queries whose true nearest neighbour (smallest exact W1,
  ties to the smaller doc id) is among the top-m docs of an estimator ranked by (value, doc id).
* ground truth: `exact_nn` computes W1 with `ft_exact_w1_lists` for every doc that can still be the
  nearest — the docs whose centroid distance ‖E μ − E ν‖ (a lower bound of W1 by Jensen) does not
  exceed the exact W1 of the query's Flowtree top-8 (an upper bound) — so the answer is the exact
  argmin over all n docs.  (On the 300-d mixtures the bound prunes little and nearly every doc is
  solved; on the 2-d image grid it prunes most.)
* tuning (App. B.2 :889-891): c1 takes the 10 values giving first-stage recall
  p1 ∈ {0.90, …, 0.99} on the tuning queries; c2 runs over a lattice; a configuration is feasible
  when its predicted recall on the tuning queries reaches the target; the feasible one with the
  smallest measured GPU time wins.  Predicted recall comes from the full Quadtree and Flowtree
  rows: for a pipeline ending in the exact stage a query succeeds iff its true NN survives both
  pruning steps (the exact stage then ranks it first); a Quadtree → Flowtree pipeline with final
  count c2 succeeds iff it survives the Quadtree step and ranks < c2 by Flowtree among the c1.
  The Flowtree-insertion rule of :893 (c2 = max(10, 2·c_next)) is reported beside the tuned c2.

Estimates, ground truth and pipelines all run in the library's kernels; this module only ranks
their outputs (numpy) and times the pipeline calls (CUDA events).
"""
from __future__ import annotations

import json
import math

import numpy as np

KNN_K_MAX = 8192          # ft_knn's largest k (the selection kernels' capacity)
C2_LATTICE = (1, 2, 3, 4, 5, 6, 8, 10, 12, 15, 20, 25, 30, 40, 50, 65, 80, 100, 130, 160, 200, 250, 320, 400,
              500, 650, 800, 1000, 1300, 1600, 2000, 2500, 3200, 4000, 5000)


# ------------------------------------------------------------------------------------------------
# ranking arithmetic (host, numpy)
# ------------------------------------------------------------------------------------------------
def ranks_of(rows, target):
    """0-based position of doc target[q] in row q ordered by (value, doc id)."""
    rows = np.asarray(rows)
    target = np.asarray(target, np.int64)
    nq, n = rows.shape
    v = rows[np.arange(nq), target]
    ids = np.arange(n)[None, :]
    less = (rows < v[:, None]).sum(1)
    tie = ((rows == v[:, None]) & (ids < target[:, None])).sum(1)
    return (less + tie).astype(np.int64)


def recall_at(ranks, ms):
    """{m: fraction of queries whose true NN ranks < m}; non-decreasing in m by construction."""
    ranks = np.asarray(ranks)
    return {int(m): float(np.mean(ranks < m)) for m in ms}


def c1_for_recall(ranks, p):
    """Smallest c such that a fraction ≥ p of the queries has rank < c (App. B.2 :889)."""
    r = np.sort(np.asarray(ranks))
    need = max(1, math.ceil(p * len(r) - 1e-9))
    return int(r[need - 1]) + 1


def within_ranks(qt_rows, ft_rows, target, c1s):
    """[nq, len(c1s)]: the Flowtree rank of the true NN among the Quadtree top-c1 docs (by (value,
    id) in both), or a large sentinel when the NN is not among them."""
    qt_rows = np.asarray(qt_rows); ft_rows = np.asarray(ft_rows)
    nq, n = qt_rows.shape
    ids = np.arange(n)
    c1s = np.asarray(c1s, np.int64)
    out = np.full((nq, len(c1s)), np.iinfo(np.int64).max // 2, np.int64)
    for q in range(nq):
        t = int(target[q])
        order = np.lexsort((ids, qt_rows[q]))
        pos = np.empty(n, np.int64)
        pos[order] = ids
        ft_t = ft_rows[q, t]
        better = (ft_rows[q] < ft_t) | ((ft_rows[q] == ft_t) & (ids < t))
        bp = np.sort(pos[better])
        cnt = np.searchsorted(bp, c1s, side="left")          # better docs inside the top-c1
        ok = pos[t] < c1s
        out[q, ok] = cnt[ok]
    return out


def pipeline_recall(qt_rank, within, c1_index, c2, final_k, exact_last=True):
    """Predicted recall of QT(c1) → FT(c2) [→ Exact(final_k)] from `within_ranks` columns."""
    wr = within[:, c1_index]
    if exact_last:
        return float(np.mean(wr < c2))
    return float(np.mean(wr < final_k))


# ------------------------------------------------------------------------------------------------
# GPU: full rows, exact ground truth, timed pipelines
# ------------------------------------------------------------------------------------------------
def rows(ds, q_off, q_ids, q_w, which):
    """Full [nq, n] estimate rows on the host (Quadtree or exhaustive Flowtree)."""
    import torch
    nq = len(q_off) - 1
    out = torch.empty((nq, ds.n), dtype=torch.float64, device="cuda")
    (ds.quadtree if which == "qt" else ds.flowtree)(q_off, q_ids, q_w, out=out)
    return out.cpu().numpy()


def _means(X, off, ids, w):
    Xd = np.asarray(X, np.float64)
    off = np.asarray(off, np.int64)
    seg = np.repeat(np.arange(len(off) - 1), np.diff(off))
    wt = np.asarray(w, np.float64)
    num = np.zeros((len(off) - 1, Xd.shape[1]))
    np.add.at(num, seg, Xd[np.asarray(ids, np.int64)] * wt[:, None])
    den = np.zeros(len(off) - 1)
    np.add.at(den, seg, wt)
    return num / den[:, None]


def exact_nn(ft, ds, X, doc_off, ids, w, q_off, q_ids, q_w, ft_rows=None, ub_top=8, max_cells=1 << 24):
    """(nn id [nq], W1 [nq, ≤10] of the 10 nearest, docs solved [nq]): the exact nearest neighbour
    of each query over all n docs (column 0 of W1 is its distance).  Every doc whose centroid lower bound is ≤ the upper bound (1 + 1e-6 slack for FP32
    costs) is solved exactly with `ft_exact_w1_lists`."""
    import torch
    nq = len(q_off) - 1
    n = ds.n
    if ft_rows is None:
        ft_rows = rows(ds, q_off, q_ids, q_w, "ft")
    top = np.argsort(ft_rows, axis=1, kind="stable")[:, :ub_top]
    ub = ft.ft_exact_w1_lists(ds.h, q_off, q_ids, q_w, torch.from_numpy(top.astype(np.int64)).cuda())
    ub = ub.cpu().numpy().min(1)
    dm = _means(X, doc_off, ids, w)
    qm = _means(X, q_off, q_ids, q_w)
    nn = np.empty(nq, np.int64)
    val = np.full((nq, 10), np.inf)
    solved = np.empty(nq, np.int64)
    q_off = np.asarray(q_off, np.int64)
    per = max(1, max_cells // max(n, 1))
    for a in range(0, nq, per):
        b = min(nq, a + per)
        lb = np.sqrt(((qm[a:b, None, :] - dm[None, :, :]) ** 2).sum(-1)) if dm.shape[1] <= 8 else \
            np.sqrt(np.maximum(0.0, (qm[a:b] ** 2).sum(1)[:, None] + (dm ** 2).sum(1)[None, :]
                               - 2.0 * qm[a:b] @ dm.T))
        cand = lb <= ub[a:b, None] * (1 + 1e-6) + 1e-12
        width = int(cand.sum(1).max())
        lists = np.full((b - a, width), -1, np.int64)
        for r in range(b - a):
            c = np.nonzero(cand[r])[0]
            lists[r, :len(c)] = c
            solved[a + r] = len(c)
        lo, hi = int(q_off[a]), int(q_off[b])
        sub_off = q_off[a:b + 1] - lo
        d_lists = torch.from_numpy(lists).cuda()
        ex = ft.ft_exact_w1_lists(ds.h, sub_off, q_ids[lo:hi], q_w[lo:hi], d_lists)
        kk = min(10, width)
        ids_k, val_k = ft.ft_topk(ex, kk, ids=d_lists)
        nn[a:b] = ids_k[:, 0].cpu().numpy()
        val[a:b, :kk] = val_k.cpu().numpy()
    ds.synchronize()
    return nn, val, solved


def time_pipeline(ft, ds, q_off, q_ids, q_w, c1, c2, k, reps=3):
    """Median CUDA-event time (ms) of the QT(c1) → FT(c2) → Exact(k) pipeline on the batch, and
    its ids; c2 == k runs the two-stage QT → FT pipeline (`ft_knn`) instead."""
    import torch
    from . import pipeline
    times, ids = [], None
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if c2 == k:
            ids = torch.empty((len(q_off) - 1, k), dtype=torch.int64, device="cuda")
            val = torch.empty((len(q_off) - 1, k), dtype=torch.float64, device="cuda")
            ds.knn(q_off, q_ids, q_w, k, c1, out_ids=ids, out_val=val)
        else:
            ids, _ = pipeline.knn_qt_ft_exact(ft, ds, q_off, q_ids, q_w, c1, c2, k)
        e1.record()
        e1.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
    ids = ids.cpu().numpy() if hasattr(ids, "cpu") else np.asarray(ids)
    return float(np.median(times)), ids


def tune(ft, ds, wl, tune_q, target=0.9, final_k=1, exact_last=True, qt_rank=None, within=None,
         c1s=None, time_configs=True, reps=1):
    """App. B.2 grid search: (feasible candidates sorted by measured time, best predicted recall)."""
    res = []
    best_rec = 0.0
    for ci, c1 in enumerate(c1s):
        top = min(c1, KNN_K_MAX)
        grid = sorted({c for c in C2_LATTICE if final_k <= c < top} | {top}) if exact_last else [final_k]
        for c2 in grid:
            rec = pipeline_recall(qt_rank, within, ci, c2, final_k, exact_last)
            best_rec = max(best_rec, rec)
            if rec < target:
                continue
            row = {"c1": int(c1), "c2": int(c2), "final_k": final_k, "pred_recall": rec}
            if time_configs:
                q = wl.subset_queries(tune_q)
                ms, _ = time_pipeline(ft, ds, q.q_off, q.q_ids, q.q_w, int(c1), int(c2) if exact_last else final_k,
                                      final_k, reps)
                row["ms"] = ms
                row["ms_per_query"] = ms / tune_q
            res.append(row)
            if exact_last:
                break                    # larger c2 at this c1 is feasible too, and slower
    res.sort(key=lambda r: r.get("ms", 0.0))
    return res, best_rec


# ------------------------------------------------------------------------------------------------
# CLI: recall curves + tuned pipelines per config (results/recall_*.jsonl)
# ------------------------------------------------------------------------------------------------
def run_config(name, n_tune=300, n_eval=200, n_docs=None, ms=(1, 2, 5, 10, 20, 50, 100, 200, 500, 1000),
               log=print):
    import time
    from . import build, workloads
    build.build()
    from . import flowtree as ft
    t0 = time.time()
    wl = workloads.make(name, n_docs=n_docs, n_queries=n_tune + n_eval)
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
    qt = rows(ds, wl.q_off, wl.q_ids, wl.q_w, "qt")
    fl = rows(ds, wl.q_off, wl.q_ids, wl.q_w, "ft")
    nn, w1, solved = exact_nn(ft, ds, wl.X, wl.doc_off, wl.ids, wl.w, wl.q_off, wl.q_ids, wl.q_w, ft_rows=fl)
    t_gt = time.time() - t0
    qt_rank, ft_rank = ranks_of(qt, nn), ranks_of(fl, nn)
    tq, ev = slice(0, n_tune), slice(n_tune, n_tune + n_eval)
    out = {"config": name, "n": ds.n, "n_tune": n_tune, "n_eval": n_eval,
           "ground_truth": {"docs_solved_mean": float(solved.mean()), "seconds": round(t_gt, 1),
                            # how far the NN stands out: W1 of the 2nd / 10th nearest over the NN's
                            "w1_2nd_over_nn_median": float(np.median(w1[:, 1] / w1[:, 0])),
                            "w1_10th_over_nn_median": float(np.median(w1[:, 9] / w1[:, 0]))},
           "recall_eval": {"quadtree": recall_at(qt_rank[ev], ms), "flowtree": recall_at(ft_rank[ev], ms)}}
    log(json.dumps(out))
    c1s = [c1_for_recall(qt_rank[tq], p) for p in np.arange(0.90, 0.995, 0.01)]
    c1s = [c for c in c1s if c <= KNN_K_MAX] or [KNN_K_MAX]     # ft_knn's prefilter capacity
    within = within_ranks(qt[tq], fl[tq], nn[tq], c1s)
    within_ev = None
    results = []
    for final_k, exact_last in ((1, True), (5, False)):
        cands, best_rec = tune(ft, ds, wl, n_tune, 0.9, final_k, exact_last, qt_rank[tq], within, c1s)
        if not cands:                       # SPEC: no feasible configuration → report the best recall
            row = {"pipeline": "QT->FT->Exact" if exact_last else "QT->FT", "final_k": final_k,
                   "feasible": False, "best_pred_recall": best_rec, "c1_max": int(c1s[-1])}
            results.append(row)
            log(json.dumps({"config": name, **row}))
            continue
        best = cands[0]
        # held-out evaluation of the chosen parameters: run the pipeline on the eval queries
        q_off = wl.q_off[n_tune:] - wl.q_off[n_tune]
        lo = int(wl.q_off[n_tune])
        ms_ev, ids = time_pipeline(ft, ds, q_off, wl.q_ids[lo:], wl.q_w[lo:], best["c1"],
                                   best["c2"] if exact_last else final_k, final_k)
        hit = np.mean([nn[n_tune + r] in ids[r, :final_k] for r in range(n_eval)])
        row = {"pipeline": "QT->FT->Exact" if exact_last else "QT->FT", "final_k": final_k, "target": 0.9,
               "tuned": best, "eval_recall": float(hit), "eval_ms_per_query": ms_ev / n_eval,
               "candidates_considered": len(cands)}
        if exact_last:                      # the Flowtree-insertion rule of PAPER.md:893
            c2h = max(10, 2 * final_k)
            if within_ev is None:
                within_ev = within_ranks(qt[ev], fl[ev], nn[ev], [best["c1"]])
            ms_h, ids_h = time_pipeline(ft, ds, q_off, wl.q_ids[lo:], wl.q_w[lo:], best["c1"], c2h, final_k)
            row["insertion_rule"] = {"c2": c2h, "eval_recall": float(np.mean(
                [nn[n_tune + r] in ids_h[r, :final_k] for r in range(n_eval)])),
                "pred_eval_recall": pipeline_recall(None, within_ev, 0, c2h, final_k, True),
                "eval_ms_per_query": ms_h / n_eval}
        results.append(row)
        log(json.dumps({"config": name, **row}))
    out["pipelines"] = results
    return out



def main(argv=None):
    import argparse
    p = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    p.add_argument("--configs", default="text,reviews,image")
    p.add_argument("--tune", type=int, default=300)
    p.add_argument("--eval", type=int, default=200)
    p.add_argument("--docs", type=int, default=None)
    p.add_argument("--out", default=None)
    a = p.parse_args(argv)
    rows_out = []
    for name in a.configs.split(","):
        rows_out.append(run_config(name, a.tune, a.eval, a.docs))
    if a.out:
        with open(a.out, "w") as f:
            for r in rows_out:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
