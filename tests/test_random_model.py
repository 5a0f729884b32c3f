"""The random sphere model (§3.2 :206-223, Theorem 5).

CPU: the generator's invariants (unit norms, ε-caps, determinism) and Theorem 5's success criteria
evaluated by brute force on the ORACLE's tree (loops over points, no shared code with
`random_model.trial_success`): ε → 0 isolates every planted pair; Flowtree success is implied by
Quadtree success.  GPU: the library's criteria equal the brute-force oracle criteria on the same
trees (bit-exact paths), and its search-mode estimates over the competitor docs equal the oracle's.
"""
import numpy as np
import pytest

import oracle
from paper_1910_04126_b200 import random_model as rm


def brute_criteria(inst, T):
    """H_k by walking both paths; Quadtree: H_k holds exactly 2 points; Flowtree: no other x_j, y_j."""
    P = T.paths
    n_pts = P.shape[0]
    qt_ok = ft_ok = True
    for k in range(inst.s):
        a, b = int(inst.planted[k]), int(inst.query[k])
        t = 0
        while t + 1 < P.shape[1] and P[a, t + 1] >= 0 and P[a, t + 1] == P[b, t + 1]:
            t += 1
        cell = P[a, t]
        members = [p for p in range(n_pts) if P[p, t] == cell]
        if sorted(members) != sorted([a, b]):
            qt_ok = False
        others = set(inst.planted.tolist()) | set(inst.query.tolist())
        others -= {a, b}
        if any(m in others for m in members):
            ft_ok = False
    return qt_ok, ft_ok


def test_generator_invariants():
    inst = rm.generate_instance(300, 10, 10, 0.25, seed=5)
    X = inst.X.astype(np.float64)
    assert np.all(np.abs(np.linalg.norm(X, axis=1) - 1.0) < 1e-6)
    d = np.linalg.norm(X[inst.query] - X[inst.planted], axis=1)
    assert np.all(d <= 0.25 + 1e-6) and np.all(d > 0)
    assert len(set(inst.planted.tolist())) == 10
    again = rm.generate_instance(300, 10, 10, 0.25, seed=5)
    assert np.array_equal(inst.X, again.X) and np.array_equal(inst.planted, again.planted)
    with pytest.raises(ValueError):
        rm.generate_instance(5, 10, 10, 0.25, seed=1)


def test_cap_is_uniform_in_angle():
    """In d = 3 the cap's polar angle has CDF (1 − cos θ)/(1 − cos θmax) (Archimedes)."""
    rng = np.random.default_rng(1)
    x = np.array([0.0, 0.0, 1.0])
    eps = 0.5
    tmax = 2 * np.arcsin(eps / 2)
    th = np.array([np.arccos(np.clip(rm._cap_point(rng, x, eps) @ x, -1, 1)) for _ in range(4000)])
    qs = np.quantile(th, [0.25, 0.5, 0.75])
    expect = [np.arccos(1 - p * (1 - np.cos(tmax))) for p in (0.25, 0.5, 0.75)]
    assert np.allclose(qs, expect, atol=0.01)


def test_tiny_eps_isolates_every_pair():
    inst = rm.generate_instance(200, 10, 10, 1e-6, seed=3)
    T = oracle.Tree(inst.X, seed=11, max_depth=32)
    assert brute_criteria(inst, T) == (True, True)


@pytest.mark.parametrize("seed", range(6))
def test_flowtree_success_implied_by_quadtree(seed):
    inst = rm.generate_instance(2000, 10, 10, 0.25, seed=seed)
    T = oracle.Tree(inst.X, seed=100 + seed, max_depth=32)
    qt_ok, ft_ok = brute_criteria(inst, T)
    assert ft_ok or not qt_ok


@pytest.mark.gpu
def test_library_criteria_and_search_match_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_04126_b200 import build
    build.build()
    from paper_1910_04126_b200 import flowtree as ft
    seen = set()
    for seed in range(12):
        inst = rm.generate_instance(1500, 10, 10, 0.02, seed=seed)
        T = oracle.Tree(inst.X, seed=seed, max_depth=32)
        ix = ft.Index(inst.X, seed=seed, max_depth=32)
        assert np.array_equal(ix.paths(), T.paths)
        _, count = ix.nodes()
        got = rm.trial_success(inst, ix.paths(), count)
        assert got == brute_criteria(inst, T)
        seen.add(got)
        # search mode: the library's estimates over the competitor docs equal the oracle's
        off, ids, w = rm.competitors(inst, ix.paths(), 30, seed + 1)
        ds = ft.Dataset(ix, off, ids, w)
        q_off = np.array([0, inst.s], np.int64)
        q_ids = np.sort(inst.query).astype(np.int32)
        q_w = np.ones(inst.s, np.uint32)
        qt = ds.quadtree(q_off, q_ids, q_w)[0]
        fl = ds.flowtree(q_off, q_ids, q_w)[0]
        for dd in range(len(off) - 1):
            a = ids[off[dd]:off[dd + 1]]
            aw = w[off[dd]:off[dd + 1]]
            assert qt[dd] == T.qt(a, aw, q_ids, q_w)[1]
            ref = T.ft(a, aw, q_ids, q_w)
            assert abs(fl[dd] - ref) <= 1e-5 * abs(ref)
    assert len(seen) >= 2          # ε = 0.02 mixes successes and failures of both criteria
