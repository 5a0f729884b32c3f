"""Pins of the CPU oracle to things other than itself.  CPU only.

Every test here compares the oracle against: values hand-worked from the paper's rules
(tests/golden, with citations), published reference vectors, an LP, an exhaustive enumeration,
an independent recursive partitioner, a 1-D CDF closed form, or invariants the paper states.
"""
import itertools

import numpy as np
import pytest
from hypothesis import given, settings, HealthCheck
from hypothesis import strategies as st

import oracle
import ft_testlib as H


# ---------------------------------------------------------------------------------------------
# O2: SplitMix64 reference vector
# ---------------------------------------------------------------------------------------------
def test_splitmix64_reference_vector():
    g = H.golden("splitmix64.json")
    got = [oracle.splitmix64(g["seed"], i) for i in range(len(g["outputs"]))]
    assert got == [int(v) for v in g["outputs"]]


def test_sigma_from_seed_golden():
    """O2's seed → σ mapping pinned to σ computed by hand from the PUBLISHED SplitMix64 outputs
    (tests/golden/sigma_from_seed.json, exact rational arithmetic, reading R3).  A
    wrong shift (z >> 12), scale, or output index fails it."""
    g = H.golden("sigma_from_seed.json")
    for c in g["cases"]:
        X = np.zeros((2, g["d"]), np.float32)
        X[1, :] = np.float32(c["phi_f32"])
        T = oracle.Tree(X, seed=g["seed"], max_depth=8)
        assert T.phi == float.fromhex(c["phi"])
        assert [float(v) for v in T.sigma] == [float.fromhex(h) for h in c["sigma"]], c["phi_f32"]


def test_sigma_in_range_and_deterministic():
    X = np.random.default_rng(0).standard_normal((50, 7)).astype(np.float32)
    a = oracle.Tree(X, seed=99)
    b = oracle.Tree(X, seed=99)
    assert np.array_equal(a.sigma, b.sigma) and np.array_equal(a.paths, b.paths)
    assert np.all(a.sigma >= 0) and np.all(a.sigma < a.phi)            # σ_i uniform in [0, Φ]
    assert not np.array_equal(a.sigma, oracle.Tree(X, seed=100).sigma)


# ---------------------------------------------------------------------------------------------
# Appendix A hand-worked examples (golden)
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("fname", ["appendixA_example1.json", "appendixA_example2.json"])
def test_appendix_examples(fname):
    g = H.golden(fname)
    X = np.array(g["X"], np.float32)
    T = oracle.Tree(X, sigma=g["sigma"], max_depth=g["max_depth"])
    assert T.phi == g["phi"] and T.l_root == g["l_root"] and T.d_star == g["d_star"]
    assert T.n_nodes == g["n_nodes"]
    assert T.paths.tolist() == g["paths"]
    for c in g["cases"]:
        mi, mw = zip(*c["mu"]); ni, nw = zip(*c["nu"])
        f = T.flow(mi, mw, ni, nw)
        got = [[int(s), int(d), int(m), int(v)] for s, d, m, v in zip(f["src"], f["dst"], f["mass"], f["node"])]
        assert got == c["flow"], c["name"]
        assert T.ft(mi, mw, ni, nw) == c["ft"], c["name"]
        num, val = T.qt(mi, mw, ni, nw)
        assert num == c["qt_num"] and val == c["qt"], c["name"]
        # exact W1 of the hand example, by LP: pins the golden w1 column and Flowtree >= W1
        assert abs(H.exact_w1(X, mi, mw, ni, nw) - c["w1"]) < 1e-9
        assert c["ft"] >= c["w1"] - 1e-12


def test_spec_micro_examples():
    g = H.golden("spec_micro.json")
    T = oracle.Tree(np.array(g["single_point"]["X"], np.float32), seed=3)
    assert T.n_nodes == g["single_point"]["n_nodes"] and T.d_star == g["single_point"]["d_star"]
    T = oracle.Tree(np.array(g["two_points_1d"]["X"], np.float32), seed=5)
    leaves = {int(p[p >= 0][-1]) for p in T.paths}
    assert len(leaves) == g["two_points_1d"]["n_leaves"] and T.d_star >= 1
    dp = g["delta_pair"]
    T = oracle.Tree(np.array(dp["X"], np.float32), seed=11)
    assert T.ft([0], [1], [1], [1]) == dp["ft"]
    f = T.flow([0], [1], [1], [1])
    assert [[int(f["src"][0]), int(f["dst"][0]), int(f["mass"][0])]] == dp["flow"]
    assert T.ft([0, 1], [3, 5], [0, 1], [3, 5]) == 0.0
    e = g["exact_w1_1d"]
    mi, mw = zip(*e["mu"]); ni, nw = zip(*e["nu"])
    assert abs(H.exact_w1(np.array(e["X"]), mi, mw, ni, nw) - e["w1"]) < 1e-12
    q = g["qt_level1_split"]
    T = oracle.Tree(np.array(q["X"], np.float32), sigma=q["sigma"])
    assert T.qt([0], [1], [1], [1])[1] == q["qt"]


# ---------------------------------------------------------------------------------------------
# O1-O5 vs the independent recursive partitioner
# ---------------------------------------------------------------------------------------------
def _check_tree_vs_brute(X, sigma, D):
    T = oracle.Tree(X, sigma=sigma, max_depth=D)
    B = H.brute_tree(X, sigma, D)
    assert T.phi == B["phi"]
    assert T.n_nodes == B["n_nodes"]
    assert T.d_star == B["d_star"]
    assert np.array_equal(T.paths, B["paths"])
    assert np.array_equal(T.node_depth, B["depth"])
    assert np.array_equal(T.node_parent, B["parent"])
    if T.phi > 0:
        assert T.l_root == H.l_root_of(T.phi)
    return T


@pytest.mark.parametrize("seed", range(6))
def test_tree_matches_bruteforce_partitioner(seed):
    rng = np.random.default_rng(seed)
    N, d = [(30, 1), (40, 2), (60, 3), (25, 5), (80, 2), (12, 8)][seed]
    X = rng.standard_normal((N, d)).astype(np.float32)
    if seed % 2:
        X[3] = X[7]                       # duplicate coordinates share a depth-D leaf
    Xd = X.astype(np.float64)
    phi = float((Xd.max(0) - Xd.min(0)).max())
    sigma = rng.uniform(0, phi, size=d)
    for D in (2, 4, 32):
        T = _check_tree_vs_brute(X, sigma, D)
        assert T.d_star <= D
        if D == 32 and seed % 2 == 0:
            # no duplicates, cap not binding: exactly |X| leaves
            leaves = {int(p[p >= 0][-1]) for p in T.paths}
            assert len(leaves) == N


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(1, 30), st.integers(1, 3), st.integers(1, 6), st.integers(0, 2**32 - 1), st.booleans())
def test_tree_bruteforce_hypothesis(N, d, D, seed, grid):
    rng = np.random.default_rng(seed)
    if grid:   # integer grid points: many points on cell boundaries and duplicates
        X = rng.integers(0, 4, size=(N, d)).astype(np.float32)
    else:
        X = rng.standard_normal((N, d)).astype(np.float32)
    Xd = X.astype(np.float64)
    phi = float((Xd.max(0) - Xd.min(0)).max())
    sigma = rng.uniform(0, phi, size=d) if phi > 0 else np.zeros(d)
    if grid and seed % 3 == 0:
        sigma = np.zeros(d)   # boundary case: u can reach exactly 1 (top cell clamp)
    _check_tree_vs_brute(X, sigma, D)


# ---------------------------------------------------------------------------------------------
# O6-O9 on tiny random instances: LP, brute force, invariants
# ---------------------------------------------------------------------------------------------
def _rand_instance(rng, N=12, d=2, D=3, smax=5, wmax=4):
    X = rng.standard_normal((N, d)).astype(np.float32)
    T = oracle.Tree(X, seed=int(rng.integers(1 << 30)), max_depth=D)
    sa, sb = np.minimum(rng.integers(1, smax + 1, size=2), N)
    a = rng.choice(N, sa, replace=False); b = rng.choice(N, sb, replace=False)
    aw = rng.integers(1, wmax + 1, size=sa); bw = rng.integers(1, wmax + 1, size=sb)
    return X, T, a, aw, b, bw


def _check_pair(X, T, a, aw, b, bw):
    W, U = int(aw.sum()), int(bw.sum())
    f = T.flow(a, aw, b, bw)
    assert f["W"] == W and f["U"] == U
    # marginals (exact integers): Σ_dst f(x,·) = w_x·U, Σ_src f(·,y) = u_y·W
    for x, wx in zip(a, aw):
        assert int(f["mass"][f["src"] == x].sum()) == int(wx) * U
    for y, uy in zip(b, bw):
        assert int(f["mass"][f["dst"] == y].sum()) == int(uy) * W
    # support bound: ≤ s_μ + s_ν − 1 triples (PAPER.md:512 gives ≤ 2s)
    assert len(f["src"]) <= len(a) + len(b) - 1
    # each (src, dst) pair at most once
    assert len(set(zip(f["src"].tolist(), f["dst"].tolist()))) == len(f["src"])
    # tree cost of the flow == QT numerator, exactly in integers (fact 3 of SURVEY §8(a))
    num, qt = T.qt(a, aw, b, bw)
    tm = H.tree_metric(T.paths, T.d_star, f["src"], f["dst"])      # ω-weights: l_root := D*
    cost_int = sum(int(m) * int(round(tm[i, i])) for i, m in enumerate(f["mass"]))
    assert cost_int == num
    # QT value == tree-metric W1 computed by LP
    lp = H.tree_w1_lp(T.paths, T.l_root, a, aw, b, bw)
    assert abs(qt - lp) <= 1e-9 * max(1.0, lp)
    # the greedy flow is tree-optimal: its tree cost equals the LP optimum
    tm_true = H.tree_metric(T.paths, T.l_root, f["src"], f["dst"])
    tree_cost = sum(float(m) * tm_true[i, i] for i, m in enumerate(f["mass"])) / (W * U)
    assert abs(tree_cost - lp) <= 1e-9 * max(1.0, lp)
    # fact 2: the amount matched at node v is min(mμ(v), mν(v)) − Σ_children min(...)
    _check_matched_per_node(T, a, aw * U, b, bw * W, f)
    # Flowtree >= exact W1 (the tree flow is feasible for Eq. (1))
    ft = T.ft(a, aw, b, bw)
    w1 = H.exact_w1(X, a, aw, b, bw)
    assert ft >= w1 - 1e-9 * max(1.0, w1)
    # swap symmetry: the flow transposes (same emission order), value identical
    g = T.flow(b, bw, a, aw)
    assert np.array_equal(g["src"], f["dst"]) and np.array_equal(g["dst"], f["src"])
    assert np.array_equal(g["mass"], f["mass"])
    assert T.ft(b, bw, a, aw) == ft
    return ft, w1


def _check_matched_per_node(T, a, ma, b, mb, f):
    def node_mass(ids, m):
        out = {}
        for x, mx in zip(ids, m):
            for v in T.paths[x]:
                if v >= 0:
                    out[int(v)] = out.get(int(v), 0) + int(mx)
        return out
    A, B = node_mass(a, ma), node_mass(b, mb)
    children = {}
    for v in range(T.n_nodes):
        p = int(T.node_parent[v])
        if p >= 0:
            children.setdefault(p, []).append(v)
    matched = {}
    for m, v in zip(f["mass"], f["node"]):
        matched[int(v)] = matched.get(int(v), 0) + int(m)
    for v in set(A) | set(B):
        expect = min(A.get(v, 0), B.get(v, 0)) - sum(min(A.get(c, 0), B.get(c, 0)) for c in children.get(v, []))
        assert matched.get(v, 0) == expect


@pytest.mark.parametrize("seed", range(25))
def test_pair_invariants_random(seed):
    rng = np.random.default_rng(1000 + seed)
    X, T, a, aw, b, bw = _rand_instance(rng, N=14, d=1 + seed % 3, D=2 + seed % 4)
    _check_pair(X, T, a, aw, b, bw)


@settings(max_examples=30, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(0, 2**32 - 1))
def test_pair_invariants_hypothesis(seed):
    rng = np.random.default_rng(seed)
    X, T, a, aw, b, bw = _rand_instance(rng, N=int(rng.integers(2, 16)), d=int(rng.integers(1, 4)),
                                        D=int(rng.integers(1, 6)), smax=6, wmax=5)
    _check_pair(X, T, a, aw, b, bw)


def test_identity_flow_and_zero():
    rng = np.random.default_rng(7)
    X, T, a, aw, _, _ = _rand_instance(rng, N=20, d=3, D=4, smax=6)
    f = T.flow(a, aw, a, aw)
    W = int(aw.sum())
    assert np.array_equal(f["src"], f["dst"])                          # SPEC.md:172 identity
    assert sorted(zip(f["src"].tolist(), f["mass"].tolist())) == sorted(zip(a.tolist(), (aw * W).tolist()))
    assert T.ft(a, aw, a, aw) == 0.0 and T.qt(a, aw, a, aw) == (0, 0.0)


def test_birkhoff_bruteforce_tiny(tiny):
    """Uniform s=8 on the tiny config: exact W1 by all 8! permutations; LP agrees; FT >= W1."""
    T = oracle.Tree(tiny.X, seed=tiny.tree_seed, max_depth=tiny.max_depth)
    for qi in range(2):
        b, bw = tiny.query(qi)
        for di in range(3):
            a, aw = tiny.doc(di)
            bf = H.birkhoff_w1(tiny.X, a, b)
            assert abs(bf - H.exact_w1(tiny.X, a, aw, b, bw)) < 1e-9
            assert T.ft(a, aw, b, bw) >= bf - 1e-12


def test_exact_w1_1d_cdf():
    rng = np.random.default_rng(5)
    for _ in range(10):
        X = np.sort(rng.uniform(0, 10, size=9)).astype(np.float32)[:, None]
        a = rng.choice(9, 4, replace=False); b = rng.choice(9, 3, replace=False)
        aw = rng.integers(1, 5, size=4); bw = rng.integers(1, 5, size=3)
        cdf = H.w1_1d_cdf(X[a, 0], aw, X[b, 0], bw)
        assert abs(cdf - H.exact_w1(X, a, aw, b, bw)) < 1e-9


def test_oracle_exact_w1_pins(tiny):
    """O11 (oracle.exact_w1) against the Birkhoff permutation brute force (uniform s = 8 on the
    tiny config) and the 1-D CDF closed form with integer weights; never above Flowtree."""
    T = oracle.Tree(tiny.X, seed=tiny.tree_seed, max_depth=tiny.max_depth)
    for qi in range(2):
        b, bw = tiny.query(qi)
        for di in range(3):
            a, aw = tiny.doc(di)
            w1 = oracle.exact_w1(tiny.X, a, aw, b, bw)
            assert abs(w1 - H.birkhoff_w1(tiny.X, a, b)) < 1e-9
            assert T.ft(a, aw, b, bw) >= w1 - 1e-12
    rng = np.random.default_rng(17)
    for _ in range(10):
        X = np.sort(rng.uniform(0, 10, size=9)).astype(np.float32)[:, None]
        a = rng.choice(9, 4, replace=False); b = rng.choice(9, 3, replace=False)
        aw = rng.integers(1, 5, size=4); bw = rng.integers(1, 5, size=3)
        assert abs(H.w1_1d_cdf(X[a, 0], aw, X[b, 0], bw) - oracle.exact_w1(X, a, aw, b, bw)) < 1e-9


def test_flowtree_equals_w1_when_pairs_isolated():
    """Random-model special case: if the smallest cell containing x_k also
    contains y_k and no other support point, the tree flow is the planted perfect matching and
    Flowtree = W1."""
    rng = np.random.default_rng(3)
    s = 6
    # Φ = 64 and σ = 0 align the depth-4 grid with multiples of 8: cell [8j, 8j+8) holds only the
    # planted pair (x_j, y_j); two extra non-support points pin the range to [0, 64].
    xs = 8.0 * np.arange(1, s + 1) + 1.0
    ys = xs + rng.uniform(0.5, 5.0, size=s)
    X = np.concatenate([xs, ys, [0.0, 64.0]]).astype(np.float32)[:, None]
    T = oracle.Tree(X, sigma=[0.0], max_depth=32)
    assert T.phi == 64.0
    a = np.arange(s); b = np.arange(s, 2 * s)
    f = T.flow(a, np.ones(s), b, np.ones(s))
    assert sorted(zip(f["src"].tolist(), f["dst"].tolist())) == [(k, s + k) for k in range(s)]
    ft = T.ft(a, np.ones(s), b, np.ones(s))
    assert abs(ft - H.exact_w1(X, a, np.ones(s), b, np.ones(s))) < 1e-9
    assert abs(ft - float(np.mean(X[b, 0].astype(np.float64) - X[a, 0].astype(np.float64)))) < 1e-12


def test_errors():
    T = oracle.Tree(np.zeros((3, 2), np.float32) + np.arange(3, dtype=np.float32)[:, None], seed=1)
    with pytest.raises(oracle.OracleError) as e:
        T.qt([0, 0], [1, 1], [1], [1])
    assert e.value.code == oracle.OR_EINVAL                         # duplicate id
    with pytest.raises(oracle.OracleError) as e:
        T.qt([5], [1], [1], [1])
    assert e.value.code == oracle.OR_ERANGE                         # id out of range
    with pytest.raises(oracle.OracleError) as e:
        T.ft([0], [0], [1], [1])
    assert e.value.code == oracle.OR_EINVAL                         # zero mass
    with pytest.raises(oracle.OracleError) as e:
        T.ft([0], [70000], [1], [1])
    assert e.value.code == oracle.OR_EOVERFLOW                      # W > 65535


def test_degenerate_trees():
    # Φ = 0: a lone root leaf; every estimate is 0
    T = oracle.Tree(np.ones((4, 3), np.float32), seed=2)
    assert T.n_nodes == 1 and T.d_star == 0
    assert T.qt([0, 1], [1, 2], [2], [5]) == (0, 0.0)
    assert T.ft([0, 1], [1, 2], [2], [5]) == 0.0
    # all points duplicated except one: the duplicates share a depth-D leaf
    X = np.array([[0.0], [0.0], [0.0], [1.0]], np.float32)
    T = oracle.Tree(X, sigma=[0.3], max_depth=5)
    assert len({tuple(T.paths[i]) for i in range(3)}) == 1 and T.d_star == 5
    f = T.flow([0, 1], [1, 1], [2, 3], [1, 1])                     # NW corner inside the shared leaf
    assert f["node"][0] == T.paths[0][5]


# ---------------------------------------------------------------------------------------------
# O10 k-NN vs a full sort by (value, id)
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("prefilter_m", [0, 30, 100, 7])
def test_knn_matches_full_sort(tiny, prefilter_m):
    T = oracle.Tree(tiny.X, seed=tiny.tree_seed, max_depth=tiny.max_depth)
    k = 5
    for qi in range(tiny.nq):
        b, bw = tiny.query(qi)
        ft = [T.ft(*tiny.doc(i), b, bw) for i in range(tiny.n)]
        qt = [T.qt(*tiny.doc(i), b, bw)[1] for i in range(tiny.n)]
        if prefilter_m == 0 or prefilter_m >= tiny.n:
            cand = list(range(tiny.n))
        else:
            cand = sorted(range(tiny.n), key=lambda i: (qt[i], i))[:prefilter_m]
        want = sorted(cand, key=lambda i: (ft[i], i))[:k]
        ids, vals = T.knn(tiny.doc_off, tiny.ids, tiny.w, b, bw, k, prefilter_m)
        assert ids.tolist() == want
        assert vals.tolist() == [ft[i] for i in want]
    # k larger than the candidate count pads with (-1, +inf)
    ids, vals = T.knn(tiny.doc_off[:11], tiny.ids, tiny.w, b, bw, 12, 0)
    assert ids[10:].tolist() == [-1, -1] and np.all(np.isinf(vals[10:]))
    with pytest.raises(oracle.OracleError):
        T.knn(tiny.doc_off, tiny.ids, tiny.w, b, bw, 12, 10)      # 0 < prefilter_m < k
