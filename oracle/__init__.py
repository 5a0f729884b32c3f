"""CPU oracle for the Flowtree hot path (arXiv 1910.04126) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1910_04126_b200`` never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, fp64, no FMA contraction); this module is
argument marshalling over ctypes plus a gcc build step.  Step numbers O1..O10 and the PAPER.md
citations are in the C file's header.  Parity status of each function:

* ``Tree`` (O1-O5): pinned by SURVEY Appendix A fixtures, SPEC micro-examples and an independent
  brute-force recursive partitioner (tests/test_oracle_pins.py).  The SplitMix64 -> σ mapping is
  pinned only by the published SplitMix64 reference outputs.
* ``qt`` (O6-O7): pinned by the tree-metric LP (scipy.optimize.linprog) and hand values.
* ``flow`` / ``ft`` (O8-O9): pinned by marginals, the ≤ s_μ+s_ν−1 bound, tree cost == QT
  numerator, LP tree-optimality, Flowtree ≥ exact W1 (Birkhoff brute force / LP), the hand-worked
  tie-break example (golden), and the random-model isolation case (Flowtree = W1).
* ``knn`` (O10): pinned against a full Python sort by (value, id).
* ``exact_w1`` (O11): W1 of Eq. (1) as the transportation LP (scipy HiGHS, FP64 costs) on the
  cross-scaled integer masses; pinned by the Birkhoff permutation brute force on uniform
  equal-size supports and the 1-D CDF closed form (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

OR_OK, OR_EINVAL, OR_ERANGE, OR_EOVERFLOW, OR_ENOMEM, OR_ECAP = range(6)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


# ORACLE_SANITIZE=1 (tests/test_oracle_sanitizers.py): load an AddressSanitizer + UBSan build
_SAN = os.environ.get("ORACLE_SANITIZE") == "1"
_SAN_LIB_PATH = os.path.join(_HERE, "liboracle_san.so")


def build_oracle(force: bool = False, sanitize: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no FMA contraction, no fast-math); with
    ``sanitize`` an -fsanitize=address,undefined build (abort on the first report)."""
    path = _SAN_LIB_PATH if sanitize else _LIB_PATH
    if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC):
        tmp = path + f".tmp{os.getpid()}"
        extra = ["-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
                 "-fno-omit-frame-pointer"] if sanitize else []
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-Wall"] + extra + [
            "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, path)
    return path


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = ctypes.CDLL(build_oracle(sanitize=_SAN))
        P = ctypes.c_void_p
        i32, i64, u64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        lib.or_splitmix64.restype = u64
        lib.or_splitmix64.argtypes = [u64, u64]
        lib.or_build.restype = ctypes.c_int
        lib.or_build.argtypes = [P, i64, i32, P, u64, i32, ctypes.POINTER(P)]
        lib.or_tree_free.argtypes = [P]
        lib.or_tree_info.argtypes = [P, P, P, P, P]
        lib.or_tree_vectors.argtypes = [P, P, P]
        lib.or_tree_paths.argtypes = [P, P]
        lib.or_tree_nodes.argtypes = [P, P, P, P]
        lib.or_qt.restype = ctypes.c_int
        lib.or_qt.argtypes = [P, P, P, i32, P, P, i32, P, P]
        lib.or_flow.restype = ctypes.c_int
        lib.or_flow.argtypes = [P, P, P, i32, P, P, i32, P, P, P, P, i32, P, P, P]
        lib.or_ft.restype = ctypes.c_int
        lib.or_ft.argtypes = [P, P, P, P, i32, P, P, i32, P]
        lib.or_dist.restype = f64
        lib.or_dist.argtypes = [P, i32, i32, i32]
        lib.or_knn.restype = ctypes.c_int
        lib.or_knn.argtypes = [P, P, P, i64, P, P, P, P, i32, i32, i64, P, P]
        _lib = lib
        return lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def splitmix64(seed: int, i: int) -> int:
    return int(_load().or_splitmix64(seed, i))


def _support(ids, w):
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.uint32)
    assert ids.shape == w.shape
    return ids, w


class Tree:
    """Oracle quadtree (O1-O5).  ``sigma`` given explicitly overrides the seeded shift."""

    def __init__(self, X: np.ndarray, seed: int = 0, max_depth: int = 32, sigma=None):
        lib = _load()
        self.X = np.ascontiguousarray(X, dtype=np.float32)
        if self.X.ndim == 1:
            self.X = self.X[:, None].copy()
        self.N, self.d = self.X.shape
        h = ctypes.c_void_p()
        sig = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.float64)
        rc = lib.or_build(_ptr(self.X), self.N, self.d, None if sig is None else _ptr(sig),
                          ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(max_depth), ctypes.byref(h))
        if rc != OR_OK:
            raise OracleError(rc, "build")
        self._h = h
        phi = ctypes.c_double(); l_root = ctypes.c_int32(); d_star = ctypes.c_int32(); M = ctypes.c_int64()
        lib.or_tree_info(h, ctypes.byref(phi), ctypes.byref(l_root), ctypes.byref(d_star), ctypes.byref(M))
        self.phi, self.l_root, self.d_star, self.n_nodes = phi.value, l_root.value, d_star.value, M.value
        self.mn = np.zeros(self.d, np.float64)
        self.sigma = np.zeros(self.d, np.float64)
        lib.or_tree_vectors(h, _ptr(self.mn), _ptr(self.sigma))
        self.paths = np.zeros((self.N, self.d_star + 1), np.int32)
        lib.or_tree_paths(h, _ptr(self.paths))
        self.node_depth = np.zeros(self.n_nodes, np.int32)
        self.node_parent = np.zeros(self.n_nodes, np.int32)
        self.node_count = np.zeros(self.n_nodes, np.int32)
        lib.or_tree_nodes(h, _ptr(self.node_depth), _ptr(self.node_parent), _ptr(self.node_count))

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and _lib is not None:
                _lib.or_tree_free(self._h)
                self._h = None
        except Exception:
            pass

    # --- O6/O7 ------------------------------------------------------------------------------
    def qt(self, mu_ids, mu_w, nu_ids, nu_w):
        """Returns (num, value): integer numerator and the Quadtree estimate (O7)."""
        a, aw = _support(mu_ids, mu_w)
        b, bw = _support(nu_ids, nu_w)
        num = ctypes.c_uint64(); val = ctypes.c_double()
        rc = _load().or_qt(self._h, _ptr(a), _ptr(aw), len(a), _ptr(b), _ptr(bw), len(b),
                           ctypes.byref(num), ctypes.byref(val))
        if rc != OR_OK:
            raise OracleError(rc, "qt")
        return num.value, val.value

    # --- O8 ---------------------------------------------------------------------------------
    def flow(self, mu_ids, mu_w, nu_ids, nu_w):
        """Returns dict(src, dst, mass, node, W, U) in emission order (O8)."""
        a, aw = _support(mu_ids, mu_w)
        b, bw = _support(nu_ids, nu_w)
        cap = len(a) + len(b)
        src = np.zeros(cap, np.int32); dst = np.zeros(cap, np.int32)
        mass = np.zeros(cap, np.uint64); node = np.zeros(cap, np.int32)
        n = ctypes.c_int32(); W = ctypes.c_uint64(); U = ctypes.c_uint64()
        rc = _load().or_flow(self._h, _ptr(a), _ptr(aw), len(a), _ptr(b), _ptr(bw), len(b),
                             _ptr(src), _ptr(dst), _ptr(mass), _ptr(node), cap, ctypes.byref(n),
                             ctypes.byref(W), ctypes.byref(U))
        if rc != OR_OK:
            raise OracleError(rc, "flow")
        k = n.value
        return dict(src=src[:k].copy(), dst=dst[:k].copy(), mass=mass[:k].copy(), node=node[:k].copy(),
                    W=W.value, U=U.value)

    # --- O9 ---------------------------------------------------------------------------------
    def ft(self, mu_ids, mu_w, nu_ids, nu_w) -> float:
        a, aw = _support(mu_ids, mu_w)
        b, bw = _support(nu_ids, nu_w)
        val = ctypes.c_double()
        rc = _load().or_ft(self._h, _ptr(self.X), _ptr(a), _ptr(aw), len(a), _ptr(b), _ptr(bw), len(b),
                           ctypes.byref(val))
        if rc != OR_OK:
            raise OracleError(rc, "ft")
        return val.value

    def dist(self, x: int, y: int) -> float:
        return float(_load().or_dist(_ptr(self.X), self.d, int(x), int(y)))

    # --- O10 --------------------------------------------------------------------------------
    def knn(self, doc_off, ids, w, q_ids, q_w, k: int, prefilter_m: int = 0):
        """k-NN of one query over the CSR dataset: exhaustive Flowtree (prefilter_m <= 0 or >= n)
        or Quadtree top-m -> Flowtree top-k.  Returns (ids int64[k], values f64[k])."""
        doc_off = np.ascontiguousarray(doc_off, dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        w = np.ascontiguousarray(w, dtype=np.uint32)
        qa, qw = _support(q_ids, q_w)
        n = len(doc_off) - 1
        out_ids = np.zeros(k, np.int64); out_val = np.zeros(k, np.float64)
        rc = _load().or_knn(self._h, _ptr(self.X), _ptr(doc_off), n, _ptr(ids), _ptr(w), _ptr(qa),
                            _ptr(qw), len(qa), int(k), int(prefilter_m), _ptr(out_ids), _ptr(out_val))
        if rc != OR_OK:
            raise OracleError(rc, "knn")
        return out_ids, out_val


def exact_w1(X, mu_ids, mu_w, nu_ids, nu_w) -> float:
    """O11 — W1(μ, ν) of PAPER.md:21-26 (Eq. (1)): min Σ τ_ij ‖x_i − y_j‖ over transport plans τ
    with marginals μ, ν.  Solved as the transportation LP on the cross-scaled integer masses
    (a_i = w_i U, b_j = u_j W, divided by W U at the end; reading R13), FP64 costs, by scipy's
    HiGHS (a library LP solver as the step, no other arithmetic)."""
    from scipy.optimize import linprog
    Xd = np.asarray(X, np.float64)
    mu_ids = np.asarray(mu_ids, np.int64); nu_ids = np.asarray(nu_ids, np.int64)
    w = np.asarray(mu_w, np.float64); u = np.asarray(nu_w, np.float64)
    W, U = w.sum(), u.sum()
    a, b = w * U, u * W
    C = np.sqrt(((Xd[mu_ids][:, None, :] - Xd[nu_ids][None, :, :]) ** 2).sum(-1))
    p, q = C.shape
    A_eq = np.zeros((p + q, p * q))
    for i in range(p):
        A_eq[i, i * q:(i + 1) * q] = 1.0
    for j in range(q):
        A_eq[p + j, j::q] = 1.0
    # Costs and plans are non-negative and the marginals are consistent (Σa = Σb = W·U), so the LP is
    # feasible and bounded.  With the tight tolerances HiGHS' simplex occasionally reports
    # "unbounded" on marginals of ~1e8 (a 19 x 19 image-like pair found by the randomised sweep):
    # the SAME LP is then re-solved with the solver's default tolerances, then by its
    # interior-point method — a library retry, no other arithmetic.
    res = None
    for method, opts in (("highs", {"primal_feasibility_tolerance": 1e-10, "dual_feasibility_tolerance": 1e-10}),
                         ("highs", {}), ("highs-ipm", {})):
        res = linprog(C.ravel(), A_eq=A_eq, b_eq=np.concatenate([a, b]), bounds=(0, None), method=method,
                      options=opts)
        if res.status == 0:
            break
    if res.status != 0:
        raise OracleError(-1, "exact_w1: " + res.message)
    return float(res.fun) / (W * U)


def dataset_pairs(tree: Tree, doc_off, ids, w, q_off, q_ids, q_w, pairs, which="qt"):
    """Evaluate the oracle on an explicit list of (query, doc) pairs.  Returns f64[len(pairs)]
    (and the integer numerators for which='qt')."""
    out = np.zeros(len(pairs), np.float64)
    nums = np.zeros(len(pairs), np.uint64)
    for t, (qi, di) in enumerate(pairs):
        a0, a1 = int(doc_off[di]), int(doc_off[di + 1])
        b0, b1 = int(q_off[qi]), int(q_off[qi + 1])
        if which == "qt":
            nums[t], out[t] = tree.qt(ids[a0:a1], w[a0:a1], q_ids[b0:b1], q_w[b0:b1])
        else:
            out[t] = tree.ft(ids[a0:a1], w[a0:a1], q_ids[b0:b1], q_w[b0:b1])
    return (nums, out) if which == "qt" else out
