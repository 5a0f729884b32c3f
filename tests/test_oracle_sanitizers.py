"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY §5 "race detection /
sanitizers": host oracle under -fsanitize=address,undefined).  A subprocess loads the sanitized
build of oracle/oracle.c (ORACLE_SANITIZE=1, libasan preloaded into the interpreter) and runs every
entry point — build (incl. depth-capped multi-point leaves and Φ = 0), Quadtree, flow, Flowtree,
k-NN exhaustive and prefiltered — on the tiny config and the Appendix A fixtures; any report
aborts the process (-fno-sanitize-recover=all).  CPU only."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import oracle, ft_testlib as H
from paper_1910_04126_b200 import workloads
assert oracle._load()._name.endswith("liboracle_san.so")
wl = workloads.make("tiny")
T = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
for q in range(wl.nq):
    qi, qw = wl.query(q)
    for d in range(0, wl.n, 7):
        di, dw = wl.doc(d)
        T.qt(di, dw, qi, qw); T.flow(di, dw, qi, qw); T.ft(di, dw, qi, qw)
T.knn(wl.doc_off, wl.ids, wl.w, wl.q_ids[:8], wl.q_w[:8], 5, 0)
T.knn(wl.doc_off, wl.ids, wl.w, wl.q_ids[:8], wl.q_w[:8], 5, 30)
for name in ("appendixA_example1.json", "appendixA_example2.json"):
    g = H.golden(name)
    Tg = oracle.Tree(np.array(g["X"], np.float32), sigma=g["sigma"], max_depth=g["max_depth"])
    for c in g["cases"]:
        mi, mw = [p[0] for p in c["mu"]], [p[1] for p in c["mu"]]
        ni, nw = [p[0] for p in c["nu"]], [p[1] for p in c["nu"]]
        Tg.flow(mi, mw, ni, nw); Tg.qt(mi, mw, ni, nw); Tg.ft(mi, mw, ni, nw)
Xc = np.random.default_rng(1).standard_normal((60, 3)).astype(np.float32); Xc[10:20] = Xc[0]
Tc = oracle.Tree(Xc, seed=3, max_depth=2)
Tc.flow(list(range(0, 30)), [1] * 30, list(range(15, 50)), [2] * 35)
oracle.Tree(np.zeros((4, 2), np.float32), seed=1)
print("SANITIZED-OK")
'''


@pytest.mark.slow
def test_oracle_clean_under_asan_ubsan(tmp_path):
    libasan = subprocess.run(["gcc", "-print-file-name=libasan.so"], capture_output=True, text=True).stdout.strip()
    if not os.path.isabs(libasan):
        pytest.skip("libasan not available")
    env = dict(os.environ, ORACLE_SANITIZE="1", LD_PRELOAD=libasan,
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1", UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True, env=env, timeout=600)
    assert p.returncode == 0 and "SANITIZED-OK" in p.stdout, (p.stdout[-2000:], p.stderr[-4000:])
