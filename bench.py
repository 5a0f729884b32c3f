#!/usr/bin/env python
"""bench.py — Flowtree k-NN hot path on B200 (BASELINE.json metric, reviews-like config).

One step = one pass of the whole hot path over one batch of queries:
ft_knn(queries, k=10, prefilter_m=1000) = query prep → Quadtree over all n=100k docs → top-1000
→ distance table → Flowtree rerank → top-10, through the C ABI with inputs already in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun, one process per GPU): by default every rank holds the dataset and answers its
own batch of queries — the path shards by query with no data-path collective, so
scaling is weak; the device time is the max over ranks (NCCL all-reduce of the timings only).
--shard docs splits the docs instead: every rank answers the whole batch over its
doc range and the ranks exchange top-m candidate lists over NCCL (strong scaling).
Prints one JSON line on rank 0.  --impl reference times the CPU oracle (the only other place
this file runs oracle/) on the same config, metric and unit.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Flowtree (query,doc) estimates/sec and k-NN queries/sec at n=100k; % of HBM roofline"
CONFIG = "reviews"
WORKLOAD = "reviews-like (BASELINE configs[2]): X 100k x R^300 mixture, n=100k docs, s~U{10..90}, Zipf(1.1) ids"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM-style copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def int8_peak_tops(clocks_held: bool):
    """Dense int8 tensor peak: the measured bf16 peak (burst when the SM clock held at max during
    the run, sustained otherwise) x the nominal int8/bf16 ratio 4.5/2.25 (B200_PROFILING.md gives
    4.5 POPS dense for fp8; B200 sm_100a runs kind::i8 at the same rate)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    ratio = 4.5 / 2.25
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        key = "bf16_tflops" if clocks_held else "bf16_tflops_sustained"
        if key in j:
            return (float(j[key]) * ratio, f"measured bf16 {'burst' if clocks_held else 'sustained'} "
                                           f"(MEASURED_PEAKS.json {key}) x nominal int8/bf16 ratio 4.5/2.25")
    return 4500.0, "fallback (B200_PROFILING.md 4.5 POPS dense 8-bit)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_info():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def oracle_knn_rate(wl, tree, qsel, threads):
    """Oracle k-NN pipeline (QT over all docs -> top-m -> FT -> top-k) for the queries qsel, one
    query per host thread.  Returns (queries/s, wall seconds)."""
    def one(q):
        b, bw = wl.query(q)
        return tree.knn(wl.doc_off, wl.ids, wl.w, b, bw, wl.k, wl.prefilter_m)
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, qsel))
    dt = time.perf_counter() - t0
    return len(qsel) / dt, dt


# ---------------------------------------------------------------------------------------------
def run_reference(args):
    rank, world, _ = dist_info()
    if rank != 0:
        return 0                                   # rank 0 alone runs the CPU oracle
    import oracle
    from paper_1910_04126_b200 import workloads
    wl = workloads.make(CONFIG)
    tree = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    threads = os.cpu_count() or 1
    per_step = max(threads, 16)
    rng = np.random.default_rng(0)
    times = []
    for s in range(args.warmup + args.steps):
        qsel = rng.choice(wl.nq, per_step, replace=False)
        rate, dt = oracle_knn_rate(wl, tree, qsel, threads)
        if s >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = per_step * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64/f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "n": wl.n, "queries_per_step": per_step,
                                         "k": wl.k, "prefilter_m": wl.prefilter_m},
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": "oracle",
                         "sample": f"{per_step} random queries per step x full n={wl.n}, "
                                   f"QT->top-{wl.prefilter_m}->FT->top-{wl.k}, one query per host thread"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# per-config lines (BASELINE.json configs; the stand-ins for the paper's per-dataset Table 2,
# PAPER.md:352-364): k-NN batch, Quadtree over all docs, exhaustive Flowtree on a query subset
FT_SUBSET = {"tiny": 4, "text": 64, "reviews": 64, "image": 16, "stress": 8}


def measure_configs(ft, workloads, torch, dev, stream, peak, flush, names):
    out = {}

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        ms = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        return statistics.median(ms)

    for name in names:
        t0 = time.perf_counter()
        wl = workloads.make(name)
        gen_s = time.perf_counter() - t0
        ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
        ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
        nq, n, k, m = wl.nq, ds.n, wl.k, wl.prefilter_m
        qi = torch.from_numpy(wl.q_ids).to(dev)
        qw = torch.from_numpy(wl.q_w.view(np.int32)).to(dev).view(torch.uint32)
        oi = torch.empty((nq, k), dtype=torch.int64, device=dev)
        ov = torch.empty((nq, k), dtype=torch.float64, device=dev)
        reps = 2 if name == "image" else 3
        knn_ms = timed(lambda: ds.knn(wl.q_off, qi, qw, k, m, out_ids=oi, out_val=ov, stream=stream), reps)
        # end to end through the C ABI: queries from pinned host memory, answers back to pinned host
        # memory (the call copies both ways on the stream; the events bracket the copies)
        qi_pin = torch.from_numpy(wl.q_ids.copy()).pin_memory()
        qw_pin = torch.from_numpy(wl.q_w.view(np.int32).copy()).pin_memory().view(torch.uint32)
        oi_pin = torch.empty((nq, k), dtype=torch.int64).pin_memory()
        ov_pin = torch.empty((nq, k), dtype=torch.float64).pin_memory()
        e2e_ms = timed(lambda: ds.knn(wl.q_off, qi_pin, qw_pin, k, m, out_ids=oi_pin, out_val=ov_pin, stream=stream),
                       reps)
        # Quadtree over all docs for the whole batch (8 B per doc tree node + 16 B per pair)
        out_qt = torch.empty((nq, n), dtype=torch.float64, device=dev)
        qt_ms = timed(lambda: ds.quadtree(wl.q_off, qi, qw, out=out_qt, stream=stream), 3)
        del out_qt
        qt_bpp = (8 * ds.n_qt + 16 * n) / n
        # exhaustive Flowtree (FT kernel alone; its distance table timed beside it): 8 B per doc
        # support point + 16 B per pair
        nqf = min(nq, FT_SUBSET[name])
        sub = wl.subset_queries(nqf)
        si = torch.from_numpy(sub.q_ids).to(dev)
        sw = torch.from_numpy(sub.q_w.view(np.int32)).to(dev).view(torch.uint32)
        out_ft = torch.empty((nqf, n), dtype=torch.float64, device=dev)
        ds.flowtree(sub.q_off, si, sw, out=out_ft, stream=stream)
        ft.ft_profile_enable(ds.h, True)
        ft.ft_profile_reset(ds.h)
        for _ in range(2):
            flush.zero_()
            ds.flowtree(sub.q_off, si, sw, out=out_ft, stream=stream)
        st = ft.profile_dict(ds.h)
        ft.ft_profile_enable(ds.h, False)
        del out_ft
        f_ms, d_ms = st["flowtree"][0] / 2, st["dist_table"][0] / 2
        ft_bpp = (8 * ds.nnz + 16 * n) / n
        qt_rate, ft_rate = nq * n / (qt_ms / 1e3), nqf * n / (f_ms / 1e3)
        out[name] = {
            "n": n, "N": int(wl.X.shape[0]), "d": int(wl.X.shape[1]), "queries": nq, "k": k, "prefilter_m": m,
            "knn_ms_per_batch": knn_ms, "knn_queries_per_s": nq / (knn_ms / 1e3),
            "e2e_queries_per_s": nq / (e2e_ms / 1e3),
            "e2e_h2d_bytes": 8 * (nq + 1) + 4 * len(wl.q_ids) + 4 * len(wl.q_w), "e2e_d2h_bytes": nq * k * 16,
            "qt_pairs_per_s": qt_rate, "qt_bytes_per_pair": qt_bpp, "qt_frac_hbm": qt_rate * qt_bpp / 1e9 / peak,
            "ft_queries": nqf, "ft_pairs_per_s": ft_rate, "ft_bytes_per_pair": ft_bpp,
            "ft_frac_hbm": ft_rate * ft_bpp / 1e9 / peak, "ft_dist_table_ms": d_ms,
            "ft_pairs_per_s_incl_table": nqf * n / ((f_ms + d_ms) / 1e3), "gen_s": round(gen_s, 1)}
        ds.close()
        ix.close()
        del wl, qi, qw, oi, ov, si, sw
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------------------------
def run_b200(args):
    import torch
    rank, world, local = dist_info()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        dist = None
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_1910_04126_b200 import flowtree as ft, parallel, workloads

    Q = args.queries
    docs_mode = args.shard == "docs"
    wl_all = workloads.make(CONFIG, n_queries=Q if docs_mode else Q * world)
    if docs_mode:
        q_off, q_ids_h, q_w_h = wl_all.q_off, wl_all.q_ids, wl_all.q_w
    else:
        q_off, q_ids_h, q_w_h, _ = parallel.shard_queries(wl_all.q_off, wl_all.q_ids, wl_all.q_w, rank, world)
    wl = wl_all
    k, m = wl.k, wl.prefilter_m

    t_build = time.perf_counter()
    ix = ft.Index(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
    t_load = time.perf_counter()
    if docs_mode:
        d_off, d_ids, d_w, d_base = parallel.shard_docs(wl.doc_off, wl.ids, wl.w, rank, world)
        ds = ft.Dataset(ix, d_off, d_ids, d_w)
        shard = parallel.LibShard(ft, ds, d_base)
    else:
        ds = ft.Dataset(ix, wl.doc_off, wl.ids, wl.w)
    t_done = time.perf_counter()
    build_s, load_s = t_load - t_build, t_done - t_load

    stream = torch.cuda.current_stream()
    q_ids = torch.from_numpy(q_ids_h).to(dev)
    q_w = torch.from_numpy(q_w_h.view(np.int32)).to(dev).view(torch.uint32)
    out_ids = torch.empty((Q, k), dtype=torch.int64, device=dev)
    out_val = torch.empty((Q, k), dtype=torch.float64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        if docs_mode:
            parallel.knn_doc_sharded(shard, q_off, q_ids, q_w, k, m, dist)
        else:
            ds.knn(q_off, q_ids, q_w, k, m, out_ids=out_ids, out_val=out_val, stream=stream)

    def barrier_sync():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    ds.synchronize(stream)
    ft.ft_profile_enable(ds.h, True)
    ft.ft_profile_reset(ds.h)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ft.ft_launch_count()
    clocks = ClockSampler(local)
    barrier_sync()
    for i in range(args.steps):
        flush.zero_()                         # L2 flush (512 MiB write > 126 MB L2), outside the events
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    barrier_sync()
    clk = clocks.stop()
    launches = (ft.ft_launch_count() - launches0) / args.steps
    ds.synchronize(stream)
    t_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    stages = ft.profile_dict(ds.h)
    units = {"dist_table": ft.ft_profile_units(ds.h, 4), "flowtree": ft.ft_profile_units(ds.h, 5),
             "dist_flops": ft.ft_profile_units(ds.h, ft.FT_PROF_DIST_FLOPS)}
    ft.ft_profile_enable(ds.h, False)
    t_ms = parallel.max_over_ranks(t_ms, dist, dev)
    jobq = Q if docs_mode else world * Q                 # queries the whole job answers per step
    value = jobq * args.steps / (t_ms / 1e3)

    # ---- live roofline of the step's kernels; `roofline` is the dominant one (largest device time) ----
    # algorithmic bytes (SURVEY §8(d) and DESIGN.md §7): Quadtree 8 B per doc tree node + 16 B per doc
    # per query scan; distance table rows·(4d + 4 s_q); Flowtree pairs·(8 s_doc + 16) — the last two
    # counted on the device by the library during the timed region.
    peak, peak_src = measured_peaks()
    n_qt = ds.n_qt
    qt_bytes = Q * (8 * n_qt + 16 * ds.n)
    alg_bytes = {"quadtree": qt_bytes * stages["quadtree"][1], "dist_table": units["dist_table"],
                 "flowtree": units["flowtree"]}
    kern = {"quadtree": "k_qt (Quadtree estimate, a3) in the fused prefilter (a3+a4: 1/32-sample scan, "
                        "threshold scan appending candidates, list top-m; the stage time includes the selection)",
            "dist_table": "k_dist_i8 (tcgen05 kind::i8 exact distance table, a5)",
            "flowtree": "k_ftd (lane-per-pair Flowtree estimate, a6) + k_flowtree (list mode: pairs sharing an M-node)"}
    traffic_all = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic_all = json.load(f)
    rooflines = {}
    for stg, b in alg_bytes.items():
        ms, n = stages[stg]
        if n == 0 or ms <= 0 or b <= 0:
            continue
        ach = b / (ms / 1e3) / 1e9
        rooflines[stg] = {"bound": "hbm", "kernel": kern[stg], "achieved": ach, "peak": peak, "unit": "GB/s",
                          "frac": ach / peak, "traffic": traffic_all.get(f"{stg}_dram_bytes_per_launch"),
                          "algorithmic_bytes_per_launch": b / n, "launch_ms": ms / n, "launches": n,
                          "share_of_step": ms / max(t_ms, 1e-9), "peak_source": peak_src}
    if "quadtree" in rooflines:
        # SURVEY §8(d) counts the doc record once per PAIR; the kernel reads it once per 32-query
        # chunk, so this per-pair figure can exceed the HBM peak — the chunk-amortised figure is the
        # bytes the kernel actually has to stream
        rq = rooflines["quadtree"]
        rq["note"] = "per-pair algorithmic bytes (record per pair, SURVEY 8(d)); records are read once per 32 queries"
        rq["frac_chunk_amortised"] = rq["frac"] / 32.0
    if "dist_table" in rooflines and units["dist_flops"] > 0:
        # the distance table is a contraction on the int8 tensor pipe: its roofline is the tensor one.
        # Algorithmic ops = 2·rows·s_q·d (one multiply-add per coordinate of every entry);
        # the exact three-limb kernel executes nine int8 products per algorithmic multiply-add (plus
        # column padding to 16), reported as "executed" beside it.
        held = bool(clk.get("sm_mhz") and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.97 * clk["sm_max_mhz"])
        i8_peak, i8_src = int8_peak_tops(held)
        ms_d, n_d = stages["dist_table"]
        ach_t = units["dist_flops"] / (ms_d / 1e3) / 1e12
        byte_line = rooflines.pop("dist_table")
        # the kernel's arithmetic type is an exact 24-bit fixed-point product carried out as 3 x 3
        # int8 limb products: its tensor peak is the int8 peak / 9.  The int8-peak and TF32-peak
        # fractions of the same algorithmic ops are reported beside it (the latter is round 1's
        # 3xTF32 framing, comparable across rounds).
        i24_peak = i8_peak / 9.0
        tf32_peak = i8_peak * (1.1 / 4.5)
        rooflines["dist_table"] = {
            "bound": "tensor", "kernel": kern["dist_table"], "achieved": ach_t, "peak": i24_peak,
            "unit": "TOP/s (exact 24-bit products, 9 int8 limb MMAs each)", "frac": ach_t / i24_peak,
            "traffic": byte_line["traffic"],
            "algorithmic_ops_per_launch": units["dist_flops"] / n_d, "launch_ms": ms_d / n_d,
            "launches": n_d, "share_of_step": ms_d / max(t_ms, 1e-9),
            "peak_source": i8_src + " / 9 (three limbs on each side)",
            "frac_vs_int8_peak": ach_t / i8_peak, "frac_vs_tf32_peak": ach_t / tf32_peak,
            "executed_int8_ops_per_launch": 9 * units["dist_flops"] / n_d,
            "hbm_view": {"achieved_GBps": byte_line["achieved"], "frac": byte_line["frac"],
                         "algorithmic_bytes_per_launch": byte_line["algorithmic_bytes_per_launch"],
                         "note": "rows*(4d + 4 s_q): each candidate point read once per query, its distances written"},
            "note": "algorithmic ops 2*rows*s_q*d (SURVEY 8(d)); the binding resource is the gather of the "
                    "candidate rows into shared memory and the table stores (DESIGN.md section 7), not the MMAs"}
    dom = max([s for s in rooflines if s in stages], key=lambda s: stages[s][0])
    roofline = dict(rooflines[dom], dominant_stage=dom)

    # ---- kernel-level numbers over all n docs (separately timed; not part of the step) ----
    kernels = {}
    if not args.no_kernels:
        out_qt = torch.empty((Q, ds.n), dtype=torch.float64, device=dev)
        for _ in range(2):
            ds.quadtree(q_off, q_ids, q_w, out=out_qt, stream=stream)
        ft.ft_profile_enable(ds.h, True)
        ft.ft_profile_reset(ds.h)
        reps = 3
        for _ in range(reps):
            flush.zero_()
            ds.quadtree(q_off, q_ids, q_w, out=out_qt, stream=stream)
        st = ft.profile_dict(ds.h)
        qms = st["quadtree"][0] / reps
        del out_qt
        kernels["quadtree_all_docs"] = {
            "pairs": Q * ds.n, "ms": qms, "pairs_per_s": Q * ds.n / (qms / 1e3),
            "algorithmic_GBps": qt_bytes / (qms / 1e3) / 1e9, "frac_hbm": qt_bytes / (qms / 1e3) / 1e9 / peak}
        nqf = min(Q, args.ft_queries)
        sub_off = q_off[:nqf + 1]
        e = int(sub_off[-1])
        out_ft = torch.empty((nqf, ds.n), dtype=torch.float64, device=dev)
        ds.flowtree(sub_off, q_ids[:e], q_w[:e], out=out_ft, stream=stream)
        ft.ft_profile_reset(ds.h)
        flush.zero_()
        ds.flowtree(sub_off, q_ids[:e], q_w[:e], out=out_ft, stream=stream)
        st = ft.profile_dict(ds.h)
        ft.ft_profile_enable(ds.h, False)
        fms, tms = st["flowtree"][0], st["dist_table"][0]
        ft_bytes = nqf * (8 * ds.nnz + 16 * ds.n)      # 8 B per doc support point + 16 B per doc
        kernels["flowtree_all_docs"] = {
            "queries": nqf, "pairs": nqf * ds.n, "ms_flowtree_kernel": fms, "ms_dist_table": tms,
            "pairs_per_s": nqf * ds.n / (fms / 1e3), "algorithmic_GBps": ft_bytes / (fms / 1e3) / 1e9,
            "frac_hbm": ft_bytes / (fms / 1e3) / 1e9 / peak,
            "pairs_per_s_incl_table": nqf * ds.n / ((fms + tms) / 1e3)}
        del out_ft
        # the paper's three-stage pipeline (Table 5: Quadtree 424 -> Flowtree 9 -> Exact 1), full batch
        from paper_1910_04126_b200 import pipeline
        c1, c2 = min(424, ds.n), min(9, ds.n)
        for _ in range(2):
            pipeline.knn_qt_ft_exact(ft, ds, q_off, q_ids, q_w, c1, c2, 1, stream=stream)
        p_ms = 0.0
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pipeline.knn_qt_ft_exact(ft, ds, q_off, q_ids, q_w, c1, c2, 1, stream=stream)
            e1.record(stream)
            e1.synchronize()
            p_ms += e0.elapsed_time(e1) / 3
        kernels["pipeline_qt_ft_exact"] = {"c1": c1, "c2": c2, "k": 1, "queries": Q, "ms": p_ms,
                                           "queries_per_s": Q / (p_ms / 1e3)}

    # ---- e2e: same metric through the C ABI with pinned HOST buffers ----
    qi_pin = torch.from_numpy(q_ids_h.copy()).pin_memory()
    qw_pin = torch.from_numpy(q_w_h.view(np.int32).copy()).pin_memory().view(torch.uint32)
    oi_pin = torch.empty((Q, k), dtype=torch.int64).pin_memory()
    ov_pin = torch.empty((Q, k), dtype=torch.float64).pin_memory()
    def e2e_step():
        if docs_mode:
            ri, rv = parallel.knn_doc_sharded(shard, q_off, qi_pin, qw_pin, k, m, dist)
            oi_pin.copy_(ri, non_blocking=True)
            ov_pin.copy_(rv, non_blocking=True)
        else:
            ds.knn(q_off, qi_pin, qw_pin, k, m, out_ids=oi_pin, out_val=ov_pin, stream=stream)

    for _ in range(2):
        e2e_step()
    barrier_sync()
    e_ms = 0.0
    for i in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        e1.synchronize()
        e_ms += e0.elapsed_time(e1)
    barrier_sync()
    e_ms = parallel.max_over_ranks(e_ms, dist, dev)
    h2d = 8 * (Q + 1) + 4 * len(q_ids_h) + 4 * len(q_w_h)
    d2h = Q * k * (8 + 8)
    e2e = {"value": jobq * args.steps / (e_ms / 1e3), "unit": "queries/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h}

    # ---- every BASELINE.json config on its own (rank 0 at N=1) ----
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = measure_configs(ft, workloads, torch, dev, stream, peak, flush,
                                  ["tiny", "text", "reviews", "image", "stress"])

    # ---- CPU baseline: the oracle, rank 0 at N=1 only, bounded sample ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        tree = oracle.Tree(wl.X, seed=wl.tree_seed, max_depth=wl.max_depth)
        threads = os.cpu_count() or 1
        nsamp = max(16, threads * 2)
        rate, dt = oracle_knn_rate(wl, tree, list(range(nsamp)), threads)
        cpu = {"value": rate, "unit": "queries/s", "cores": threads, "kind": "oracle",
               "sample": f"first {nsamp} queries x full n={wl.n}, QT->top-{m}->FT->top-{k}, one query per host "
                         f"thread ({dt:.1f} s wall)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if docs_mode else "weak",
            "vs_baseline": None, "dtype": "u64/f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": ds.n, "N": wl.X.shape[0], "d": wl.X.shape[1],
                       "queries_per_rank": Q, "global_batch": jobq, "k": k, "prefilter_m": m,
                       "parallelism": f"{'doc' if docs_mode else 'query'}-sharded x{world}",
                       "l2": "flushed (512 MiB write) between timed steps",
                       "qt_records": int(n_qt), "nnz": int(ds.nnz)},
            "ft_estimates_per_s": kernels.get("flowtree_all_docs", {}).get("pairs_per_s"),
            "qt_estimates_per_s": kernels.get("quadtree_all_docs", {}).get("pairs_per_s"),
            "roofline": roofline, "rooflines_by_stage": rooflines, "kernels": kernels, "configs": configs,
            "stages_ms_per_step": {s: v[0] / args.steps for s, v in stages.items()},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk, "cpu_baseline": cpu,
            "build_s": build_s, "load_s": load_s,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--queries", type=int, default=1000, help="queries per rank per step")
    p.add_argument("--ft-queries", type=int, default=64, help="queries for the exhaustive Flowtree kernel line")
    p.add_argument("--no-kernels", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-configs", action="store_true", help="skip the per-config lines (all five BASELINE configs)")
    p.add_argument("--shard", default="queries", choices=["queries", "docs"],
                   help="multi-GPU layout: replicate docs and split queries (weak), or split docs (strong)")
    args = p.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
