"""Thin Python binding of the C ABI in ``include/flowtree.h`` (ctypes; argument marshalling only).

Every function has the C name and forwards to ``libflowtree_b200.so``; all of the method's
arithmetic runs in that library's CUDA kernels.  There is no fallback: if the library is missing
the import fails loudly (build it with ``python -m paper_1910_04126_b200.build``).

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); torch CUDA outputs make the
call asynchronous on ``stream`` (a ``torch.cuda.Stream`` or raw ``cudaStream_t`` int; default:
torch's current stream when a torch CUDA tensor is involved, else the legacy default stream).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FT_LIB (development hook, tools/variants.py): an alternative build of the same library
LIB_PATH = os.environ.get("FT_LIB") or os.path.join(_HERE, "libflowtree_b200.so")

FT_OK, FT_EINVAL, FT_ERANGE, FT_EOVERFLOW, FT_ENOMEM, FT_ECUDA, FT_ESTATE = range(7)
STATUS_NAMES = {0: "FT_OK", 1: "FT_EINVAL", 2: "FT_ERANGE", 3: "FT_EOVERFLOW", 4: "FT_ENOMEM",
                5: "FT_ECUDA", 6: "FT_ESTATE"}

EXPORTED = ["ft_build_quadtree", "ft_build_quadtree_shift", "ft_index_info", "ft_index_paths",
            "ft_index_sigma", "ft_index_nodes", "ft_load_dataset", "ft_dataset_info",
            "ft_quadtree_estimate", "ft_flowtree_estimate", "ft_flowtree_flow", "ft_knn",
            "ft_synchronize", "ft_index_free", "ft_dataset_free", "ft_last_error",
            "ft_profile_enable", "ft_profile_reset", "ft_profile_read", "ft_profile_units",
            "ft_profile_stage_name", "ft_launch_count", "ft_topk", "ft_flowtree_estimate_lists",
            "ft_exact_w1_lists", "ft_set_option", "ft_get_option"]
FT_NUM_STAGES = 7
# ft_set_option keys (include/flowtree.h)
(FT_OPT_VOCAB_HASH, FT_OPT_WARP_ONLY, FT_OPT_QT_HASH, FT_OPT_SELECT_RADIX, FT_OPT_EXACT_START_NW,
 FT_OPT_TABLE_CHUNK, FT_OPT_TABLE_BUDGET_MB, FT_OPT_QT_WAVES, FT_OPT_FTD_CARVEOUT, FT_OPT_DEBUG,
 FT_OPT_PREFILTER_UNFUSED, FT_OPT_QT_PAIR_OFF, FT_OPT_DIST_QMAJOR) = range(13)
FT_NUM_OPTIONS = 13
FT_PROF_DIST_FLOPS = FT_NUM_STAGES   # ft_profile_units slot: distance-table algorithmic flops


class FlowtreeError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status


def _load_lib():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1910_04126_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    st = ctypes.c_int
    sig = {
        "ft_build_quadtree": (st, [P, i64, i32, u64, i32, P]),
        "ft_build_quadtree_shift": (st, [P, i64, i32, P, i32, P]),
        "ft_index_info": (st, [P, P, P, P, P]),
        "ft_index_paths": (st, [P, P]),
        "ft_index_sigma": (st, [P, P]),
        "ft_index_nodes": (st, [P, P, P]),
        "ft_load_dataset": (st, [P, P, i64, P, P, P]),
        "ft_dataset_info": (st, [P, P, P, P, P]),
        "ft_quadtree_estimate": (st, [P, P, i32, P, P, P, i64, P, P]),
        "ft_flowtree_estimate": (st, [P, P, i32, P, P, P, i64, P, P]),
        "ft_flowtree_flow": (st, [P, i32, P, P, i64, P, P, P, P, i32, P]),
        "ft_knn": (st, [P, P, i32, P, P, i32, i64, P, P, P]),
        "ft_synchronize": (st, [P, P]),
        "ft_index_free": (None, [P]),
        "ft_dataset_free": (None, [P]),
        "ft_last_error": (ctypes.c_char_p, []),
        "ft_profile_enable": (st, [P, i32]),
        "ft_profile_reset": (st, [P]),
        "ft_profile_read": (st, [P, i32, P, P]),
        "ft_profile_units": (st, [P, i32, P]),
        "ft_profile_stage_name": (ctypes.c_char_p, [i32]),
        "ft_launch_count": (u64, []),
        "ft_topk": (st, [P, i64, P, i64, i64, i64, i32, i32, P, P, P]),
        "ft_flowtree_estimate_lists": (st, [P, P, i32, P, P, P, i64, i64, P, P]),
        "ft_exact_w1_lists": (st, [P, P, i32, P, P, P, i64, i64, P, P]),
        "ft_set_option": (st, [i32, i64]),
        "ft_get_option": (st, [i32, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load_lib()


def _check(rc):
    if rc != FT_OK:
        raise FlowtreeError(rc, _lib.ft_last_error().decode())


# ------------------------------------------------------------------------------------------------
# marshalling helpers
# ------------------------------------------------------------------------------------------------
def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a, dtype):
    """(pointer, keepalive, is_cuda) for a numpy array or torch tensor of the given numpy dtype."""
    if a is None:
        return None, None, False
    if _is_torch(a):
        import torch
        want = {np.int32: torch.int32, np.int64: torch.int64, np.uint32: torch.uint32,
                np.float32: torch.float32, np.float64: torch.float64}[dtype]
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"expected a contiguous tensor of {want}, got {a.dtype}")
        return ctypes.c_void_p(a.data_ptr()), a, a.is_cuda
    arr = np.ascontiguousarray(a, dtype=dtype)
    return ctypes.c_void_p(arr.ctypes.data), arr, False


def _stream_ptr(stream, any_cuda):
    if stream is None:
        if not any_cuda:
            return None
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


# ------------------------------------------------------------------------------------------------
# C ABI, same names
# ------------------------------------------------------------------------------------------------
def ft_build_quadtree(X, seed: int, max_depth: int = 32):
    Xp, Xk, _ = _ptr(X, np.float32)
    N, d = (Xk.shape if Xk.ndim == 2 else (Xk.shape[0], 1))
    h = ctypes.c_void_p()
    _check(_lib.ft_build_quadtree(Xp, N, d, ctypes.c_uint64(seed & (2**64 - 1)), max_depth, ctypes.byref(h)))
    return h


def ft_build_quadtree_shift(X, sigma, max_depth: int = 32):
    Xp, Xk, _ = _ptr(X, np.float32)
    N, d = (Xk.shape if Xk.ndim == 2 else (Xk.shape[0], 1))
    sp, sk, _ = _ptr(sigma, np.float64)
    h = ctypes.c_void_p()
    _check(_lib.ft_build_quadtree_shift(Xp, N, d, sp, max_depth, ctypes.byref(h)))
    return h


def ft_index_info(ix):
    phi = ctypes.c_double(); l_root = ctypes.c_int32(); d_star = ctypes.c_int32(); M = ctypes.c_int64()
    _check(_lib.ft_index_info(ix, ctypes.byref(phi), ctypes.byref(l_root), ctypes.byref(d_star), ctypes.byref(M)))
    return phi.value, l_root.value, d_star.value, M.value


def ft_index_paths(ix, N: int):
    _, _, d_star, _ = ft_index_info(ix)
    out = np.empty((N, d_star + 1), np.int32)
    _check(_lib.ft_index_paths(ix, ctypes.c_void_p(out.ctypes.data)))
    return out


def ft_index_sigma(ix, d: int):
    out = np.empty(d, np.float64)
    _check(_lib.ft_index_sigma(ix, ctypes.c_void_p(out.ctypes.data)))
    return out


def ft_index_nodes(ix):
    M = ft_index_info(ix)[3]
    depth = np.empty(M, np.int32); count = np.empty(M, np.int32)
    _check(_lib.ft_index_nodes(ix, ctypes.c_void_p(depth.ctypes.data), ctypes.c_void_p(count.ctypes.data)))
    return depth, count


def ft_load_dataset(ix, doc_off, ids, w):
    op, ok, _ = _ptr(doc_off, np.int64)
    ip, ik, _ = _ptr(ids, np.int32)
    wp, wk, _ = _ptr(w, np.uint32)
    h = ctypes.c_void_p()
    _check(_lib.ft_load_dataset(ix, op, len(ok) - 1, ip, wp, ctypes.byref(h)))
    return h


def ft_dataset_info(ds):
    n = ctypes.c_int64(); nnz = ctypes.c_int64(); nqt = ctypes.c_int64(); ms = ctypes.c_int32()
    _check(_lib.ft_dataset_info(ds, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(nqt), ctypes.byref(ms)))
    return n.value, nnz.value, nqt.value, ms.value


def _estimate(fn, ds, q_off, q_ids, q_w, docs, out, stream):
    q_off = np.ascontiguousarray(q_off, dtype=np.int64)
    nq = len(q_off) - 1
    ip, ik, ic = _ptr(q_ids, np.int32)
    wp, wk, wc = _ptr(q_w, np.uint32)
    dp, dk, dc = _ptr(docs, np.int64)
    if docs is None:
        n_docs = ft_dataset_info(ds)[0]
    else:
        n_docs = len(dk)
    if out is None:
        out = np.empty((nq, n_docs), np.float64)
    op, ok, oc = _ptr(out, np.float64)
    sp = _stream_ptr(stream, ic or wc or dc or oc)
    _check(fn(ds, ctypes.c_void_p(q_off.ctypes.data), nq, ip, wp, dp, n_docs, op, sp))
    return out


def ft_quadtree_estimate(ds, q_off, q_ids, q_w, docs=None, out=None, stream=None):
    """Quadtree estimates [nq, n_docs]."""
    return _estimate(_lib.ft_quadtree_estimate, ds, q_off, q_ids, q_w, docs, out, stream)


def ft_flowtree_estimate(ds, q_off, q_ids, q_w, docs=None, out=None, stream=None):
    """Flowtree estimates [nq, n_docs]."""
    return _estimate(_lib.ft_flowtree_estimate, ds, q_off, q_ids, q_w, docs, out, stream)


def ft_flowtree_flow(ds, q_ids, q_w, doc: int, cap: int = 1 << 16):
    """Flow triples of one (query, doc) pair in canonical order: dict(src, dst, mass, node)."""
    ip, ik, _ = _ptr(q_ids, np.int32)
    wp, wk, _ = _ptr(q_w, np.uint32)
    src = np.empty(cap, np.int32); dst = np.empty(cap, np.int32)
    mass = np.empty(cap, np.uint64); node = np.empty(cap, np.int32)
    n = ctypes.c_int32()
    _check(_lib.ft_flowtree_flow(ds, len(ik), ip, wp, int(doc), ctypes.c_void_p(src.ctypes.data),
                                 ctypes.c_void_p(dst.ctypes.data), ctypes.c_void_p(mass.ctypes.data),
                                 ctypes.c_void_p(node.ctypes.data), cap, ctypes.byref(n)))
    k = n.value
    return dict(src=src[:k].copy(), dst=dst[:k].copy(), mass=mass[:k].copy(), node=node[:k].copy())


def ft_knn(ds, q_off, q_ids, q_w, k: int, prefilter_m: int = 0, out_ids=None, out_val=None, stream=None):
    """k-NN by Flowtree (optionally Quadtree-prefiltered): (ids int64 [nq,k], values f64 [nq,k])."""
    q_off = np.ascontiguousarray(q_off, dtype=np.int64)
    nq = len(q_off) - 1
    ip, ik, ic = _ptr(q_ids, np.int32)
    wp, wk, wc = _ptr(q_w, np.uint32)
    if out_ids is None:
        out_ids = np.empty((nq, k), np.int64)
    if out_val is None:
        out_val = np.empty((nq, k), np.float64)
    oip, oik, oic = _ptr(out_ids, np.int64)
    ovp, ovk, ovc = _ptr(out_val, np.float64)
    sp = _stream_ptr(stream, ic or wc or oic or ovc)
    _check(_lib.ft_knn(ds, ctypes.c_void_p(q_off.ctypes.data), nq, ip, wp, int(k), int(prefilter_m), oip, ovp, sp))
    return out_ids, out_val


def ft_topk(vals, k: int, ids=None, id_base: int = 0, out_ids=None, out_val=None, stream=None):
    """Per row the k smallest (value, id) of a DEVICE [rows, L] float64 tensor, ties by id; ids is
    a device int64 [rows, L] tensor or None (id = id_base + column).  Returns device tensors."""
    import torch
    rows, L = vals.shape
    if out_ids is None:
        out_ids = torch.empty((rows, k), dtype=torch.int64, device=vals.device)
    if out_val is None:
        out_val = torch.empty((rows, k), dtype=torch.float64, device=vals.device)
    vp, vk, _ = _ptr(vals, np.float64)
    ip, ik, _ = _ptr(ids, np.int64)
    oip, oik, _ = _ptr(out_ids, np.int64)
    ovp, ovk, _ = _ptr(out_val, np.float64)
    _check(_lib.ft_topk(vp, vals.stride(0), ip, ids.stride(0) if ids is not None else 0, int(id_base), L, rows,
                        int(k), oip, ovp, _stream_ptr(stream, True)))
    return out_ids, out_val


def ft_flowtree_estimate_lists(ds, q_off, q_ids, q_w, docs, out=None, stream=None):
    """Flowtree estimates of per-query candidate lists: docs is a DEVICE int64 [nq, n] tensor of doc
    indices (negative = skipped, +inf out; >= n: NaN and FT_ERANGE); returns a DEVICE float64 [nq, n] tensor."""
    import torch
    q_off = np.ascontiguousarray(q_off, dtype=np.int64)
    nq = len(q_off) - 1
    n = docs.shape[1]
    if out is None:
        out = torch.empty((nq, n), dtype=torch.float64, device=docs.device)
    ip, ik, ic = _ptr(q_ids, np.int32)
    wp, wk, wc = _ptr(q_w, np.uint32)
    dp, dk, _ = _ptr(docs, np.int64)
    op, ok, _ = _ptr(out, np.float64)
    _check(_lib.ft_flowtree_estimate_lists(ds, ctypes.c_void_p(q_off.ctypes.data), nq, ip, wp, dp, docs.stride(0), n,
                                           op, _stream_ptr(stream, True)))
    return out


def ft_exact_w1_lists(ds, q_off, q_ids, q_w, docs, out=None, stream=None):
    """Exact W1 of per-query candidate lists (DEVICE int64 [nq, n] doc indices; negative =
    skipped, +inf out); returns a DEVICE float64 [nq, n] tensor."""
    import torch
    q_off = np.ascontiguousarray(q_off, dtype=np.int64)
    nq = len(q_off) - 1
    n = docs.shape[1]
    if out is None:
        out = torch.empty((nq, n), dtype=torch.float64, device=docs.device)
    ip, ik, ic = _ptr(q_ids, np.int32)
    wp, wk, wc = _ptr(q_w, np.uint32)
    dp, dk, _ = _ptr(docs, np.int64)
    op, ok, _ = _ptr(out, np.float64)
    _check(_lib.ft_exact_w1_lists(ds, ctypes.c_void_p(q_off.ctypes.data), nq, ip, wp, dp, docs.stride(0), n, op,
                                  _stream_ptr(stream, True)))
    return out


def ft_synchronize(ds, stream=None):
    _check(_lib.ft_synchronize(ds, _stream_ptr(stream, stream is not None)))


def ft_index_free(ix):
    _lib.ft_index_free(ix)


def ft_dataset_free(ds):
    _lib.ft_dataset_free(ds)


def ft_last_error() -> str:
    return _lib.ft_last_error().decode()


def ft_profile_enable(ds, enable: bool = True):
    _check(_lib.ft_profile_enable(ds, 1 if enable else 0))


def ft_profile_reset(ds):
    _check(_lib.ft_profile_reset(ds))


def ft_profile_read(ds, stage: int):
    """(total device ms, timed launches) of one stage since the last reset."""
    ms = ctypes.c_double(); n = ctypes.c_int64()
    _check(_lib.ft_profile_read(ds, stage, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def ft_profile_units(ds, stage: int) -> int:
    """Algorithmic bytes counted on the device for a stage since the last reset."""
    v = ctypes.c_uint64()
    _check(_lib.ft_profile_units(ds, stage, ctypes.byref(v)))
    return int(v.value)


def ft_profile_stage_name(stage: int) -> str:
    return _lib.ft_profile_stage_name(stage).decode()


def ft_set_option(option: int, value: int):
    _check(_lib.ft_set_option(int(option), int(value)))


def ft_get_option(option: int) -> int:
    v = ctypes.c_int64(0)
    _check(_lib.ft_get_option(int(option), ctypes.byref(v)))
    return v.value


def ft_launch_count() -> int:
    return int(_lib.ft_launch_count())


def profile_dict(ds):
    """{stage name: (total ms, launches)} for every stage."""
    return {ft_profile_stage_name(s): ft_profile_read(ds, s) for s in range(FT_NUM_STAGES)}


# ------------------------------------------------------------------------------------------------
# owning wrappers
# ------------------------------------------------------------------------------------------------
class Index:
    """Owns an ``ft_index`` (the device-resident quadtree)."""

    def __init__(self, X, seed: int = 0, max_depth: int = 32, sigma=None):
        X = np.ascontiguousarray(X, dtype=np.float32)
        if X.ndim == 1:
            X = X[:, None].copy()
        self.N, self.d = X.shape
        self.h = ft_build_quadtree(X, seed, max_depth) if sigma is None else ft_build_quadtree_shift(X, sigma, max_depth)
        self.phi, self.l_root, self.d_star, self.n_nodes = ft_index_info(self.h)

    def paths(self):
        return ft_index_paths(self.h, self.N)

    def sigma(self):
        return ft_index_sigma(self.h, self.d)

    def nodes(self):
        return ft_index_nodes(self.h)

    def close(self):
        if self.h is not None:
            ft_index_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Dataset:
    """Owns an ``ft_dataset`` (the node-sorted layout); keeps its Index alive."""

    def __init__(self, index: Index, doc_off, ids, w):
        self.index = index
        self.h = ft_load_dataset(index.h, doc_off, ids, w)
        self.n, self.nnz, self.n_qt, self.max_s = ft_dataset_info(self.h)

    def quadtree(self, q_off, q_ids, q_w, docs=None, out=None, stream=None):
        return ft_quadtree_estimate(self.h, q_off, q_ids, q_w, docs, out, stream)

    def flowtree(self, q_off, q_ids, q_w, docs=None, out=None, stream=None):
        return ft_flowtree_estimate(self.h, q_off, q_ids, q_w, docs, out, stream)

    def flow(self, q_ids, q_w, doc):
        return ft_flowtree_flow(self.h, q_ids, q_w, doc)

    def knn(self, q_off, q_ids, q_w, k, prefilter_m=0, out_ids=None, out_val=None, stream=None):
        return ft_knn(self.h, q_off, q_ids, q_w, k, prefilter_m, out_ids, out_val, stream)

    def synchronize(self, stream=None):
        ft_synchronize(self.h, stream)

    def close(self):
        if self.h is not None:
            ft_dataset_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
