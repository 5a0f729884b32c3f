"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol that
include/flowtree.h declares, the Python binding mirrors those names, and the product package never
touches the oracle (no compute calls — there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flowtree.h")
PKG = os.path.join(ROOT, "paper_1910_04126_b200")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ft_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1910_04126_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_calls():
    names = _declared()
    for need in ["ft_build_quadtree", "ft_load_dataset", "ft_quadtree_estimate", "ft_flowtree_estimate", "ft_knn"]:
        assert need in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_mirrors_the_abi(lib):
    from paper_1910_04126_b200 import flowtree
    assert sorted(flowtree.EXPORTED) == _declared()
    for name in _declared():
        assert callable(getattr(flowtree, name))


def test_sm100a_code_in_library():
    import subprocess
    from paper_1910_04126_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_product_never_references_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                code = "\n".join(l for l in text.splitlines() if not l.strip().startswith(("#", "//", "*", "/*")))
                assert not re.search(r"\bimport oracle\b|from oracle\b|liboracle|oracle\.c\b", code), f


def test_host_errors_without_gpu(lib):
    """Argument errors detected on the host return status codes without touching the device."""
    lib.ft_build_quadtree.restype = ctypes.c_int
    lib.ft_last_error.restype = ctypes.c_char_p
    h = ctypes.c_void_p()
    rc = lib.ft_build_quadtree(None, ctypes.c_int64(0), ctypes.c_int32(1), ctypes.c_uint64(0), ctypes.c_int32(5),
                               ctypes.byref(h))
    assert rc == 1 and b"NULL" in lib.ft_last_error()
    lib.ft_knn.restype = ctypes.c_int
    rc = lib.ft_knn(None, None, 1, None, None, 5, 0, None, None, None)
    assert rc == 6                                   # FT_ESTATE: NULL dataset


def test_options_roundtrip_without_gpu():
    """ft_set_option / ft_get_option (test and tuning options, no environment reads) work on the
    host and reject unknown keys and out-of-range values."""
    from paper_1910_04126_b200 import flowtree as ft
    for o in range(ft.FT_NUM_OPTIONS):
        assert ft.ft_get_option(o) == 0
    ft.ft_set_option(ft.FT_OPT_TABLE_CHUNK, 3)
    assert ft.ft_get_option(ft.FT_OPT_TABLE_CHUNK) == 3
    ft.ft_set_option(ft.FT_OPT_TABLE_CHUNK, 0)
    for bad in [(ft.FT_NUM_OPTIONS, 1), (-1, 1), (ft.FT_OPT_DEBUG, -1), (ft.FT_OPT_FTD_CARVEOUT, 101)]:
        with pytest.raises(ft.FlowtreeError):
            ft.ft_set_option(*bad)
