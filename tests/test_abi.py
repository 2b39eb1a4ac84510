"""CPU: libskel.so loads, exports every symbol include/skel.h declares, and rejects bad calls
without touching a GPU."""
import ctypes
import os
import re

import pytest

from paper_2104_05877_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "skel.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:sk_status|void|const char\*|int64_t|size_t)\s+(sk_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ("sk_sketch", "sk_select_cols", "sk_select_rows", "sk_id_coeffs", "sk_residual",
              "sk_select_cols_cpqr", "sk_gather_cols", "sk_rand_lupp", "sk_create", "sk_destroy"):
        assert n in names
    assert names == _lib.EXPORTS


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for n in declared():
        assert hasattr(lib, n), n
    assert lib.sk_version().decode().startswith("skel")


def test_null_context_is_an_argument_error():
    lib = _lib.load()
    assert lib.sk_sketch(None, None, 1, 1, 1, 1, 0, 8, 0, None, 1) == _lib.SK_E_ARG
    assert lib.sk_select_cols(None, None, 1, 1, 1, 1, None, None, 1, None, 1, None, None) == _lib.SK_E_ARG
    assert lib.sk_last_error(None).decode() == "null context"
    lib.sk_destroy(None)


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(OSError):
        _lib._lib = None
        try:
            _lib.load(str(tmp_path / "nope.so"))
        finally:
            _lib._lib = None


def test_header_compiles_as_c_and_cxx(tmp_path):
    """include/skel.h is self-contained for C and C++ callers (it declares the C ABI only)."""
    import shutil
    import subprocess
    for cc, lang in (("gcc", "c"), ("g++", "c++")):
        if shutil.which(cc) is None:
            pytest.skip(f"{cc} not available")
        r = subprocess.run([cc, "-fsyntax-only", "-Wall", "-Werror", "-x", lang, HEADER], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_round2_entry_points_reject_bad_calls_without_a_gpu():
    """The round-2 entry points validate before touching a device: NULL context -> SK_E_ARG;
    sk_nccl_unique_id(NULL) -> SK_E_ARG; sk_create_dist with an impossible partition -> SK_E_ARG."""
    lib = _lib.load()
    E = _lib.SK_E_ARG
    assert lib.sk_set_sketch_tuning(None, 0, 0, 0, 0, 0) == E
    assert lib.sk_sketch_power_ortho(None, None, 1, 1, 1, 1, 0, 8, 0, 1, None, 1, None) == E
    assert lib.sk_sketch_dual(None, None, 0, 1, 1, 1, 1, 1, 0, 0, 0, None, 1, None, 1) == E
    assert lib.sk_id_estimate_cols(None, None, 1, 1, 1, None, 1, None, 1, None) == E
    assert lib.sk_id_estimate_rows(None, None, 1, 1, 1, None, 1, None, 1, None) == E
    assert lib.sk_set_dist_exchange(None, 0) == E
    assert lib.sk_dist_info(None, None, None, None, None, None) == E
    assert lib.sk_nccl_unique_id(None) == E
    h = ctypes.c_void_p()
    uid = (ctypes.c_char * 128)()
    # rank outside [0, world), negative column count: rejected before NCCL or CUDA is touched
    assert lib.sk_create_dist(ctypes.byref(h), 0, None, uid, 2, 2, 100, 0, 50) == E
    assert lib.sk_create_dist(ctypes.byref(h), 0, None, uid, 0, 1, 100, 60, 50) == E
    assert not h.value
