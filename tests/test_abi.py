"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
symbol include/sagesched.h declares (no compute calls)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2603_07917_b200 import _build, _lib

HEADER = os.path.join(os.path.dirname(_build.PKG_DIR), "include", "sagesched.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return ctypes.CDLL(_build.LIB_PATH)


def test_every_declared_symbol_is_exported(lib):
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(header_functions()) == set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_tcgen05_kernel_in_sass():
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB_PATH], capture_output=True,
                          text=True).stdout
    if "k_topk_tc" not in sass:
        pytest.skip("tcgen05 kernel not built yet")
    assert "UTCIMMA" in sass or "UTCQMMA" in sass or "UTCHMMA" in sass
    assert "UTMALDG" in sass


def test_version_and_error_string_without_gpu(lib):
    lib.ss_version.restype = ctypes.c_int
    assert lib.ss_version() >= 10000
    lib.ss_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.ss_last_error(), bytes)
    # bad arguments are rejected before touching the device
    lib.ss_bank_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int64,
                                   ctypes.c_int32, ctypes.c_int64, ctypes.c_int64]
    h = ctypes.c_void_p()
    assert lib.ss_bank_create(ctypes.byref(h), 0, 0, 384, 0, 0) == _lib.SS_ERR_ARG
    assert b"bank_create" in lib.ss_last_error()
