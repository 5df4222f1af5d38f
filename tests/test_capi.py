"""The C-ABI library loads and exports every symbol declared in include/skelb200.h
(no compute calls: runs without a GPU)."""

import ctypes
import os
import re

from paper_2001_11619_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "skelb200.h")).read()
    return sorted(set(re.findall(r"^int\s+(skb_\w+)\s*\(", src, flags=re.M)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_bindings_cover_header():
    assert set(declared()) <= set(_lib.SIGNATURES)
    _lib.load()
    assert _lib.load().skb_version() == 1


def test_descriptor_layouts():
    # SkbGemm is 4 pointers + 7 int64 + 2 doubles + 2 int32 + int64 = 120 bytes
    assert _lib.GEMM_DT.itemsize == 120
    assert _lib.MAT_DT.itemsize == 32
