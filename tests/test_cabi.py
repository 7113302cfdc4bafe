"""The C-ABI library loads and exports every symbol include/dgb200.h
declares (no device calls: runs on the CPU-only build box)."""

import os
import re

from paper_2504_04673_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "dgb200.h")).read()
    declared = set(re.findall(r"^\s*(?:const char\*|int64_t|int)\s+(dg_\w+)\s*\(", hdr, re.M))
    assert declared, "no declarations parsed"
    h = _lib.load_library()
    for name in sorted(declared):
        assert hasattr(h, name), name
    assert declared == set(_lib.EXPORTED)


def test_version_and_launch_counter():
    h = _lib.load_library()
    assert h.dg_version() >= 1
    assert h.dg_launch_count() >= 0
