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


def test_header_constants_mirrored():
    """Every DG_* constant the Python side mirrors equals the header's."""
    hdr = open(os.path.join(ROOT, "include", "dgb200.h")).read()
    defs = {k: v for k, v in re.findall(r"^#define\s+(DG_\w+)\s+\(?([0-9xXa-fA-F]+)", hdr, re.M)}
    mirrored = [k for k in dir(_lib) if k.startswith("DG_") and isinstance(getattr(_lib, k), int)
                and k in defs]
    assert "DG_MAX_LOCAL" in mirrored
    for k in mirrored:
        assert getattr(_lib, k) == int(defs[k], 0), k
