"""The C-ABI library loads on a CPU-only host and exports every entry point
declared in include/fvb.h (no compute calls without a GPU)."""

import ctypes
import os
import re

from paper_1207_1571_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "fvb.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fvb_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared()
    assert len(names) >= 30
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), n
    assert set(_lib.EXPORTS) == set(names)


def test_version_and_error_channel():
    assert _lib.lib.fvb_version() >= 100
    assert isinstance(_lib.last_error(), str)


def test_library_is_sm100a():
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob
