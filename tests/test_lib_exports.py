"""CPU checks of the C-ABI boundary: the in-tree library loads and exports
exactly the entry points include/hcamg.h declares (no compute calls)."""

import ctypes
import os
import re

import pytest

from paper_2602_23613_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hcamg.h")).read()
    return sorted(set(re.findall(r"\b(hcamg_[a-z_0-9]+)\s*\(", text)) - {"hcamg_precond_fn"})


def test_header_matches_binding_table():
    assert header_symbols() == sorted(_lib.EXPORTS)


@pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="libhcamg.so not built")
def test_library_exports_every_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    loaded = _lib.load()
    assert loaded.hcamg_version() == 1


def test_no_cpu_fallback_when_library_missing(monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libhcamg.so")
    with pytest.raises(_lib.NativeUnavailable):
        _lib.load()
