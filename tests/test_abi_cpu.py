"""CPU-side checks of the C ABI: the library loads and exports every symbol
declared in include/gcharm.h (no compute calls: no GPU here)."""
import ctypes
import os
import re

from conftest import ROOT

from paper_2008_05712_b200 import _lib


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gcharm.h")).read()
    return sorted(set(re.findall(r"\b(gc_[a-z0-9_]+)\s*\(", src)) - {"gc_status"})


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    names = set(_lib.SIGNATURES) | {"gc_last_error", "gc_version"}
    assert set(declared_symbols()) <= names, set(declared_symbols()) - names


def test_version_and_error_strings():
    L = _lib.load()
    assert b"sm_100a" in L.gc_version()
    assert isinstance(L.gc_last_error(), bytes)


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
