"""Host-side checks (no GPU): libhet.so builds for sm_100a, loads, and exports
every entry point include/het.h declares; the binding has the same names."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "het.h")).read()
    return sorted(set(re.findall(r"^\s*(?:het_status_t|const char\*)\s+(het_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2112_07221_b200 import build
    build.build()
    import ctypes
    return ctypes.CDLL(build.LIB)


def test_header_declares_boundary():
    syms = declared_symbols()
    for s in ["het_cache_create", "het_lookup", "het_update", "het_evict", "het_sync", "het_stats",
              "het_read_global", "het_get_unique_id", "het_cache_destroy", "het_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_binding_names_match(lib):
    from paper_2112_07221_b200 import het
    for s in declared_symbols():
        assert s in het.EXPORTS, s
        if s != "het_last_error":
            assert callable(getattr(het, s, None)) or s.startswith("het_debug"), s


def test_sass_is_sm100a():
    from paper_2112_07221_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never imports or links oracle/."""
    pkg = os.path.join(ROOT, "paper_2112_07221_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.lower(), f
