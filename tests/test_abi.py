"""The C-ABI library builds, loads and exports every symbol include/*.h declares (no GPU needed)."""
import ctypes
import glob
import os
import re

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2306_17486_b200", "libhelmsolve_b200.so")


def declared_symbols():
    names = set()
    for hdr in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(hdr).read()
        names |= set(re.findall(r"HS_API\s+[\w\s\*]+?\b(hs_\w+)\s*\(", text))
    return sorted(names)


def test_header_declares_entry_points():
    names = declared_symbols()
    for must in ("hs_helm_apply", "hs_vcycle", "hs_fgmres_solve", "hs_last_error"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built (run __graft_entry__.build())")
def test_library_loads_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    lib.hs_abi_version.restype = ctypes.c_int
    assert lib.hs_abi_version() >= 1


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_ctypes_signatures_cover_header():
    from paper_2306_17486_b200 import _lib

    missing = [n for n in declared_symbols() if n not in _lib.SIGNATURES]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_config_errors_need_no_gpu():
    # argument validation happens before any device work
    from paper_2306_17486_b200 import _lib

    lib = _lib.load()
    h = _lib.HsHierarchy()
    h.num_levels = 3
    h.relax_pre, h.relax_post = 2, 1
    assert lib.hs_vcycle_workspace_bytes(ctypes.byref(h), 1) == 0
    assert "relax_pre" in _lib.last_error()
