"""The drop-in boundary loads on a CPU-only host and exports every symbol
include/rocp_b200.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import paper_2007_10798_b200 as rocp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rocp_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(rocp_[a-z0-9_]+)\s*\(", src))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(rocp.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 40
    for name in names:
        assert hasattr(lib, name), name
    assert names == {n for n, _, _ in rocp.SIGNATURES}


def test_binding_loads_without_gpu():
    L = rocp.lib()
    assert L.rocp_nccl_id_size() >= 0


def test_no_cpu_fallback_in_product():
    """The product package never imports or links the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2007_10798_b200")
    pat = re.compile(r"(from\s+oracle|import\s+oracle|rocp_oracle|librocp_oracle|orc_[a-z_]+\()")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h", "Makefile")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f
