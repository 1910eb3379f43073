"""The C-ABI libraries load and export every symbol include/*.h declares
(no compute calls -- CPU-safe)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2503_02354_b200")


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^[A-Za-z_][\w \*]*?\b(coe_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


@pytest.mark.parametrize("lib, header", [("libcoe_planner.so", "coe_planner.h"), ("libcoe_cuda.so", "coe_cuda.h")])
def test_library_exports_header(lib, header):
    path = os.path.join(PKG, lib)
    if not os.path.exists(path):
        pytest.fail(f"{lib} not built (run python build.py)")
    handle = ctypes.CDLL(path)
    names = declared(header)
    assert len(names) >= 5
    missing = [n for n in names if not hasattr(handle, n)]
    assert not missing, missing
