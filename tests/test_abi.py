"""CPU-side checks of the boundary: libhsgn.so loads and exports every symbol
include/hsgn.h declares (no compute calls without a GPU), and the product
package never reaches into oracle/."""
import os
import re

import pytest

from paper_2510_07539_b200 import build as B
from paper_2510_07539_b200 import hsgn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hsgn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hsgn_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    path = B.build()
    assert os.path.exists(path)
    L = hsgn.load_library(path)
    decl = _declared()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(hsgn.SYMBOLS) == decl
    # a pure host call: status strings
    assert L.hsgn_status_string(0) == b"ok"
    assert b"coercivity" in L.hsgn_status_string(-3)
    assert b"NCCL" in L.hsgn_status_string(-9)                  # HSGN_E_COMM


def test_diag_struct_matches_header():
    """the ctypes mirror of hsgn_diag has the header's fields in order"""
    src = open(os.path.join(ROOT, "include", "hsgn.h")).read()
    body = src[:src.index("} hsgn_diag;")].rsplit("typedef struct {", 1)[1]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"\b(\w+)\s*;", body)
    assert names == [n for n, _ in hsgn.Diag._fields_]


def test_library_is_sm100a():
    path = B.build()
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2510_07539_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", txt, re.M), f
                assert "hsgn_oracle" not in txt and "orc_" not in txt, f


def test_solver_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        hsgn.Solver(64)
