"""CPU-side checks of the C-ABI boundary: the library loads without a GPU
and exports every entry point include/mpo_b200.h declares; the ctypes
signature table covers exactly that set."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mpo_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(mpo_\w+)\s*\(", text, flags=re.M)))


def test_header_parses():
    syms = declared_symbols()
    assert "mpo_tnrsvd" in syms and "mpo_sparse_convert" in syms
    assert len(syms) >= 30


def test_library_exports_every_declared_symbol():
    from paper_1707_07803_b200 import _lib
    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_ctypes_table_matches_header():
    from paper_1707_07803_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import paper_1707_07803_b200 as m
    with pytest.raises(RuntimeError):
        m.tnrsvd(m.random_mpo([2] * 6, [2] * 6, [2] * 5, seed=0), 2, q=0)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1707_07803_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), f
                assert "mposvd_oracle" not in src, f
