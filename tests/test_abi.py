"""The C-ABI library loads and exports every symbol include/vanka_b200.h
declares (no compute calls: CPU only)."""

import ctypes
import os
import re

from conftest import ROOT
from paper_2409_14222_b200 import _lib as L

HEADER = os.path.join(ROOT, "include", "vanka_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^VK_API\s+[\w\s\*]+?\b(vk_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_api():
    syms = declared_symbols()
    assert "vk_patches_apply" in syms and "vk_spmv" in syms and len(syms) >= 25


def test_library_exports_every_declared_symbol():
    lib = L.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    assert sorted(L.SIGNATURES) == declared_symbols()


def test_version_and_error_without_gpu():
    lib = L.load()
    assert lib.vk_version() == 1
    # argument validation runs before any device work
    rc = lib.vk_spmv(None, None, None, 1.0, 0.0, None)
    assert rc == L.VK_ERR_ARG
    assert "vk_spmv" in L.last_error()


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2409_14222_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "from oracle" not in src and "import oracle" not in src, fn
