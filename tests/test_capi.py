"""The C-ABI library loads without a GPU and exports every symbol that
include/lsrm_b200.h declares; the ctypes table matches the header."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lsrm_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lsrm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_2604_05182_b200 import build
    from paper_2604_05182_b200._native import LIB_PATH
    build.build()
    lib = ctypes.CDLL(LIB_PATH)
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_covers_header():
    from paper_2604_05182_b200._native import SIGNATURES, lib
    assert sorted(SIGNATURES) == declared()
    l = lib()
    assert l.lsrm_abi_version() == 1
    assert l.lsrm_partition_workspace(100, 64) > 0
    assert l.lsrm_compact_workspace(1000) > 1000


def test_header_arity_matches_ctypes():
    from paper_2604_05182_b200._native import SIGNATURES
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for name, (_, args) in SIGNATURES.items():
        m = re.search(name + r"\s*\(([^)]*)\)", src)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), (name, len(params), len(args))
