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


def test_host_boundary_argument_checks_without_gpu():
    """The boundary's argument checks run before any CUDA call, so they hold
    on a CPU-only host: lsrm_h2d_rows rejects a row stride shorter than the
    row and null buffers, and an empty transfer is a no-op; lsrm_gemm_tc
    rejects an MN-major operand whose row stride is shorter than its rows
    and more than 32 problems."""
    import ctypes as C
    import numpy as np
    from paper_2604_05182_b200 import _ops
    from paper_2604_05182_b200._native import lib
    l = lib()
    a = np.zeros((4, 8), np.float32)
    assert l.lsrm_h2d_rows(1, a.ctypes.data, 4, None, 4, 8, 16, 8, None) == 1   # ld < row
    assert l.lsrm_h2d_rows(1, None, 8, None, 4, 8, 16, 8, None) == 1          # null source
    assert l.lsrm_h2d_rows(1, a.ctypes.data, 8, None, 0, 8, None, 8, None) == 0   # empty
    assert b"h2d_rows" in l.lsrm_last_error()

    def gemm(m, n, k, lda, ldb, flags, count=1):
        p = _ops.GemmProblem(m, n, k, 4096, lda, 8192, ldb, 16384, n, None, None, 0, flags, 0)
        arr = (_ops.GemmProblem * count)(*([p] * count))
        return l.lsrm_gemm_tc(C.cast(arr, C.c_void_p), count, None)
    assert gemm(64, 64, 128, 32, 128, _ops.GEMM_A_MN) == 1        # A^T row stride < m
    assert gemm(64, 64, 128, 128, 32, _ops.GEMM_B_MN) == 1        # W row stride < n
    assert gemm(64, 64, 128, 128, 128, 0, count=33) == 1          # > 32 problems
