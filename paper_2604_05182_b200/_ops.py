"""Thin device-op wrappers over the C ABI used by the host modules."""

import torch

from . import _dev as D
from ._native import call

_ES = {torch.float32: 4, torch.bfloat16: 2, torch.float64: 8, torch.int64: 8,
       torch.int32: 4}


def gather_rows(src: torch.Tensor, index: torch.Tensor, out=None) -> torch.Tensor:
    """out[i] = src[index[i]] for a 2-D row-major src."""
    src2 = src.reshape(src.shape[0], -1)
    n, cols = int(index.shape[0]), int(src2.shape[1])
    out = D.empty((n,) + tuple(src.shape[1:]), src.dtype) if out is None else out
    call("lsrm_gather_rows", _ES[src.dtype], src2.data_ptr(), src2.stride(0),
         index.data_ptr(), n, cols, out.data_ptr(), cols, D.stream())
    return out


def scatter_rows(src: torch.Tensor, index: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[index[i]] = src[i]."""
    src2 = src.reshape(src.shape[0], -1)
    n, cols = int(index.shape[0]), int(src2.shape[1])
    call("lsrm_scatter_rows", _ES[src.dtype], src2.data_ptr(), src2.stride(0),
         index.data_ptr(), n, cols, out.data_ptr(), cols, D.stream())
    return out


def gemm(a: torch.Tensor, b: torch.Tensor, out=None, out_dtype=None) -> torch.Tensor:
    """a [m,k] @ b [k,n] (row-major, unit column stride).  fp32 (no TF32) or
    bf16 with fp32 accumulation."""
    m, k = a.shape
    k2, n = b.shape
    assert k == k2 and a.stride(1) == 1 and b.stride(1) == 1
    if a.dtype == torch.float32:
        mode, odt = 0, torch.float32
    else:
        odt = out_dtype or torch.bfloat16
        mode = 1 if odt == torch.bfloat16 else 2
    out = D.empty((m, n), odt) if out is None else out
    call("lsrm_gemm", mode, m, n, k, a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0),
         out.data_ptr(), out.stride(0), D.stream())
    return out


def cast(src: torch.Tensor, dtype) -> torch.Tensor:
    out = D.empty(tuple(src.shape), dtype)
    to_bf16 = 1 if dtype == torch.bfloat16 else 0
    call("lsrm_cast", to_bf16, src.data_ptr(), out.data_ptr(), src.numel(), D.stream())
    return out


def layer_norm(x: torch.Tensor, gamma, beta, eps=1e-5, out_dtype=None) -> torch.Tensor:
    n, d = x.shape
    odt = out_dtype or x.dtype
    out = D.empty((n, d), odt)
    call("lsrm_layer_norm", int(x.dtype == torch.bfloat16), x.data_ptr(), n, d,
         gamma.data_ptr(), beta.data_ptr(), float(eps), int(odt == torch.bfloat16),
         out.data_ptr(), D.stream())
    return out


def gemm_ex(a: torch.Tensor, b: torch.Tensor, trans_a=False, trans_b=False, out=None,
            beta=0.0, alpha=1.0, tf32=False) -> torch.Tensor:
    """fp32 out = alpha op(a) @ op(b) + beta out (op = transpose when asked;
    tf32 allows TF32 tensor cores)."""
    m, k = (a.shape[1], a.shape[0]) if trans_a else a.shape
    k2, n = (b.shape[1], b.shape[0]) if trans_b else b.shape
    assert k == k2 and a.stride(1) == 1 and b.stride(1) == 1
    assert a.dtype == b.dtype == torch.float32
    if out is None:
        out = D.empty((m, n), torch.float32)
        beta = 0.0
    call("lsrm_gemm_f32_ex", int(trans_a), int(trans_b), m, n, k, float(alpha), a.data_ptr(),
         a.stride(0), b.data_ptr(), b.stride(0), float(beta), out.data_ptr(), out.stride(0),
         int(tf32), D.stream())
    return out
