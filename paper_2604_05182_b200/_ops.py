"""Thin device-op wrappers over the C ABI used by the host modules."""

import ctypes as C

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


class GemmProblem(C.Structure):
    """Mirror of `lsrm_gemm_problem` (include/lsrm_b200.h)."""
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
                ("a", C.c_void_p), ("lda", C.c_int64), ("bt", C.c_void_p), ("ldb", C.c_int64),
                ("c", C.c_void_p), ("ldc", C.c_int64), ("bias", C.c_void_p),
                ("res", C.c_void_p), ("ldr", C.c_int64), ("flags", C.c_int32),
                ("reserved", C.c_int32)]


GEMM_OUT_F32, GEMM_BIAS_F32, GEMM_RES_F32, GEMM_GELU, GEMM_A_MN, GEMM_B_MN = 1, 2, 4, 8, 16, 32
_MAX_PROBLEMS = 32   # problems per lsrm_gemm_tc launch


def gemm_problem(a: torch.Tensor, bt: torch.Tensor, out: torch.Tensor, bias=None, res=None,
                 gelu=False, a_mn=False, b_mn=False, k=None) -> GemmProblem:
    """One tcgen05 GEMM problem: out = act(a @ bt^T + bias) + res, with a
    [m,k] and bt [n,k] bf16 (K contiguous: bt is the weight transposed).
    a_mn: `a` is A^T as stored, [k,m]; b_mn: `bt` is B as stored, [k,n]
    (MN-major operands, no transposed copy).  k: the contraction length when
    it is shorter than an MN-major operand's rows (rows past it read as 0
    only past the operand's end, so pass k = rows unless padding is zero)."""
    m, ka = (a.shape[1], a.shape[0]) if a_mn else a.shape
    n, kb = (bt.shape[1], bt.shape[0]) if b_mn else bt.shape
    assert ka == kb and a.dtype == bt.dtype == torch.bfloat16, (ka, kb)
    k = ka if k is None else k
    assert a.stride(1) == 1 and bt.stride(1) == 1 and out.stride(1) == 1
    assert tuple(out.shape) == (m, n)
    flags = (GEMM_OUT_F32 if out.dtype == torch.float32 else 0) | (GEMM_GELU if gelu else 0)
    flags |= (GEMM_A_MN if a_mn else 0) | (GEMM_B_MN if b_mn else 0)
    if bias is not None:
        flags |= GEMM_BIAS_F32 if bias.dtype == torch.float32 else 0
    if res is not None:
        assert res.stride(1) == 1 and tuple(res.shape) == (m, n)
        flags |= GEMM_RES_F32 if res.dtype == torch.float32 else 0
    prob = GemmProblem(m, n, k, a.data_ptr(), a.stride(0), bt.data_ptr(), bt.stride(0),
                       out.data_ptr(), out.stride(0), D.ptr(bias), D.ptr(res),
                       res.stride(0) if res is not None else 0, flags, 0)
    prob.keep = (a, bt, out, bias, res)   # the descriptor holds raw pointers
    return prob


def gemm_tc(problems) -> None:
    """Run GemmProblems as ONE persistent tcgen05 launch (csrc/gemm_tc.cu)."""
    arr = (GemmProblem * len(problems))(*problems)
    call("lsrm_gemm_tc", C.cast(arr, C.c_void_p), len(problems), D.stream())


def gemm_bf16(a: torch.Tensor, bt: torch.Tensor, out=None, out_dtype=torch.bfloat16, bias=None,
              res=None, gelu=False) -> torch.Tensor:
    """a [m,k] @ bt[n,k]^T on the tcgen05 GEMM."""
    out = D.empty((a.shape[0], bt.shape[0]), out_dtype) if out is None else out
    gemm_tc([gemm_problem(a, bt, out, bias, res, gelu)])
    return out


def transpose_bf16(x: torch.Tensor, pad_to: int = 8) -> torch.Tensor:
    """[r, c] f32 -> [c, r_pad] bf16 (zero rows r..r_pad): a K-major operand."""
    r, c = x.shape
    rp = (r + pad_to - 1) // pad_to * pad_to
    out = D.empty((c, rp), torch.bfloat16)
    call("lsrm_transpose_cast_bf16", x.data_ptr(), x.stride(0), r, c, out.data_ptr(), rp,
         D.stream())
    return out


def cast_pad_bf16(x: torch.Tensor, cols_pad: int) -> torch.Tensor:
    """[r, c] f32 -> [r, cols_pad] bf16, zero columns c..cols_pad."""
    r, c = x.shape
    if cols_pad == c and x.is_contiguous():
        return cast(x, torch.bfloat16)
    out = D.empty((r, cols_pad), torch.bfloat16)
    xt = x.t().contiguous()                 # [c, r] f32 (cold path: unaligned K)
    call("lsrm_transpose_cast_bf16", xt.data_ptr(), xt.stride(0), c, r, out.data_ptr(),
         cols_pad, D.stream())
    return out


def gemm_train(a: torch.Tensor, b: torch.Tensor, trans_a=False, trans_b=False, out=None,
               beta=0.0, cache: dict = None) -> torch.Tensor:
    """fp32 out (+)= op(a) @ op(b) on the tcgen05 GEMM, bf16 operands, fp32
    accumulation (the training path's GEMMs; gemm_ex's signature; f32 or
    bf16 inputs).  Operands are only cast: a transposed operand is passed MN-major (as stored), so the
    weight-gradient GEMMs X^T . dY need no transposed copies.  A K-major
    operand with k % 8 != 0 is zero-padded (the MN-major one gets zero rows).
    `cache` (optional dict) reuses the bf16 copy of a tensor cast earlier in
    the same backward pass.  N must be a multiple of 8 (every training GEMM's
    N is: d, 4d, n_gates*d, h_kv*d_h)."""
    assert a.dtype in (torch.float32, torch.bfloat16) and b.dtype in (torch.float32,
                                                                     torch.bfloat16)
    assert beta in (0.0, 1.0)
    m, k = (a.shape[1], a.shape[0]) if trans_a else a.shape
    k2, n = (b.shape[1], b.shape[0]) if trans_b else b.shape
    assert k == k2 and n % 8 == 0, (k, k2, n)
    acc = out is not None and beta == 1.0
    dst = out if out is not None else D.empty((m, n), torch.float32)
    if m == 0 or n == 0:
        return dst
    a_mn, b_mn = trans_a, not trans_b
    kp = k if (a_mn and b_mn) else (k + 7) // 8 * 8

    def bf(x, mn):
        plain = kp == k and (x.is_contiguous() or not mn)   # the copy is cast(x) as stored
        key = (x.data_ptr(), tuple(x.shape), tuple(x.stride())) + (() if plain else (mn, kp))
        if cache is not None and key in cache:
            return cache[key][1]
        if x.dtype == torch.bfloat16 and plain and x.is_contiguous():
            return x                         # already a bf16 operand as stored
        if x.dtype == torch.bfloat16:
            x = cast(x.contiguous(), torch.float32)   # cold path: re-pad through f32
        if not mn:                           # K-major [rows, k] -> [rows, kp]
            y = cast_pad_bf16(x, kp)
        elif x.shape[1] % 8:                 # MN-major, row stride padded to 8 (cold path)
            cols = x.shape[1]
            y = cast_pad_bf16(x, (cols + 7) // 8 * 8)
            if kp != k:
                y = torch.cat([y, y.new_zeros((kp - k, y.shape[1]))])
            y = y[:, :cols]
        elif kp == k:                        # MN-major [k, cols] as stored
            y = cast(x.contiguous(), torch.bfloat16)
        else:                                # MN-major with kp - k zero rows
            y = D.empty((kp, x.shape[1]), torch.bfloat16)
            y[k:].zero_()
            call("lsrm_cast", 1, x.contiguous().data_ptr(), y.data_ptr(), x.numel(), D.stream())
        if cache is not None:
            cache[key] = (x, y)              # x kept alive: its address cannot be reused
        return y
    A, B = bf(a, a_mn), bf(b, b_mn)
    # split K when the output has too few 256 x 256 tiles to fill the GPU (the
    # weight gradients: m x n = d x d, k = tokens); partial products go to a
    # workspace and are summed in slice order (deterministic)
    tiles = -(-m // 256) * -(-n // 256)
    n_split = min(_MAX_PROBLEMS, -(-74 // tiles), kp // 512) if tiles < 74 else 1
    if n_split > 1 and (m * n) % 4 == 0:
        step = (-(-kp // n_split) + 63) // 64 * 64   # multiples of BK: 16-byte aligned slices
        cuts = [min(kp, i * step) for i in range(n_split + 1)]
        cuts = [c for i, c in enumerate(cuts) if i == 0 or c > cuts[i - 1]]
        parts = D.empty((len(cuts) - 1, m, n), torch.float32)
        probs = []
        for s_, (k0, k1) in enumerate(zip(cuts[:-1], cuts[1:])):
            As = A[k0:k1] if a_mn else A[:, k0:k1]
            Bs = B[k0:k1] if b_mn else B[:, k0:k1]
            probs.append(gemm_problem(As, Bs, parts[s_], a_mn=a_mn, b_mn=b_mn))
        gemm_tc(probs)
        if not dst.is_contiguous():
            raise ValueError("gemm_train: split-K needs a contiguous output")
        call("lsrm_sum_slices_f32", parts.data_ptr(), len(probs), m * n, dst.data_ptr(), int(acc),
             D.stream())
        return dst
    gemm_tc([gemm_problem(A, B, dst, res=dst if acc else None, a_mn=a_mn, b_mn=b_mn)])
    return dst
    kp = (k + 7) // 8 * 8
    am = transpose_bf16(a) if trans_a else cast_pad_bf16(a, kp)      # [m, kp]
    bt = cast_pad_bf16(b, kp) if trans_b else transpose_bf16(b)      # [n, kp]
    gemm_tc([gemm_problem(am, bt, dst, res=dst if acc else None)])
    return dst
