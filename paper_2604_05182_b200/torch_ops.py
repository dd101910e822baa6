"""torch.library custom ops over the C ABI (the thin "torch custom-op layer"
of the north star): one branch of NSA attention as a tensor-level op, so the
kernels compose with ordinary PyTorch code, autograd and `torch.library`
tooling.

    torch.ops.lsrm.branch_attention(q, k, v, mode, offs, rows, count, own_row)
        fp32 reference numerics (`nsa_attention.py:84-207`; csrc/attn_f32.cu).
    torch.ops.lsrm.sparse_attention(q, k, v, mode, offs, rows, count, own_row)
        -> (out, lse): bf16 tensor-core forward (csrc/attn_bwd_mma.cu) with a
        registered backward (dq, dk, dv through the deterministic key-major
        pass), i.e. a differentiable block-sparse attention op.

Shapes: q [nq, hq, dh], k / v [nk, hkv, dh] (f32); mode 0 attends every key
row (cmp), 1 the key rows of the resolved blocks rows[i, :count[i]] (sel;
offs [B + 1] are the blocks' row offsets into k / v), 2 the block own_row[i]
(win).  Index tensors are int64 offs and int32 rows / count / own_row.
"""

from typing import Optional, Tuple

import torch

from . import _dev as D
from . import _ops
from ._native import call, lib
from .errors import require

Tensor = torch.Tensor


def _check(q, k, v, mode, offs, rows, count, own_row):
    require(q.dim() == 3 and k.dim() == 3 and k.shape == v.shape, "q [nq,hq,dh], k/v [nk,hkv,dh]")
    require(q.shape[2] == k.shape[2] and q.shape[1] % k.shape[1] == 0, "head geometry mismatch")
    require(mode in (0, 1, 2), "mode must be 0 (cmp), 1 (sel) or 2 (win)")
    require(mode == 0 or offs is not None, "sel / win need block offsets")
    require(mode != 1 or (rows is not None and count is not None), "sel needs rows and count")
    require(mode != 2 or own_row is not None, "win needs own_row")


@torch.library.custom_op("lsrm::branch_attention", mutates_args=())
def branch_attention(q: Tensor, k: Tensor, v: Tensor, mode: int, offs: Optional[Tensor],
                     rows: Optional[Tensor], count: Optional[Tensor],
                     own_row: Optional[Tensor]) -> Tensor:
    _check(q, k, v, mode, offs, rows, count, own_row)
    q, k, v = (t.contiguous().float() for t in (q, k, v))
    nq, hq, dh = q.shape
    out = torch.empty_like(q)
    kmax = int(rows.shape[1]) if rows is not None else 1
    call("lsrm_attention_f32", mode, q.data_ptr(), nq, hq, int(k.shape[1]), dh, k.data_ptr(),
         v.data_ptr(), int(k.shape[0]), D.ptr(offs), D.ptr(rows), D.ptr(count), kmax,
         D.ptr(own_row), None, None, 0, out.data_ptr(), D.stream())
    return out


@branch_attention.register_fake
def _(q, k, v, mode, offs, rows, count, own_row):
    return torch.empty_like(q, dtype=torch.float32)


@torch.library.custom_op("lsrm::sparse_attention", mutates_args=())
def sparse_attention(q: Tensor, k: Tensor, v: Tensor, mode: int, offs: Optional[Tensor],
                     rows: Optional[Tensor], count: Optional[Tensor],
                     own_row: Optional[Tensor]) -> Tuple[Tensor, Tensor]:
    _check(q, k, v, mode, offs, rows, count, own_row)
    nq, hq, dh = q.shape
    hkv = int(k.shape[1])
    qb, kb, vb = (_ops.cast(t.contiguous().float(), torch.bfloat16) for t in (q, k, v))
    out = torch.empty((nq, hq, dh), dtype=torch.float32, device=q.device)
    lse = torch.empty((nq, hq), dtype=torch.float32, device=q.device)
    kmax = int(rows.shape[1]) if rows is not None else 1
    call("lsrm_attention_fwd_mma", mode, qb.data_ptr(), nq, hq, hkv, dh, kb.data_ptr(),
         vb.data_ptr(), int(k.shape[0]), D.ptr(offs), D.ptr(rows), D.ptr(count), kmax,
         D.ptr(own_row), out.data_ptr(), lse.data_ptr(), D.stream())
    return out, lse


@sparse_attention.register_fake
def _(q, k, v, mode, offs, rows, count, own_row):
    nq, hq, dh = q.shape
    return (q.new_empty((nq, hq, dh), dtype=torch.float32),
            q.new_empty((nq, hq), dtype=torch.float32))


def _setup(ctx, inputs, output):
    q, k, v, mode, offs, rows, count, own_row = inputs
    out, lse = output
    ctx.mode = mode
    ctx.save_for_backward(q, k, v, out, lse, offs, rows, count, own_row)


def _backward(ctx, dout, dlse):
    q, k, v, out, lse, offs, rows, count, own_row = ctx.saved_tensors
    mode = ctx.mode
    nq, hq, dh = q.shape
    nk, hkv = int(k.shape[0]), int(k.shape[1])
    st = D.stream()
    qb, kb, vb = (_ops.cast(t.contiguous().float(), torch.bfloat16) for t in (q, k, v))
    do32 = dout.contiguous().float()
    dob = _ops.cast(do32, torch.bfloat16)
    dq = torch.zeros((nq, hq, dh), dtype=torch.float32, device=q.device)
    dk = torch.zeros((nk, hkv, dh), dtype=torch.float32, device=q.device)
    dv = torch.zeros_like(dk)
    n_rows = int(offs.shape[0]) - 1 if offs is not None else 1
    max_row = int((offs[1:] - offs[:-1]).max()) if offs is not None and n_rows > 0 else 1
    t_offs = t_q = None
    if mode in (1, 2):   # per kv row, its queries (deterministic transposed index)
        r = rows if mode == 1 else own_row.reshape(-1, 1)
        c = count if mode == 1 else torch.ones(nq, dtype=torch.int32, device=q.device)
        kmx = int(r.shape[1])
        t_offs = torch.empty(n_rows + 1, dtype=torch.int64, device=q.device)
        t_q = torch.empty(max(nq * kmx, 1), dtype=torch.int32, device=q.device)
        wsb = lib().lsrm_transpose_rows_workspace(nq, kmx)
        tws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=q.device)
        call("lsrm_transpose_rows", r.data_ptr(), c.data_ptr(), nq, kmx, n_rows,
             t_offs.data_ptr(), t_q.data_ptr(), tws.data_ptr(), wsb, st)
    if mode == 0:
        n_slices = max(1, min(nq // 64, -(-8 * 148 // (-(-nk // 64) * hkv))))
    else:
        n_slices = max(1, min(4, nq // 1024))
    wsb = lib().lsrm_attention_bwd_workspace(nq, hq, nk, hkv, dh, n_slices)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=q.device)
    kmax = int(rows.shape[1]) if rows is not None else 1
    call("lsrm_attention_bwd_mma", mode, qb.data_ptr(), dob.data_ptr(), do32.data_ptr(),
         out.data_ptr(), lse.data_ptr(), nq, hq, hkv, dh, kb.data_ptr(), vb.data_ptr(), nk,
         D.ptr(offs), n_rows, max_row, D.ptr(rows), D.ptr(count), kmax, D.ptr(own_row),
         n_slices, D.ptr(t_offs), D.ptr(t_q), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
         ws.data_ptr(), wsb, st)
    return dq, dk, dv, None, None, None, None, None


sparse_attention.register_autograd(_backward, setup_context=_setup)
