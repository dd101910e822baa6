"""Training of the Stage-2 block: one gated NSA use, the four uses of a
layer, and the full block.

The reference is inference-only: its NSA use (`nsa_attention.py:287-327`) has
no backward.  This module adds one on the GPU path: an fp32
forward that keeps its intermediates (same kernels as `nsa_cross_attention`)
and a backward built from

  * `lsrm_attention_bwd_f32`  - the three branches (recompute; a query-major
                                dQ pass and a key-major dK/dV pass, no atomics),
  * `lsrm_gate_merge_bwd_f32` - the sigmoid-gated merge,
  * `lsrm_res_block_bwd_f32`  - the compression ResBlock under the block mean,
  * every projection / weight gradient: `lsrm_gemm_f32_ex` (cuBLAS fp32) on
                                the reference-precision path, the tcgen05
                                GEMM (`_ops.gemm_train`, bf16 operands, fp32
                                accumulation) on the fast path,

wrapped in a `torch.autograd.Function` so a `torch.optim` optimizer can step
the weights. `SparseBlockModule` adds the block around the uses (add +
LayerNorm, use gates, gated mixture + LayerNorm, FFN) with the row kernels of
csrc/block.cu forward and csrc/train_block.cu backward.  Gradients are checked against the float64 autograd restatement
`oracle/torch_nsa.py` (tests/test_training.py).

Inputs and selections are fixed per call: routing (which blocks each query
attends to) is not differentiated, exactly as in NSA training.
"""

from dataclasses import dataclass

import ctypes as C

import numpy as np
import torch

from . import _dev as D
from . import _ops
from ._native import call, lib
from .block_partition import BlockPartition, compress_rows
from .errors import require
from .nsa_attention import NsaWeights, _attn, resolve_rows, selection_rows
from .tensor_core import AttentionParams

PARAM_NAMES = ("w_q", "w_k", "w_v", "w_o", "gate_w", "gate_b",
               "ck_w1", "ck_b1", "ck_w2", "ck_b2", "cv_w1", "cv_b1", "cv_w2", "cv_b2")


@dataclass
class _Spec:
    params: AttentionParams
    n_gates: int
    part_q: BlockPartition
    part_kv: BlockPartition
    rows: torch.Tensor
    count: torch.Tensor
    fast: bool = False    # tensor-core (bf16) attention backward
    transposed: tuple = None   # (offs, queries) per kv row, built on first use
    # block-aware sequence parallelism (seq_parallel.py): the queries are the
    # rows of the query blocks this rank owns, and K/V are all-gathered from
    # their owners (their gradients reduce-scattered back) by kv_exchange
    q_local: "LocalQueries" = None
    kv_exchange: object = None


@dataclass
class LocalQueries:
    """The queries of the query blocks one rank owns: local rows are the owned
    blocks' tokens in block-major order (`seq_parallel.py` shards whole
    blocks).  own_rows: each local query's block row in the (global)
    partition; win_offs / win_ids: the local rows of every block (empty for
    blocks other ranks own) for the window branch's key-major pass."""
    part: BlockPartition
    owned: np.ndarray
    loc_tok: np.ndarray
    own_rows: torch.Tensor
    win_offs: torch.Tensor
    win_ids: torch.Tensor

    @property
    def n(self) -> int:
        return int(self.loc_tok.size)


def local_query_arrays(part: BlockPartition, owned):
    """Host arrays of LocalQueries: (owned rows ascending, global token id of
    every local row, each local row's block row, per-block offsets into the
    local rows (empty for blocks other ranks own), local row ids)."""
    owned = np.sort(np.asarray(owned, np.int64))
    occ = part.occupancy.astype(np.int64)
    loc_tok = (np.concatenate([part.tokens_in_row(int(r)) for r in owned]).astype(np.int64)
               if owned.size else np.zeros(0, np.int64))
    own_rows = np.repeat(owned, occ[owned]).astype(np.int32)
    counts = np.zeros(part.n_occupied, np.int64)
    counts[owned] = occ[owned]
    win_offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    win_ids = np.arange(loc_tok.size, dtype=np.int32)   # owned blocks in ascending order
    return owned, loc_tok, own_rows, win_offs, win_ids


def local_queries(part: BlockPartition, owned) -> LocalQueries:
    owned, loc_tok, own_rows, win_offs, win_ids = local_query_arrays(part, owned)
    return LocalQueries(part, owned, loc_tok, D.dev(own_rows), D.dev(win_offs), D.dev(win_ids))


def q_local_rows(q_local: LocalQueries, table):
    """The routing rows of the local queries (cached per table)."""
    cache = q_local.__dict__.setdefault("_rows", {})
    hit = cache.get(id(table.rows))
    if hit is None or hit[0] is not table.rows:
        idx = D.dev(q_local.loc_tok)
        rows = _ops.gather_rows(table.rows, idx)
        count = _ops.gather_rows(table.count.reshape(-1, 1), idx).reshape(-1)
        hit = (table.rows, rows, count)
        cache[id(table.rows)] = hit
    return hit[1], hit[2]


def _own_rows(spec: "_Spec"):
    if spec.n_gates != 3:
        return None
    return spec.q_local.own_rows if spec.q_local is not None else spec.part_q.dev("row_of_token")


def _mma_ok(spec: _Spec) -> bool:
    p = spec.params
    return spec.fast and p.head_dim in (16, 32, 64) and p.n_q_heads // p.n_kv_heads <= 16


def _fused_ok(spec: _Spec) -> bool:
    """Head geometries the fused tcgen05 forward takes (engine.py / DESIGN §3)."""
    from .fastpath import supported
    return supported(spec.params) and int(spec.rows.shape[1]) * (128 * spec.params.n_kv_heads //
                                                                  spec.params.n_q_heads) <= 256


_FUSED_PLANS = {}


def _fused_plan(spec: _Spec):
    """Tiles / tile-order rows / LPT item queue of the fused forward for this
    use's routing (cached per routing tensor: the plan is fixed across steps).
    Block tiles signature-sorted inside each query block, as the engine's
    default (engine.py `_build_attention_queue`); tile positions map to
    token-order query rows through `perm`."""
    from .engine import ROW_PAD, query_tiles, stream_meta
    key = (id(spec.rows), id(spec.part_q), id(spec.part_kv), spec.n_gates, id(spec.q_local))
    hit = _FUSED_PLANS.get(key)
    if hit is not None and hit["rows_ref"] is spec.rows:
        return hit
    p = spec.params
    G = p.n_q_heads // p.n_kv_heads
    self_use = spec.n_gates == 3
    pq, pk = spec.part_q, spec.part_kv
    mk = stream_meta(pk)
    rows_tok = D.host(spec.rows).astype(np.int32)
    cnt_tok = D.host(spec.count).astype(np.int32)
    ql = spec.q_local
    if ql is None:
        tok_q = pq.block_token_ids.astype(np.int64)
        blk = np.repeat(np.arange(pq.n_occupied), pq.occupancy.astype(np.int64))
    else:   # local rows are already block-major over the owned blocks
        tok_q = np.arange(ql.n, dtype=np.int64)
        blk = np.repeat(np.arange(ql.owned.size), pq.occupancy.astype(np.int64)[ql.owned])
    rows_bm = rows_tok[tok_q]
    key_s = np.sort(np.where(rows_bm >= 0, rows_bm, np.iinfo(np.int32).max), axis=1)
    sig = tuple(key_s[:, j] for j in reversed(range(key_s.shape[1])))
    perm_bm = np.lexsort(sig + (blk,))
    perm_tok = tok_q[perm_bm]
    tiles = query_tiles(pq, G, self_use, None if ql is None else ql.owned)
    rows_t = np.ascontiguousarray(rows_tok[perm_tok])
    cnt_t = np.ascontiguousarray(cnt_tok[perm_tok])
    padlen = np.diff(mk.pad_off_host)
    cmp_rows = (mk.n_blocks + ROW_PAD - 1) // ROW_PAD * ROW_PAD
    costs = []
    for first, tc, own, _ in tiles:
        r = rows_t[first:first + tc].ravel()
        c = cmp_rows + int(padlen[np.unique(r[r >= 0])].sum())
        c += int(padlen[own]) if (own >= 0 and self_use) else 0
        costs.append(c)
    hkv = p.n_kv_heads
    costs = np.repeat(np.asarray(costs, np.int64), hkv)
    codes = np.arange(costs.size, dtype=np.int64)
    order = codes[np.lexsort((codes, -costs))].astype(np.int32)
    plan = {"rows_ref": spec.rows, "meta": mk, "tiles": D.dev(tiles), "rows": D.dev(rows_t),
            "count": D.dev(cnt_t), "perm": D.dev(perm_tok.astype(np.int32)),
            "order": D.dev(order), "counter": D.zeros((1,), torch.int32),
            "kc_rows_pad": cmp_rows}
    if len(_FUSED_PLANS) > 32:
        _FUSED_PLANS.clear()
    _FUSED_PLANS[key] = plan
    return plan


def _fused_attention(spec: _Spec, q_bf, k, v, kc, vc, logits):
    """Fused tcgen05 forward of one use: per-branch outputs f32 [ng, n, d],
    per-branch lse f32 [ng, n, hq] and the gated merge (bf16 [n, d])."""
    from .engine import NsaUse
    p = spec.params
    n, d = q_bf.shape
    hq, hkv, dh = p.n_q_heads, p.n_kv_heads, p.head_dim
    ng = spec.n_gates
    plan = _fused_plan(spec)
    mk = plan["meta"]
    pk = spec.part_kv
    st = D.stream()
    m = int(k.shape[0])
    width = hkv * dh
    k_il = D.empty((hkv, mk.n_rows_pad, dh), torch.bfloat16)
    v_il = D.zeros((hkv, mk.n_rows_pad, dh + 16), torch.bfloat16)
    for src, dst, ones in ((k, k_il, 0), (v, v_il, 16)):
        call("lsrm_kv_interleave", 0, src.data_ptr(), width, m, hkv, dh, ones,
             pk.dev("block_token_ids").data_ptr(), mk.kv_off.data_ptr(), mk.n_blocks,
             mk.pad_off.data_ptr(), mk.n_rows_pad, dst.data_ptr(), st)
    bp = plan["kc_rows_pad"]
    kc_il = D.empty((hkv, bp, dh), torch.bfloat16)
    vc_il = D.zeros((hkv, bp, dh + 16), torch.bfloat16)
    for src, dst, ones in ((kc, kc_il, 0), (vc, vc_il, 16)):
        call("lsrm_kv_interleave", 0, src.data_ptr(), width, mk.n_blocks, hkv, dh, ones, None,
             None, 0, None, bp, dst.data_ptr(), st)
    gl = _ops.cast(logits, torch.bfloat16)
    merged = D.empty((n, d), torch.bfloat16)
    o_all = D.empty((ng, n, d), torch.float32)
    lse_all = D.empty((ng, n, hq), torch.float32)
    tiles = plan["tiles"]
    use = NsaUse(q_bf.data_ptr(), q_bf.stride(0), n, k_il.data_ptr(), v_il.data_ptr(),
                 mk.pad_off.data_ptr(), mk.kv_off.data_ptr(), mk.n_rows_pad, kc_il.data_ptr(),
                 vc_il.data_ptr(), mk.n_blocks, tiles.data_ptr(), int(tiles.shape[0]),
                 plan["rows"].data_ptr(), plan["count"].data_ptr(), int(spec.rows.shape[1]),
                 gl.data_ptr(), gl.stride(0), 0, ng, merged.data_ptr(), plan["perm"].data_ptr(),
                 0, 0, None, o_all.data_ptr(), lse_all.data_ptr())
    order = plan["order"]
    call("lsrm_nsa_attention_tc_multi", C.byref(use), 1, hq, hkv, dh, order.data_ptr(),
         int(order.shape[0]), plan["counter"].data_ptr(), st)
    return o_all, lse_all, merged


def _forward(spec: _Spec, x, kv, P):
    p = spec.params
    n, d = x.shape
    m = int(kv.shape[0])
    hq, hkv, dh = p.n_q_heads, p.n_kv_heads, p.head_dim
    width = hkv * dh
    part = spec.part_kv
    fast = _mma_ok(spec)
    mm = _ops.gemm_train if fast else _ops.gemm_ex   # fast: bf16 tcgen05 GEMMs
    q = mm(x, P["w_q"])
    k = mm(kv, P["w_k"])
    v = mm(kv, P["w_v"])
    if spec.kv_exchange is not None:   # All-gather-KV: every block's K/V rows
        k, v = spec.kv_exchange.gather(k), spec.kv_exchange.gather(v)
        m = int(k.shape[0])
    ck = [P[f"ck_{s}"] for s in ("w1", "b1", "w2", "b2")]
    cv = [P[f"cv_{s}"] for s in ("w1", "b1", "w2", "b2")]
    kc = compress_rows(k, width, m, width, ck, part)
    vc = compress_rows(v, width, m, width, cv, part)
    tok, offs = part.dev("block_token_ids"), part.dev("block_offsets")
    k_bm, v_bm = _ops.gather_rows(k, tok), _ops.gather_rows(v, tok)
    B = part.n_occupied
    own = _own_rows(spec)
    saved = dict(x=x, kv=kv, q=q, k=k, v=v, kc=kc, vc=vc, k_bm=k_bm, v_bm=v_bm, ck=ck, cv=cv)
    if fast and _fused_ok(spec):
        # the three branches, their gated merge and each branch's lse in ONE
        # launch of the fused tcgen05 forward (csrc/attn_tc.cu); the bias is
        # folded into the gate logits (so the backward sees a zero bias)
        bf = {name: _ops.cast(saved[name], torch.bfloat16)
              for name in ("q", "kc", "vc", "k_bm", "v_bm")}
        logits = D.empty((n, spec.n_gates * d), torch.float32)
        _ops.gemm_tc([_ops.gemm_problem(_ops.cast(x.contiguous(), torch.bfloat16),
                                        _ops.cast(P["gate_w"].contiguous(), torch.bfloat16),
                                        logits, bias=P["gate_b"], b_mn=True)])
        o_all, lse_all, merged = _fused_attention(spec, bf["q"], k, v, kc, vc, logits)
        outs = [o_all[b] for b in range(spec.n_gates)]
        saved.update(bf=bf, lse=[lse_all[b] for b in range(spec.n_gates)])
        out = mm(merged, P["w_o"])
        o = [t.view(n, d) for t in outs] + [None] * (3 - len(outs))
        saved.update(outs=o, logits=logits, merged=merged, gate_b_eff=torch.zeros_like(P["gate_b"]))
        return out, saved
    if fast:
        # branches on tensor cores (bf16 operands); lse kept for the backward
        bf = {name: _ops.cast(saved[name], torch.bfloat16)
              for name in ("q", "kc", "vc", "k_bm", "v_bm")}
        outs, lses = [], []
        for mode, kn, vn, nk in ((0, "kc", "vc", B), (1, "k_bm", "v_bm", m),
                                 (2, "k_bm", "v_bm", m))[:spec.n_gates]:
            o_b = D.empty((n, hq, dh), torch.float32)
            lse = D.empty((n, hq), torch.float32)
            call("lsrm_attention_fwd_mma", mode, bf["q"].data_ptr(), n, hq, hkv, dh,
                 bf[kn].data_ptr(), bf[vn].data_ptr(), nk, offs.data_ptr() if mode else None,
                 D.ptr(spec.rows) if mode == 1 else None,
                 D.ptr(spec.count) if mode == 1 else None, int(spec.rows.shape[1]),
                 D.ptr(own) if mode == 2 else None, o_b.data_ptr(), lse.data_ptr(), D.stream())
            outs.append(o_b)
            lses.append(lse)
        saved.update(bf=bf, lse=lses)
    else:
        q3 = q.view(n, hq, dh)
        outs = [_attn(0, q3, kc.view(B, hkv, dh), vc.view(B, hkv, dh), p),
                _attn(1, q3, k_bm.view(m, hkv, dh), v_bm.view(m, hkv, dh), p, offs=offs,
                      rows=spec.rows, count=spec.count)]
        if spec.n_gates == 3:
            outs.append(_attn(2, q3, k_bm.view(m, hkv, dh), v_bm.view(m, hkv, dh), p,
                              offs=offs, own_row=own))
    logits = mm(x, P["gate_w"])
    merged = D.empty((n, d), torch.float32)
    o = [t.view(n, d) for t in outs] + [None] * (3 - len(outs))
    call("lsrm_gated_merge_fast_f32" if fast else "lsrm_gated_merge_f32", logits.data_ptr(),
         logits.stride(0), P["gate_b"].data_ptr(), spec.n_gates, D.ptr(o[0]), D.ptr(o[1]),
         D.ptr(o[2]), n, d, merged.data_ptr(), D.stream())
    out = mm(merged, P["w_o"])
    saved.update(outs=o, logits=logits, merged=merged, gate_b_eff=P["gate_b"])
    return out, saved


def _colsum(t):
    """Column sums (bias gradients): deterministic fixed-order kernel."""
    return _colsum_dev(t.contiguous())


def _backward(spec: _Spec, P, s, dout):
    """Gradients of every input and parameter (dict keyed like PARAM_NAMES
    plus "x", "kv")."""
    p = spec.params
    n, d = s["x"].shape
    m = int(s["k"].shape[0])   # every kv row (all-gathered under sequence parallelism)
    hq, hkv, dh = p.n_q_heads, p.n_kv_heads, p.head_dim
    width = hkv * dh
    ng = spec.n_gates
    part = spec.part_kv
    B = part.n_occupied
    st = D.stream()
    g = {}
    fast = _mma_ok(spec)

    bf_cache = {}   # bf16 copies of operands used by several GEMMs of this pass

    def gx(a, b, **kw):
        if fast:
            return _ops.gemm_train(a, b, cache=bf_cache, **kw)
        return _ops.gemm_ex(a, b, **kw)
    # out = merged W_o
    dmerged = gx(dout, P["w_o"], trans_b=True)
    g["w_o"] = gx(s["merged"], dout, trans_a=True)
    # gated merge
    do = [D.empty((n, d), torch.float32) for _ in range(ng)] + [None] * (3 - ng)
    dz = D.empty((n, ng * d), torch.float32)
    o = s["outs"]
    call("lsrm_gate_merge_bwd_f32", s["logits"].data_ptr(), s["logits"].stride(0),
         s["gate_b_eff"].data_ptr(), ng, D.ptr(o[0]), D.ptr(o[1]), D.ptr(o[2]),
         dmerged.data_ptr(), n, d, int(fast), D.ptr(do[0]), D.ptr(do[1]), D.ptr(do[2]),
         dz.data_ptr(), st)
    g["gate_w"] = gx(s["x"], dz, trans_a=True)
    g["gate_b"] = _colsum(dz)
    dx = gx(dz, P["gate_w"], trans_b=True)
    # branches
    dq = D.zeros((n, d), torch.float32)
    dkc, dvc = D.zeros((B, width), torch.float32), D.zeros((B, width), torch.float32)
    dk_bm, dv_bm = D.zeros((m, width), torch.float32), D.zeros((m, width), torch.float32)
    offs = part.dev("block_offsets")
    kmax = int(spec.rows.shape[1])

    max_occ = int(np.max(part.occupancy)) if B else 1

    use_mma = fast
    bf = s.get("bf")
    # key-major pass of the mma path walks each kv row's own query list:
    # sel through the transposed routing index, win through the block's tokens
    lists = {0: (None, None), 1: (None, None), 2: (None, None)}
    if use_mma:
        if spec.transposed is None:
            kmx = int(spec.rows.shape[1])
            t_offs = D.empty((B + 1,), torch.int64)
            t_q = D.empty((max(n * kmx, 1),), torch.int32)
            wsb = lib().lsrm_transpose_rows_workspace(n, kmx)
            tws = D.empty((max(wsb, 1),), torch.uint8)
            call("lsrm_transpose_rows", spec.rows.data_ptr(), spec.count.data_ptr(), n, kmx, B,
                 t_offs.data_ptr(), t_q.data_ptr(), tws.data_ptr(), wsb, st)
            spec.transposed = (t_offs, t_q)
        lists[1] = spec.transposed
        if ng == 3 and spec.q_local is not None:
            lists[2] = (spec.q_local.win_offs, spec.q_local.win_ids)
        elif ng == 3:
            lists[2] = (part.dev("block_offsets"), part.dev("block_token_ids").to(torch.int32))

    def bwd(mode, b, k, v, nk, dk, dv, rows=None, count=None, own=None):
        # cmp has few keys and every query: slice the queries so the key-major
        # pass has >= ~8 CTAs per SM (148 SMs)
        if mode == 0:
            tiles = -(-nk // 64) * hkv
            n_slices = max(1, min(n // 64, -(-8 * 148 // tiles)))
        else:
            n_slices = max(1, min(4, n // 1024))
        ws_bytes = lib().lsrm_attention_bwd_workspace(n, hq, nk, hkv, dh, n_slices)
        ws = D.empty((ws_bytes,), torch.uint8)
        head = (nk, offs.data_ptr() if mode else None, B, max_occ, D.ptr(rows), D.ptr(count),
                kmax, D.ptr(own), n_slices)
        tail = (dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws_bytes, st)
        if use_mma:
            dob = _ops.cast(do[b], torch.bfloat16)
            call("lsrm_attention_bwd_mma", mode, bf["q"].data_ptr(), dob.data_ptr(),
                 do[b].data_ptr(), o[b].data_ptr(), s["lse"][b].data_ptr(), n, hq, hkv, dh,
                 bf[k].data_ptr(), bf[v].data_ptr(), *head, D.ptr(lists[mode][0]),
                 D.ptr(lists[mode][1]), *tail)
        else:
            call("lsrm_attention_bwd_f32", mode, s["q"].data_ptr(), do[b].data_ptr(),
                 o[b].data_ptr(), n, hq, hkv, dh, s[k].data_ptr(), s[v].data_ptr(), *head,
                 *tail)
    bwd(0, 0, "kc", "vc", B, dkc, dvc)
    bwd(1, 1, "k_bm", "v_bm", m, dk_bm, dv_bm, rows=spec.rows, count=spec.count)
    if ng == 3:
        bwd(2, 2, "k_bm", "v_bm", m, dk_bm, dv_bm, own=_own_rows(spec))
    tok = part.dev("block_token_ids")
    dk = _ops.scatter_rows(dk_bm, tok, D.empty((m, width), torch.float32))
    dv = _ops.scatter_rows(dv_bm, tok, D.empty((m, width), torch.float32))
    # compression ResBlocks under the block mean (accumulate into dk / dv)
    row_of = part.dev("row_of_token")
    occ = part.dev("occupancy")
    require(occ.dtype == torch.int64, "occupancy must be int64")
    for tag, t, dc, dt, cw in (("ck", s["k"], dkc, dk, s["ck"]), ("cv", s["v"], dvc, dv, s["cv"])):
        dr, dz1, h = (D.empty((m, width), torch.float32) for _ in range(3))
        call("lsrm_res_block_bwd_f32", t.data_ptr(), m, width, cw[0].data_ptr(),
             cw[1].data_ptr(), cw[2].data_ptr(), dc.data_ptr(), row_of.data_ptr(),
             occ.data_ptr(), dt.data_ptr(), dr.data_ptr(), dz1.data_ptr(), h.data_ptr(), st)
        g[f"{tag}_w1"] = gx(t, dz1, trans_a=True)
        g[f"{tag}_b1"] = _colsum(dz1)
        g[f"{tag}_w2"] = gx(h, dr, trans_a=True)
        g[f"{tag}_b2"] = _colsum(dr)
    if spec.kv_exchange is not None:   # every rank's partial dK / dV summed at the owners
        dk, dv = spec.kv_exchange.reduce_scatter(dk), spec.kv_exchange.reduce_scatter(dv)
    # projections
    g["w_k"] = gx(s["kv"], dk, trans_a=True)
    g["w_v"] = gx(s["kv"], dv, trans_a=True)
    dkv = gx(dk, P["w_k"], trans_b=True)
    gx(dv, P["w_v"], trans_b=True, out=dkv, beta=1.0)
    g["w_q"] = gx(s["x"], dq, trans_a=True)
    gx(dq, P["w_q"], trans_b=True, out=dx, beta=1.0)
    g["x"], g["kv"] = dx, dkv
    return g


class _NsaUseFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, spec, x, kv, *params):
        P = dict(zip(PARAM_NAMES, (t.detach().contiguous() for t in params)))
        out, saved = _forward(spec, x.detach().contiguous(), kv.detach().contiguous(), P)
        ctx.spec, ctx.P, ctx.saved = spec, P, saved
        return out

    @staticmethod
    def backward(ctx, dout):
        g = _backward(ctx.spec, ctx.P, ctx.saved, dout.contiguous())
        ctx.saved = None
        return (None, g["x"], g["kv"], *(g[name] for name in PARAM_NAMES))


class NsaUseModule(torch.nn.Module):
    """One trainable gated NSA use (fp32).  Parameters mirror `NsaWeights`
    (`nsa_attention.py:239-263`); compression ResBlocks are ck_* / cv_*."""

    def __init__(self, params: AttentionParams, n_gates: int, weights: NsaWeights = None,
                 seed: int = 0, fast_backward: bool = False, tags: tuple = ("train",)):
        super().__init__()
        require(n_gates in (2, 3), "n_gates must be 2 (cross) or 3 (self)")
        self.params, self.n_gates = params, n_gates
        self.fast_backward = fast_backward
        if weights is None:
            # tagged Philox streams (`rng.py`): distinct tags give distinct
            # parameters, like the reference's per-use tags (xs/xc/ys/yc)
            from .nsa_attention import init_nsa_weights
            weights = init_nsa_weights(seed, params, n_gates, *tags)
        for name, arr in _weight_arrays(weights).items():
            self.register_parameter(name, torch.nn.Parameter(D.dev(arr, torch.float32).clone()))

    def forward(self, x, kv, part_q: BlockPartition, part_kv: BlockPartition, sel=None,
                table=None, q_local: LocalQueries = None, kv_exchange=None):
        """q_local / kv_exchange: sequence-parallel call (x = this rank's
        query rows, kv = this rank's kv-stream rows, `table` routes every
        token of the partition)."""
        n = int(x.shape[0])
        require(x.shape[1] == self.params.model_dim, "query width != model dim")
        n_kv = kv_exchange.n_local if kv_exchange is not None else part_kv.n_tokens
        require(int(kv.shape[0]) == n_kv, "partition does not index these tokens")
        if q_local is not None:
            require(getattr(table, "rows", None) is not None and n == q_local.n,
                    "a sequence-parallel use needs a routing table and its local queries")
            rows, count = q_local_rows(q_local, table)
        elif getattr(table, "rows", None) is not None:
            rows, count = table.rows, table.count
        else:
            require(sel is not None and sel.n_queries == n, "a Selection covering every query "
                    "is required")
            rows, count = selection_rows(sel, part_kv)
            own = part_kv.block_of_token if self.n_gates == 3 else None
            rows, count, _, _, _ = resolve_rows(rows, count, part_kv, own, True)
        spec = _Spec(self.params, self.n_gates, part_q, part_kv, rows, count, self.fast_backward,
                     q_local=q_local, kv_exchange=kv_exchange)
        return _NsaUseFn.apply(spec, x, kv, *(getattr(self, nm) for nm in PARAM_NAMES))


def module_weights(mod: "NsaUseModule") -> NsaWeights:
    """The module's current parameters as host `NsaWeights` (f32 arrays), so
    trained weights feed the reference-API forward (`nsa_cross_attention`)
    and the bf16 engine."""
    from .block_partition import CompressWeights, ResBlockParams
    h = {n: getattr(mod, n).detach().float().cpu().numpy() for n in PARAM_NAMES}
    return NsaWeights(h["w_q"], h["w_k"], h["w_v"], h["w_o"], h["gate_w"], h["gate_b"],
                      CompressWeights(ResBlockParams(h["ck_w1"], h["ck_b1"], h["ck_w2"],
                                                     h["ck_b2"]),
                                      ResBlockParams(h["cv_w1"], h["cv_b1"], h["cv_w2"],
                                                     h["cv_b2"])),
                      mod.n_gates)


def _weight_arrays(w: NsaWeights) -> dict:
    ck, cv = w.compress.for_k, w.compress.for_v
    return {"w_q": w.w_q, "w_k": w.w_k, "w_v": w.w_v, "w_o": w.w_o, "gate_w": w.gate_w,
            "gate_b": w.gate_b, "ck_w1": ck.w1, "ck_b1": ck.b1, "ck_w2": ck.w2, "ck_b2": ck.b2,
            "cv_w1": cv.w1, "cv_b1": cv.b1, "cv_w2": cv.w2, "cv_b2": cv.b2}


USE_STREAMS = {"v2v": ("x", "x", 3), "v2i": ("x", "y", 2), "i2i": ("y", "y", 3),
               "i2v": ("y", "x", 2)}


@dataclass
class ResolvedRows:
    rows: torch.Tensor
    count: torch.Tensor


def resolve_plan_rows(plan_rows: dict, part_vol: BlockPartition, part_img: BlockPartition):
    """Routing-plan device rows -> fallback-resolved rows per use
    (`nsa_attention.py:123-154`), reusable across training steps."""
    parts = {"x": part_vol, "y": part_img}
    out = {}
    for use, (qs, ks, ng) in USE_STREAMS.items():
        rows, count = plan_rows[use]
        own = parts[ks].block_of_token if ng == 3 else None
        r, c, _, _, _ = resolve_rows(rows, count, parts[ks], own, True)
        out[use] = ResolvedRows(r, c)
    return out


class NsaLayerModule(torch.nn.Module):
    """The four NSA uses of one Stage-2 layer (`recon_pipeline.py:477-488`):
    v2v and v2i read the volume stream x as queries, i2i and i2v the image
    stream y; returns each use's output."""

    def __init__(self, params: AttentionParams, weights: dict = None, seed: int = 0,
                 fast_backward: bool = False, layer: int = 0):
        super().__init__()
        self.uses = torch.nn.ModuleDict({
            u: NsaUseModule(params, ng, weights=(weights or {}).get(u), seed=seed,
                            fast_backward=fast_backward, tags=("train", f"layer{layer}", u))
            for u, (_, _, ng) in USE_STREAMS.items()})

    def forward(self, x, y, part_vol, part_img, resolved: dict, shard: dict = None) -> dict:
        """shard (sequence parallelism, `seq_parallel.training_shard`): per
        stream its LocalQueries and RowExchange; x / y are then this rank's
        rows of the two streams."""
        streams = {"x": x, "y": y}
        parts = {"x": part_vol, "y": part_img}
        return {u: self.uses[u](streams[qs], streams[ks], parts[qs], parts[ks],
                                table=resolved[u],
                                q_local=shard[qs].queries if shard else None,
                                kv_exchange=shard[ks].exchange if shard else None)
                for u, (qs, ks, _) in USE_STREAMS.items()}


# ---------------------------------------------------------------------------
# the full Stage-2 block (`recon_pipeline.py:461-497`): add + LayerNorm, use
# gates, the four NSA uses, gated mixture + LayerNorm, FFN, residuals.
# Every piece is a torch.autograd.Function over this library's kernels
# (forward: csrc/block.cu row kernels; backward: csrc/train_block.cu).


def _colsum_dev(t: torch.Tensor) -> torch.Tensor:
    n, d = t.shape
    part = D.empty((max(int(lib().lsrm_colsum_parts(n)), 1) * d,), torch.float32)
    out = D.empty((d,), torch.float32)
    call("lsrm_colsum_f32", t.data_ptr(), t.stride(0), n, d, part.data_ptr(), out.data_ptr(),
         D.stream())
    return out


def _ln_bwd(x, gamma, dy, dx, accumulate):
    """dx (+)= dLN(x)/dx . dy; returns (dgamma, dbeta)."""
    from .recon_pipeline import LN_EPS
    n, d = x.shape
    parts = max(int(lib().lsrm_colsum_parts(n)), 1)
    part = D.empty((2 * parts * d + 2 * n,), torch.float32)   # partials + row mean / rstd
    dg, db = D.empty((d,), torch.float32), D.empty((d,), torch.float32)
    call("lsrm_layer_norm_bwd_f32", x.data_ptr(), x.stride(0), n, d, gamma.data_ptr(), LN_EPS,
         dy.data_ptr(), dy.stride(0), dx.data_ptr(), dx.stride(0), int(accumulate),
         part.data_ptr(), dg.data_ptr(), db.data_ptr(), D.stream())
    return dg, db


class _LinearFn(torch.autograd.Function):
    """y = x W (fp32 out; `fast`: bf16 operands on the tcgen05 GEMM)."""
    @staticmethod
    def forward(ctx, x, w, fast):
        x, w = x.detach().contiguous(), w.detach().contiguous()
        ctx.save_for_backward(x, w)
        ctx.fast = fast
        return (_ops.gemm_train if fast else _ops.gemm_ex)(x, w)

    @staticmethod
    def backward(ctx, dy):
        x, w = ctx.saved_tensors
        dy = dy.contiguous()
        if ctx.fast:   # dy's bf16 copy serves both GEMMs
            cache = {}
            return (_ops.gemm_train(dy, w, trans_b=True, cache=cache),
                    _ops.gemm_train(x, dy, trans_a=True, cache=cache), None)
        return _ops.gemm_ex(dy, w, trans_b=True), _ops.gemm_ex(x, dy, trans_a=True), None


class _AddLNFn(torch.autograd.Function):
    """(xe, x_hat) = (a + b, LN(a + b))."""
    @staticmethod
    def forward(ctx, a, b, gamma, beta, exact):
        from .recon_pipeline import NormParams, _add_ln
        xe, xh = _add_ln(a.detach().contiguous(), b.detach().contiguous(),
                         NormParams(gamma.detach(), beta.detach()), exact=bool(exact))
        ctx.save_for_backward(xe, gamma)
        return xe, xh

    @staticmethod
    def backward(ctx, dxe, dxh):
        xe, gamma = ctx.saved_tensors
        dx = dxe.contiguous().clone() if dxe is not None else torch.zeros_like(xe)
        dg, db = _ln_bwd(xe, gamma.detach().contiguous(), dxh.contiguous(), dx, True)
        return dx, dx, dg, db, None


class _GateMixLNFn(torch.autograd.Function):
    """x1 = xe + s(l_s + b_s) o_s + s(l_c + b_c) o_c; h = LN(x1)."""
    @staticmethod
    def forward(ctx, xe, logits, gate_b, o_s, o_c, gamma, beta, exact):
        from .recon_pipeline import NormParams, _gate_mix_ln
        xe, logits = xe.detach().contiguous(), logits.detach().contiguous()
        o_s, o_c = o_s.detach().contiguous(), o_c.detach().contiguous()
        x1, h = _gate_mix_ln(int(exact), xe, logits, logits.stride(0), gate_b.detach(), o_s, o_c,
                             NormParams(gamma.detach(), beta.detach()))
        ctx.save_for_backward(logits, gate_b, o_s, o_c, x1, gamma)
        return x1, h

    @staticmethod
    def backward(ctx, dx1, dh):
        logits, gate_b, o_s, o_c, x1, gamma = ctx.saved_tensors
        n, d = x1.shape
        dx = dx1.contiguous().clone() if dx1 is not None else torch.zeros_like(x1)
        dg, db = _ln_bwd(x1, gamma.detach().contiguous(), dh.contiguous(), dx, True)
        do_s, do_c = D.empty((n, d), torch.float32), D.empty((n, d), torch.float32)
        dl = D.empty((n, 2 * d), torch.float32)
        call("lsrm_gate_mix_bwd_f32", logits.data_ptr(), logits.stride(0),
             gate_b.detach().contiguous().data_ptr(), o_s.data_ptr(), o_c.data_ptr(),
             dx.data_ptr(), n, d, do_s.data_ptr(), do_c.data_ptr(), dl.data_ptr(), D.stream())
        return dx, dl, _colsum_dev(dl), do_s, do_c, dg, db, None


class _BiasActFn(torch.autograd.Function):
    """out = act(z + b) (+ residual); act 0 identity, 1 exact-erf gelu."""
    @staticmethod
    def forward(ctx, z, b, residual, act, exact):
        from .recon_pipeline import _bias_act
        z = z.detach().contiguous()
        res = residual.detach().contiguous() if residual is not None else None
        out = _bias_act(int(exact), z, b.detach().contiguous(), act, residual=res,
                        out_dtype=torch.float32)
        ctx.save_for_backward(z, b)
        ctx.act, ctx.has_res = act, residual is not None
        return out

    @staticmethod
    def backward(ctx, dout):
        z, b = ctx.saved_tensors
        dout = dout.contiguous()
        if ctx.act == 1:
            n, d = z.shape
            dz = D.empty((n, d), torch.float32)
            call("lsrm_gelu_bwd_f32", z.data_ptr(), b.detach().contiguous().data_ptr(),
                 dout.data_ptr(), n, d, dz.data_ptr(), D.stream())
        else:
            dz = dout
        return dz, _colsum_dev(dz), (dout if ctx.has_res else None), None, None


BLOCK_PARAM_NAMES = ("ln_ax_g", "ln_ax_b", "ln_ay_g", "ln_ay_b", "gate_x_w", "gate_x_b",
                     "gate_y_w", "gate_y_b", "ln_fx_g", "ln_fx_b", "ln_fy_g", "ln_fy_b",
                     "fx_w1", "fx_b1", "fx_w2", "fx_b2", "fy_w1", "fy_b1", "fy_w2", "fy_b2")


class SparseBlockModule(torch.nn.Module):
    """One trainable Stage-2 sparse block (`recon_pipeline.py:461-497`): the
    four NSA uses (`NsaLayerModule`) plus the add + LayerNorm, use gates,
    gated mixture + LayerNorm and FFN around them, all differentiable.
    forward(x, y, x_inj, y_inj, part_vol, part_img, resolved) -> (x2, y2),
    token order, fp32; `fast_backward`: bf16 tensor-core attention branches
    and TF32 GEMMs (as NsaUseModule)."""

    def __init__(self, params: AttentionParams, weights=None, seed: int = 0, layer: int = 0,
                 fast_backward: bool = False):
        super().__init__()
        from .recon_pipeline import init_sparse_block
        w = weights if weights is not None else init_sparse_block(seed, params, layer)
        self.params, self.fast = params, fast_backward
        uses = {"v2v": w.nsa_x_self, "v2i": w.nsa_x_cross, "i2i": w.nsa_y_self,
                "i2v": w.nsa_y_cross}
        self.layer = NsaLayerModule(params, weights=uses, fast_backward=fast_backward,
                                    layer=layer)
        arrays = {"ln_ax_g": w.ln_attn_x.gamma, "ln_ax_b": w.ln_attn_x.beta,
                  "ln_ay_g": w.ln_attn_y.gamma, "ln_ay_b": w.ln_attn_y.beta,
                  "gate_x_w": w.gate_x_w, "gate_x_b": w.gate_x_b,
                  "gate_y_w": w.gate_y_w, "gate_y_b": w.gate_y_b,
                  "ln_fx_g": w.ln_ffn_x.gamma, "ln_fx_b": w.ln_ffn_x.beta,
                  "ln_fy_g": w.ln_ffn_y.gamma, "ln_fy_b": w.ln_ffn_y.beta,
                  "fx_w1": w.ffn_x.w1, "fx_b1": w.ffn_x.b1, "fx_w2": w.ffn_x.w2,
                  "fx_b2": w.ffn_x.b2, "fy_w1": w.ffn_y.w1, "fy_b1": w.ffn_y.b1,
                  "fy_w2": w.ffn_y.w2, "fy_b2": w.ffn_y.b2}
        for name in BLOCK_PARAM_NAMES:
            self.register_parameter(name, torch.nn.Parameter(
                D.dev(np.asarray(arrays[name], np.float32), torch.float32).clone()))

    def _stream(self, s, e, lg, o_self, o_cross):
        exact = not self.fast
        x1, h = _GateMixLNFn.apply(e, lg, getattr(self, f"gate_{s}_b"), o_self, o_cross,
                                   getattr(self, f"ln_f{s}_g"), getattr(self, f"ln_f{s}_b"),
                                   exact)
        u = _BiasActFn.apply(_LinearFn.apply(h, getattr(self, f"f{s}_w1"), self.fast),
                             getattr(self, f"f{s}_b1"), None, 1, exact)
        return _BiasActFn.apply(_LinearFn.apply(u, getattr(self, f"f{s}_w2"), self.fast),
                                getattr(self, f"f{s}_b2"), x1, 0, exact)

    def forward(self, x, y, x_inj, y_inj, part_vol, part_img, resolved: dict, shard=None):
        """shard: see NsaLayerModule.forward (x, y, x_inj, y_inj are then this
        rank's rows; every other op of the block is row-local)."""
        exact = not self.fast
        xe, xh = _AddLNFn.apply(x, x_inj, self.ln_ax_g, self.ln_ax_b, exact)
        ye, yh = _AddLNFn.apply(y, y_inj, self.ln_ay_g, self.ln_ay_b, exact)
        lx = _LinearFn.apply(xh, self.gate_x_w, self.fast)
        ly = _LinearFn.apply(yh, self.gate_y_w, self.fast)
        o = self.layer(xh, yh, part_vol, part_img, resolved, shard=shard)
        return (self._stream("x", xe, lx, o["v2v"], o["v2i"]),
                self._stream("y", ye, ly, o["i2i"], o["i2v"]))
