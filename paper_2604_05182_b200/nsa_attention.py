"""Three-branch Native Sparse Attention on the GPU (drop-in for
`lsrm/nsa_attention.py`).

This module is the reference-API surface in float32: every function takes and
returns NumPy arrays exactly like the reference (or CUDA tensors, in which
case results stay on the device).  The arithmetic runs in the C-ABI library:
cuBLAS fp32 GEMMs for the projections (no TF32), the CUDA-core fp32 branch
kernels (csrc/attn_f32.cu) and the f64 ResBlock compression.  The bf16
tcgen05 fused path used for throughput lives in `engine.py`.

Per query token: cmp attends one compressed row per occupied block, sel the
tokens of its selected blocks, win its own block (self uses only); branch
outputs are gated by per-token sigmoid gates, summed and projected by W_o.
"""

import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev as D
from . import _ops, fastpath
from ._native import call
from .block_partition import (BlockPartition, CompressWeights, compress_block_kv,
                              init_compress_weights, compress_rows)
from .errors import (ConfigurationError, EmptyAttentionRowError, EmptyContextError,
                     require)
from .rng import normal_f32
from .tensor_core import AttentionParams

SEL_CHUNK = 512   # kept for API parity with the reference (no effect on the GPU path)


# ---------------------------------------------------------------------------
# selections


@dataclass
class Selection:
    """Per query token: distinct global ids of selected occupied KV blocks
    (`nsa_attention.py:34-54`)."""
    lists: list

    @property
    def n_queries(self) -> int:
        return len(self.lists)

    def validate(self, part: BlockPartition) -> None:
        occupied = set(int(b) for b in part.occupied_ids)
        for qi, ids in enumerate(self.lists):
            ids = [int(b) for b in ids]
            if len(set(ids)) != len(ids):
                raise ConfigurationError(f"query {qi} selects duplicate blocks {ids}")
            for b in ids:
                if b not in occupied:
                    raise ConfigurationError(f"query {qi} selects unoccupied block {b}")


def full_selection(n_queries: int, part: BlockPartition) -> Selection:
    ids = part.occupied_ids.copy()
    return Selection([ids] * n_queries)


def write_selection(fh, sel: Selection) -> None:
    """u32 query count, then per query u32 length + u32 ids (`:57-63`)."""
    fh.write(struct.pack("<I", sel.n_queries))
    for ids in sel.lists:
        ids = np.asarray(ids, dtype=np.uint32)
        fh.write(struct.pack("<I", ids.size))
        fh.write(ids.astype("<u4").tobytes())


def read_selection(fh) -> Selection:
    (n,) = struct.unpack("<I", fh.read(4))
    lists = []
    for _ in range(n):
        (ln,) = struct.unpack("<I", fh.read(4))
        lists.append(np.frombuffer(fh.read(4 * ln), dtype="<u4").astype(np.int64))
    return Selection(lists)


def selection_rows(sel: Selection, part: BlockPartition):
    """Host lists of block ids -> device (rows [n, kmax] int32, count [n])."""
    n = sel.n_queries
    lens = np.fromiter((len(l) for l in sel.lists), np.int64, n)
    kmax = max(int(lens.max()) if n else 1, 1)
    rows = np.full((n, kmax), -1, np.int32)
    if lens.sum():
        flat = np.concatenate([np.asarray(l, np.int64) for l in sel.lists if len(l)])
        r = np.searchsorted(part.occupied_ids, flat)
        ok = (r < part.n_occupied)
        ok[ok] = part.occupied_ids[r[ok]] == flat[ok]
        if not ok.all():
            raise KeyError(int(flat[~ok][0]))
        qi = np.repeat(np.arange(n), lens)
        pos = np.arange(flat.size) - np.repeat(np.cumsum(lens) - lens, lens)
        rows[qi, pos] = r
    return D.dev(rows), D.dev(lens.astype(np.int32))


# ---------------------------------------------------------------------------
# gather tables


@dataclass
class GatherTable:
    """Padded per-query token-id table realizing a Selection
    (`nsa_attention.py:115-120`).  Tables built here also carry the resolved
    block rows the GPU kernels consume (`rows`, `count`, device)."""
    ids: np.ndarray
    valid: np.ndarray
    lengths: np.ndarray
    rows: object = field(default=None, repr=False)
    count: object = field(default=None, repr=False)


def resolve_rows(rows, count, part_kv: BlockPartition, own_block=None, fallback=True,
                 want_ids=False):
    """Device fallback resolution (own block, else lowest occupied block) and
    optional token-id expansion (`nsa_attention.py:123-154`)."""
    n, kmax = int(rows.shape[0]), int(rows.shape[1])
    if n and not fallback and bool((count == 0).any()):
        qi = int(torch.nonzero(count == 0)[0, 0])
        raise EmptyAttentionRowError(f"query {qi} has an empty selection and fallback is off")
    if n and part_kv.n_occupied == 0:
        raise EmptyContextError("empty selection against an empty partition")
    own_row = None
    if own_block is not None:
        own = np.asarray(own_block if not D.is_device(own_block) else D.host(own_block))
        own_row = D.dev(np.searchsorted(part_kv.occupied_ids, own).astype(np.int32))
    res_rows = D.empty((n, kmax), torch.int32)
    res_count = D.empty((n,), torch.int32)
    lengths = D.empty((n,), torch.int64)
    st = D.stream()
    offs, tok = part_kv.dev("block_offsets"), part_kv.dev("block_token_ids")
    call("lsrm_build_gather_table", rows.data_ptr(), count.data_ptr(), n, kmax,
         D.ptr(own_row), int(fallback), offs.data_ptr(), tok.data_ptr(), 0,
         res_rows.data_ptr(), res_count.data_ptr(), None, None, lengths.data_ptr(), st)
    if not want_ids:
        return res_rows, res_count, lengths, None, None
    width = max(int(lengths.max()) if n else 1, 1)
    ids = D.empty((n, width), torch.int64)
    valid = D.empty((n, width), torch.uint8)
    call("lsrm_build_gather_table", res_rows.data_ptr(), res_count.data_ptr(), n, kmax,
         None, 1, offs.data_ptr(), tok.data_ptr(), width, None, None, ids.data_ptr(),
         valid.data_ptr(), lengths.data_ptr(), st)
    return res_rows, res_count, lengths, ids, valid


def build_gather_table(sel: Selection, part_kv: BlockPartition, own_block=None,
                       fallback: bool = True) -> GatherTable:
    """Resolve selected block ids to padded token-id rows; empty selections
    fall back to the own block, else the lowest occupied block
    (`nsa_attention.py:123-154`)."""
    rows, count = selection_rows(sel, part_kv)
    r, c, lengths, ids, valid = resolve_rows(rows, count, part_kv, own_block, fallback,
                                             want_ids=True)
    return GatherTable(D.host(ids), D.host(valid).astype(bool), D.host(lengths), r, c)


# ---------------------------------------------------------------------------
# branches


def _check_qkv(q, k, v, params):
    require(q.ndim == 3 and q.shape[1] == params.n_q_heads and q.shape[2] == params.head_dim,
            f"q shape {tuple(q.shape)} inconsistent with params {params}")
    require(k.ndim == 3 and k.shape[1] == params.n_kv_heads and k.shape[2] == params.head_dim,
            f"k shape {tuple(k.shape)} inconsistent with params {params}")
    require(tuple(v.shape) == tuple(k.shape), "v shape must match k shape")


def _attn(mode, q, k, v, params, offs=None, rows=None, count=None, own_row=None,
          ids=None, lengths=None):
    nq = int(q.shape[0])
    out = D.empty((nq, params.n_q_heads, params.head_dim), torch.float32)
    kmax = int(rows.shape[1]) if rows is not None else 1
    width = int(ids.shape[1]) if ids is not None else 0
    call("lsrm_attention_f32", mode, q.data_ptr(), nq, params.n_q_heads, params.n_kv_heads,
         params.head_dim, k.data_ptr(), v.data_ptr(), int(k.shape[0]), D.ptr(offs),
         D.ptr(rows), D.ptr(count), kmax, D.ptr(own_row), D.ptr(ids), D.ptr(lengths),
         width, out.data_ptr(), D.stream())
    return out


def cmp_attention(q, k_cmp, v_cmp, params: AttentionParams):
    """Attention over the per-block compressed rows (`nsa_attention.py:84-89`)."""
    if k_cmp.shape[0] == 0:
        raise EmptyContextError("no occupied blocks to compress-attend over")
    _check_qkv(q, k_cmp, v_cmp, params)
    on_dev = D.is_device(q)
    o = _attn(0, D.dev(q, torch.float32), D.dev(k_cmp, torch.float32),
              D.dev(v_cmp, torch.float32), params)
    return o if on_dev else D.host(o)


def _block_major(t, part: BlockPartition):
    return _ops.gather_rows(D.dev(t, torch.float32), part.dev("block_token_ids"))


def win_attention(q, k, v, part_q: BlockPartition, part_kv: BlockPartition,
                  params: AttentionParams):
    """Each query attends to the keys of its own block; self pairs only
    (`nsa_attention.py:92-112`)."""
    if part_q is not part_kv and not np.array_equal(part_q.block_of_token,
                                                    part_kv.block_of_token):
        raise ConfigurationError("window attention requires the query and key partitions "
                                 "to be the same (self-attention only)")
    require(q.shape[0] == part_kv.n_tokens == k.shape[0],
            "window attention needs one query per key token")
    _check_qkv(q, k, v, params)
    on_dev = D.is_device(q)
    o = _attn(2, D.dev(q, torch.float32), _block_major(k, part_kv), _block_major(v, part_kv),
              params, offs=part_kv.dev("block_offsets"), own_row=part_kv.dev("row_of_token"))
    return o if on_dev else D.host(o)


def sel_attention(q, k, v, part_kv: BlockPartition, sel, params: AttentionParams,
                  own_block=None, fallback: bool = True, table: GatherTable = None):
    """Attention over the union of tokens of each query's selected blocks
    (`nsa_attention.py:193-207`)."""
    if k.shape[0] == 0:
        raise EmptyContextError("selected attention over an empty token set")
    _check_qkv(q, k, v, params)
    on_dev = D.is_device(q)
    qd = D.dev(q, torch.float32)
    if table is None:
        require(sel.n_queries == q.shape[0],
                f"selection covers {sel.n_queries} queries, got {q.shape[0]}")
        rows, count = selection_rows(sel, part_kv)
        rows, count, _, _, _ = resolve_rows(rows, count, part_kv, own_block, fallback)
    elif table.rows is not None:
        rows, count = table.rows, table.count
    else:   # a caller-built table: walk its explicit token ids
        o = _attn(3, qd, D.dev(k, torch.float32), D.dev(v, torch.float32), params,
                  ids=D.dev(table.ids, torch.int64), lengths=D.dev(table.lengths, torch.int64))
        return o if on_dev else D.host(o)
    o = _attn(1, qd, _block_major(k, part_kv), _block_major(v, part_kv), params,
              offs=part_kv.dev("block_offsets"), rows=rows, count=count)
    return o if on_dev else D.host(o)


def score_topk_blocks(q, k_cmp, b_sel: int, params: AttentionParams,
                      occupied_ids=None) -> Selection:
    """Vanilla selection: blocks ranked by q.k_cmp summed over heads, ties to
    the lower block id (`nsa_attention.py:210-232`)."""
    require(b_sel >= 1, "b_sel must be at least 1")
    nb = int(k_cmp.shape[0])
    if nb == 0:
        raise EmptyContextError("scoring against zero compressed blocks")
    ids = np.arange(nb, dtype=np.int64) if occupied_ids is None else np.asarray(
        occupied_ids, np.int64)
    require(ids.size == nb, "occupied_ids must match compressed row count")
    rows, count = score_topk_rows(D.dev(q, torch.float32), D.dev(k_cmp, torch.float32),
                                  b_sel, params)
    r, c = D.host(rows), D.host(count)
    return Selection([ids[r[i, :c[i]]] for i in range(r.shape[0])])


def score_topk_rows(q, k_cmp, b_sel, params):
    nq = int(q.shape[0])
    rows = D.empty((nq, b_sel), torch.int32)
    count = D.empty((nq,), torch.int32)
    call("lsrm_score_topk", q.data_ptr(), nq, params.n_q_heads, params.n_kv_heads,
         params.head_dim, k_cmp.data_ptr(), int(k_cmp.shape[0]), b_sel, rows.data_ptr(),
         count.data_ptr(), D.stream())
    return rows, count


# ---------------------------------------------------------------------------
# gated combination


@dataclass
class NsaWeights:
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray
    gate_w: np.ndarray
    gate_b: np.ndarray
    compress: CompressWeights
    n_gates: int


def init_nsa_weights(seed: int, params: AttentionParams, n_gates: int, *tags,
                     scale: float = 0.02) -> NsaWeights:
    """`nsa_attention.py:252-263`."""
    d = params.model_dim
    kv_w = params.n_kv_heads * params.head_dim
    return NsaWeights(
        w_q=normal_f32(seed, (d, d), scale, *tags, "wq"),
        w_k=normal_f32(seed, (d, kv_w), scale, *tags, "wk"),
        w_v=normal_f32(seed, (d, kv_w), scale, *tags, "wv"),
        w_o=normal_f32(seed, (d, d), scale, *tags, "wo"),
        gate_w=normal_f32(seed, (d, n_gates * d), scale, *tags, "gate"),
        gate_b=np.zeros(n_gates * d, dtype=np.float32),
        compress=init_compress_weights(seed, kv_w, *tags),
        n_gates=n_gates)


def nsa_gates(x, w: NsaWeights):
    """Per-token sigmoid gate vectors, one width-d slice per branch
    (`nsa_attention.py:266-271`)."""
    on_dev = D.is_device(x)
    xd = D.dev(x, torch.float32)
    n, d = xd.shape
    logits = _ops.gemm(xd, D.weight(w.gate_w))
    g = D.empty((n, w.n_gates * d), torch.float32)
    gb = D.weight(w.gate_b)
    call("lsrm_sigmoid_f32", logits.data_ptr(), logits.stride(0), gb.data_ptr(),
         n, w.n_gates * d, g.data_ptr(), D.stream())
    g = g if on_dev else D.host(g)
    return tuple(g[:, i * d:(i + 1) * d] for i in range(w.n_gates))


def _combine_dev(xd, outs, w: NsaWeights):
    n, d = xd.shape
    logits = _ops.gemm(xd, D.weight(w.gate_w))
    merged = D.empty((n, d), torch.float32)
    o = [t.reshape(n, d) for t in outs] + [None] * (3 - len(outs))
    gb = D.weight(w.gate_b)
    call("lsrm_gated_merge_f32", logits.data_ptr(), logits.stride(0), gb.data_ptr(),
         w.n_gates, D.ptr(o[0]), D.ptr(o[1]), D.ptr(o[2]), n, d, merged.data_ptr(),
         D.stream())
    return _ops.gemm(merged, D.weight(w.w_o))


def combine_nsa_branches(x, branch_outs, w: NsaWeights):
    """Gate, sum (f64), project by W_o (`nsa_attention.py:274-284`)."""
    require(len(branch_outs) == w.n_gates,
            f"{len(branch_outs)} branch outputs for {w.n_gates} gates")
    on_dev = D.is_device(x)
    out = _combine_dev(D.dev(x, torch.float32),
                       [D.dev(o, torch.float32) for o in branch_outs], w)
    return out if on_dev else D.host(out)


def nsa_cross_attention(x, kv_feats, part_q: BlockPartition, part_kv: BlockPartition,
                        sel, w: NsaWeights, params: AttentionParams,
                        table: GatherTable = None, b_sel: int = None,
                        return_selection: bool = False):
    """One gated sparse attention use, fp32 (`nsa_attention.py:287-327`)."""
    d = params.model_dim
    require(x.shape[1] == d, f"query width {x.shape[1]} != model dim {d}")
    if fastpath.active() and not return_selection:
        r = fastpath.nsa_use(x, kv_feats, part_q, part_kv, sel, w, params, table)
        if r is not None:
            return r
    on_dev = D.is_device(x)
    xd = D.dev(x, torch.float32)
    kvd = D.dev(kv_feats, torch.float32)
    n = int(xd.shape[0])
    hq, hkv, dh = params.n_q_heads, params.n_kv_heads, params.head_dim
    q = _ops.gemm(xd, D.weight(w.w_q)).reshape(n, hq, dh)
    k = _ops.gemm(kvd, D.weight(w.w_k))
    v = _ops.gemm(kvd, D.weight(w.w_v))
    nkv = int(kvd.shape[0])
    width = hkv * dh
    require(nkv == part_kv.n_tokens, "partition does not index these tokens")
    if part_kv.n_occupied == 0:
        raise EmptyContextError("no occupied blocks to compress-attend over")
    k_cmp = compress_rows(k, width, nkv, width, w.compress.for_k, part_kv)
    v_cmp = compress_rows(v, width, nkv, width, w.compress.for_v, part_kv)
    is_self = w.n_gates == 3
    if sel is None:
        require(b_sel is not None, "either a Selection or a scoring budget b_sel is required")
        rows, count = score_topk_rows(q, k_cmp.reshape(-1, hkv, dh), b_sel, params)
        table = None
        sel_obj = None
    else:
        sel_obj = sel
    if getattr(table, "rows", None) is not None:   # this package's GatherTable
        rows, count = table.rows, table.count
    else:
        if sel_obj is not None:
            require(sel_obj.n_queries == n, f"selection covers {sel_obj.n_queries} queries, got {n}")
            rows, count = selection_rows(sel_obj, part_kv)
        own = part_kv.block_of_token if is_self else None
        rows, count, _, _, _ = resolve_rows(rows, count, part_kv, own, True)
    tok = part_kv.dev("block_token_ids")
    k_bm = _ops.gather_rows(k, tok)
    v_bm = _ops.gather_rows(v, tok)
    kc3, vc3 = k_cmp.reshape(-1, hkv, dh), v_cmp.reshape(-1, hkv, dh)
    k3, v3 = k_bm.reshape(nkv, hkv, dh), v_bm.reshape(nkv, hkv, dh)
    outs = [_attn(0, q, kc3, vc3, params),
            _attn(1, q, k3, v3, params, offs=part_kv.dev("block_offsets"), rows=rows,
                  count=count)]
    if is_self:
        # win_attention's contract (`nsa_attention.py:92-112`): self pairs only
        if part_q is not part_kv and not np.array_equal(part_q.block_of_token,
                                                        part_kv.block_of_token):
            raise ConfigurationError("window attention requires the query and key partitions "
                                     "to be the same (self-attention only)")
        require(n == part_kv.n_tokens, "window attention needs one query per key token")
        outs.append(_attn(2, q, k3, v3, params, offs=part_kv.dev("block_offsets"),
                          own_row=part_kv.dev("row_of_token")))
    out = _combine_dev(xd, outs, w)
    out = out if on_dev else D.host(out)
    if return_selection:
        if sel_obj is None:
            r, c = D.host(rows), D.host(count)
            sel_obj = Selection([part_kv.occupied_ids[r[i, :c[i]]] for i in range(n)])
        return out, sel_obj
    return out
