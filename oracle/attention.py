"""Three-branch NSA attention with gated merge (TEST INFRASTRUCTURE ONLY).

Restates `lsrm/nsa_attention.py:84-327`.
"""

import math
from dataclasses import dataclass

import numpy as np

from .numerics import (ACC, DTYPE, AttentionParams, OracleError, affine,
                       dense_attention, sigmoid)
from .partition import Partition, compress_block_kv

SEL_CHUNK = 512


@dataclass
class GatherTable:
    """Padded per-query key-id rows (`nsa_attention.py:115-120`)."""
    ids: np.ndarray
    valid: np.ndarray
    lengths: np.ndarray


@dataclass
class NsaWeights:
    """One gated NSA use (`nsa_attention.py:239-249`).  compress =
    ((w1,b1,w2,b2) for k, (w1,b1,w2,b2) for v)."""
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray
    gate_w: np.ndarray
    gate_b: np.ndarray
    compress: tuple
    n_gates: int


def build_gather_table(lists, part_kv: Partition, own_block=None,
                       fallback=True) -> GatherTable:
    """Block lists -> concatenated token ids in selection order; empty lists
    fall back to the own block, else the lowest occupied block
    (`nsa_attention.py:123-154`)."""
    row_of = part_kv.row_of_block()
    toks = []
    for qi, ids in enumerate(lists):
        ids = [int(b) for b in ids]
        if not ids:
            if not fallback:
                raise OracleError("EmptyAttentionRowError", f"query {qi}")
            if own_block is not None:
                ids = [int(own_block[qi])]
            elif part_kv.n_occupied:
                ids = [int(part_kv.occupied_ids[0])]
            else:
                raise OracleError("EmptyContextError", "empty partition")
        toks.append(np.concatenate([part_kv.tokens_in_row(row_of[b]) for b in ids]))
    lengths = np.array([t.size for t in toks], np.int64)
    width = int(lengths.max()) if toks else 1
    ids_tab = np.zeros((len(toks), width), np.int64)
    valid = np.zeros((len(toks), width), bool)
    for i, t in enumerate(toks):
        ids_tab[i, :t.size] = t
        valid[i, :t.size] = True
    return GatherTable(ids_tab, valid, lengths)


def _gathered_attention(q, k, v, tab: GatherTable, params: AttentionParams):
    """Length-sorted chunks of padded-gather attention in f64
    (`nsa_attention.py:157-190`)."""
    n = q.shape[0]
    hkv, g, dh = params.n_kv_heads, params.group_size, params.head_dim
    out = np.zeros((n, params.n_q_heads, dh), DTYPE)
    scale = 1.0 / math.sqrt(dh)
    order = np.argsort(tab.lengths, kind="stable")
    q64, k64, v64 = (np.asarray(a, ACC) for a in (q, k, v))
    for lo in range(0, n, SEL_CHUNK):
        rows = order[lo:lo + SEL_CHUNK]
        w = int(tab.lengths[rows].max())
        ids = tab.ids[rows, :w]
        kg = k64[ids].transpose(0, 2, 3, 1)             # [C,hkv,dh,K]
        vg = v64[ids].transpose(0, 2, 1, 3)             # [C,hkv,K,dh]
        s = np.matmul(q64[rows].reshape(-1, hkv, g, dh), kg) * scale
        s = s + np.where(tab.valid[rows, :w], 0.0, -np.inf)[:, None, None, :]
        s = s - s.max(axis=3, keepdims=True)
        p = np.exp(s)
        p = p / p.sum(axis=3, keepdims=True)
        out[rows] = np.matmul(p, vg).reshape(-1, params.n_q_heads, dh).astype(DTYPE)
    return out


def cmp_attention(q, k_cmp, v_cmp, params):
    """`nsa_attention.py:84-89`."""
    if k_cmp.shape[0] == 0:
        raise OracleError("EmptyContextError", "no compressed blocks")
    return dense_attention(q, k_cmp, v_cmp, params)


def sel_attention(q, k, v, part_kv, lists, params, own_block=None,
                  fallback=True, table=None):
    """`nsa_attention.py:193-207`."""
    if k.shape[0] == 0:
        raise OracleError("EmptyContextError", "no keys")
    if table is None:
        table = build_gather_table(lists, part_kv, own_block, fallback)
    return _gathered_attention(q, k, v, table, params)


def win_attention(q, k, v, part: Partition, params):
    """Dense attention inside each occupied block (`nsa_attention.py:92-112`)."""
    out = np.zeros((q.shape[0], params.n_q_heads, params.head_dim), DTYPE)
    for r in range(part.n_occupied):
        t = part.tokens_in_row(r)
        out[t] = dense_attention(q[t], k[t], v[t], params)
    return out


def score_topk_blocks(q, k_cmp, b_sel, params, occupied_ids=None):
    """Unscaled q.k_cmp summed over heads; stable descending top-b_sel
    (`nsa_attention.py:210-232`)."""
    nb = k_cmp.shape[0]
    if nb == 0:
        raise OracleError("EmptyContextError", "no compressed blocks")
    ids = np.arange(nb) if occupied_ids is None else np.asarray(occupied_ids)
    heads = np.arange(params.n_q_heads) // params.group_size
    sc = np.einsum("qhd,bhd->qb", np.asarray(q, ACC),
                   np.asarray(k_cmp, ACC)[:, heads, :])
    top = np.argsort(-sc, axis=1, kind="stable")[:, :min(b_sel, nb)]
    return [ids[r].astype(np.int64) for r in top]


def nsa_gates(x, w: NsaWeights):
    """`nsa_attention.py:266-271`."""
    g = sigmoid(affine(x, w.gate_w, w.gate_b))
    d = x.shape[1]
    return [g[:, i * d:(i + 1) * d] for i in range(w.n_gates)]


def combine_branches(x, outs, w: NsaWeights):
    """Gated f64 sum of branch outputs, f32, then W_o (`nsa_attention.py:274-284`)."""
    merged = np.zeros(x.shape, ACC)
    for g, o in zip(nsa_gates(x, w), outs):
        merged += g.astype(ACC) * np.asarray(o, ACC)
    return affine(merged.astype(DTYPE), w.w_o)


def nsa_use(x, kv_feats, part_q: Partition, part_kv: Partition, lists,
            w: NsaWeights, params: AttentionParams, table=None, b_sel=None):
    """One gated NSA use (`nsa_attention.py:287-327`); lists=None selects by
    score with budget b_sel."""
    n, d = x.shape
    q = affine(x, w.w_q).reshape(n, params.n_q_heads, params.head_dim)
    k = affine(kv_feats, w.w_k).reshape(-1, params.n_kv_heads, params.head_dim)
    v = affine(kv_feats, w.w_v).reshape(-1, params.n_kv_heads, params.head_dim)
    k_cmp, v_cmp = compress_block_kv(k, v, part_kv, w.compress)
    if lists is None:
        lists = score_topk_blocks(q, k_cmp, b_sel, params, part_kv.occupied_ids)
        table = None
    is_self = w.n_gates == 3
    own = part_kv.block_of_token if is_self else None
    outs = [cmp_attention(q, k_cmp, v_cmp, params).reshape(n, d),
            sel_attention(q, k, v, part_kv, lists, params, own, True,
                          table).reshape(n, d)]
    if is_self:
        outs.append(win_attention(q, k, v, part_kv, params).reshape(n, d))
    return combine_branches(x, outs, w)
