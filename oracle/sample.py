"""One gated NSA use evaluated for a SUBSET of its queries (TEST
INFRASTRUCTURE ONLY).

Every output row of `nsa_cross_attention` (`lsrm/nsa_attention.py:287-327`)
depends only on its own query row and the full key/value side, so the
oracle can check a GPU layer at full BASELINE size (C3/C4/C5) on a sample of
query rows in seconds: the K/V projections and the block compression run
over the whole KV stream exactly as `nsa_use` does; Q, the three branches,
the gates and W_o run for the sampled rows only.  The window branch of a
sampled query attends its whole own block (`nsa_attention.py:92-112`).
"""

import numpy as np

from .attention import (NsaWeights, cmp_attention, combine_branches,
                        sel_attention)
from .numerics import AttentionParams, affine, dense_attention
from .partition import Partition, compress_block_kv


def nsa_use_rows(x, kv_feats, part_q: Partition, part_kv: Partition, lists,
                 w: NsaWeights, params: AttentionParams, qids) -> np.ndarray:
    """Rows `qids` (token ids of the query stream) of
    `nsa_use(x, kv_feats, part_q, part_kv, lists, w, params)`; `lists` is the
    full per-query selection (indexed by token id)."""
    qids = np.asarray(qids, np.int64)
    n, d = qids.size, x.shape[1]
    q = affine(x[qids], w.w_q).reshape(n, params.n_q_heads, params.head_dim)
    k = affine(kv_feats, w.w_k).reshape(-1, params.n_kv_heads, params.head_dim)
    v = affine(kv_feats, w.w_v).reshape(-1, params.n_kv_heads, params.head_dim)
    k_cmp, v_cmp = compress_block_kv(k, v, part_kv, w.compress)
    is_self = w.n_gates == 3
    own = part_kv.block_of_token[qids] if is_self else None
    outs = [cmp_attention(q, k_cmp, v_cmp, params).reshape(n, d),
            sel_attention(q, k, v, part_kv, [lists[i] for i in qids], params, own,
                          True).reshape(n, d)]
    if is_self:
        outs.append(_window_rows(q, qids, k, v, part_kv, params).reshape(n, d))
    return combine_branches(x[qids], outs, w)


def _window_rows(q, qids, k, v, part: Partition, params):
    out = np.zeros((qids.size, params.n_q_heads, params.head_dim), np.float32)
    row_of = part.row_of_block()
    blk = part.block_of_token[qids]
    for b in np.unique(blk):
        sel = np.nonzero(blk == b)[0]
        t = part.tokens_in_row(row_of[int(b)])
        out[sel] = dense_attention(q[sel], k[t], v[t], params)
    return out


def strided_sample(n: int, target: int) -> np.ndarray:
    """~`target` token ids spread evenly over [0, n) (every block region of
    the token order is represented)."""
    step = max(1, n // max(1, target))
    return np.arange(0, n, step, dtype=np.int64)
