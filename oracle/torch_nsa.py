"""Differentiable float64 restatement of one gated NSA use (TEST
INFRASTRUCTURE ONLY) - the oracle for the backward pass.

The reference has no backward (SURVEY.md §7 hard part 9). Its
forward (`nsa_attention.py:287-327`, restated in NumPy in
`oracle/attention.py:nsa_use`) is re-expressed with torch f64 operations, so
autograd supplies exact gradients. The tests pin this restatement to the
NumPy oracle's forward (<= 1e-12) and check it with `torch.autograd.gradcheck`
on a tiny instance.

Key sets are dense masks (fine at test sizes): cmp sees every compressed row,
sel the tokens of the query's resolved selected blocks, win its own block.
"""

import math

import numpy as np
import torch


def _gelu(z):
    return 0.5 * z * (1.0 + torch.erf(z / math.sqrt(2.0)))


def res_block(x, w1, b1, w2, b2):
    """x + gelu(x W1 + b1) W2 + b2 (`block_partition.py:141-144`)."""
    return x + _gelu(x @ w1 + b1) @ w2 + b2


def key_masks(part_q, part_kv, lists, is_self):
    """Dense [Nq, Nkv] bool masks for the sel and win branches (token order).
    lists: per query the (already fallback-resolved) selected block ids."""
    nq, nk = len(lists), part_kv.block_of_token.shape[0]
    row_of = part_kv.row_of_block()
    sel = np.zeros((nq, nk), bool)
    for i, ids in enumerate(lists):
        for b in ids:
            sel[i, part_kv.tokens_in_row(row_of[int(b)])] = True
    win = None
    if is_self:
        win = part_q.block_of_token[:, None] == part_kv.block_of_token[None, :]
    return torch.from_numpy(sel), (torch.from_numpy(win) if win is not None else None)


def _attention(q, k, v, mask, group):
    """softmax(q k^T / sqrt(dh)) v per head; q [n,hq,dh], k/v [m,hkv,dh]."""
    dh = q.shape[2]
    heads = torch.arange(q.shape[1]) // group
    s = torch.einsum("nhd,mhd->nhm", q, k[:, heads, :]) / math.sqrt(dh)
    if mask is not None:
        s = s.masked_fill(~mask[:, None, :], float("-inf"))
    p = torch.softmax(s, dim=2)
    return torch.einsum("nhm,mhd->nhd", p, v[:, heads, :])


def nsa_use(x, kv, w, params, part_kv, sel_mask, win_mask):
    """x [Nq,d], kv [Nkv,d] f64 tensors; w: dict of f64 tensors w_q w_k w_v w_o
    gate_w gate_b and ck = (w1,b1,w2,b2), cv = (...). Returns [Nq, d]."""
    n, d = x.shape
    hq, hkv, dh = params.n_q_heads, params.n_kv_heads, params.head_dim
    group = hq // hkv
    q = (x @ w["w_q"]).reshape(n, hq, dh)
    k = (kv @ w["w_k"]).reshape(-1, hkv, dh)
    v = (kv @ w["w_v"]).reshape(-1, hkv, dh)
    m = k.shape[0]
    bid = torch.from_numpy(np.asarray(part_kv.block_of_token, np.int64))
    uniq, inv = torch.unique(bid, return_inverse=True)
    occ = torch.bincount(inv).to(x.dtype)

    def compress(t, p):
        r = res_block(t.reshape(m, hkv * dh), *p)
        s = torch.zeros((uniq.numel(), hkv * dh), dtype=x.dtype).index_add(0, inv, r)
        return (s / occ[:, None]).reshape(-1, hkv, dh)
    kc, vc = compress(k, w["ck"]), compress(v, w["cv"])
    outs = [_attention(q, kc, vc, None, group), _attention(q, k, v, sel_mask, group)]
    if win_mask is not None:
        outs.append(_attention(q, k, v, win_mask, group))
    g = torch.sigmoid(x @ w["gate_w"] + w["gate_b"])
    merged = sum(g[:, b * d:(b + 1) * d] * o.reshape(n, d) for b, o in enumerate(outs))
    return merged @ w["w_o"]


def layer_norm(x, gamma, beta, eps=1e-5):
    """`tensor_core.py:139-146` (biased variance)."""
    mu = x.mean(dim=1, keepdim=True)
    var = ((x - mu) ** 2).mean(dim=1, keepdim=True)
    return (x - mu) / torch.sqrt(var + eps) * gamma + beta


def sparse_block(x, y, x_inj, y_inj, wb, params, parts, masks):
    """One Stage-2 sparse block, f64 autograd (`recon_pipeline.py:461-497`).
    wb: dict of f64 tensors: uses[v2v|v2i|i2i|i2v] (nsa_use weight dicts),
    ln_ax/ln_ay/ln_fx/ln_fy = (gamma, beta), gate_x/gate_y = (W, b),
    ffn_x/ffn_y = (w1, b1, w2, b2). parts[use] = the KV partition,
    masks[use] = (sel, win)."""
    def ffn(h, w):
        return _gelu(h @ w[0] + w[1]) @ w[2] + w[3]
    d = x.shape[1]
    xe, ye = x + x_inj, y + y_inj
    xh, yh = layer_norm(xe, *wb["ln_ax"]), layer_norm(ye, *wb["ln_ay"])
    gx = torch.sigmoid(xh @ wb["gate_x"][0] + wb["gate_x"][1])
    gy = torch.sigmoid(yh @ wb["gate_y"][0] + wb["gate_y"][1])

    def use(name, q, kv):
        return nsa_use(q, kv, wb["uses"][name], params, parts[name], *masks[name])
    x1 = xe + gx[:, :d] * use("v2v", xh, xh) + gx[:, d:] * use("v2i", xh, yh)
    y1 = ye + gy[:, :d] * use("i2i", yh, yh) + gy[:, d:] * use("i2v", yh, xh)
    return (x1 + ffn(layer_norm(x1, *wb["ln_fx"]), wb["ffn_x"]),
            y1 + ffn(layer_norm(y1, *wb["ln_fy"]), wb["ffn_y"]))
