"""Stage-2 sparse residual block around the four NSA uses (TEST INFRASTRUCTURE ONLY).

Restates `lsrm/recon_pipeline.py:374-512` (weights, `sparse_block_forward`)
and the initialisers it uses (`nsa_attention.py:252-263`,
`block_partition.py:127-138`, `recon_pipeline.py:78-90`).
"""

from dataclasses import dataclass

import numpy as np

from .attention import NsaWeights, nsa_use
from .numerics import ACC, DTYPE, affine, gelu, layer_norm, sigmoid
from .rng import normal_f32

USES = ("v2v", "v2i", "i2i", "i2v")


def init_nsa_weights(seed, params, n_gates, *tags, scale=0.02):
    d = params.model_dim
    w = params.n_kv_heads * params.head_dim

    def rb(name):
        return (normal_f32(seed, (w, w), 0.02, *tags, name, "w1"),
                np.zeros(w, DTYPE),
                normal_f32(seed, (w, w), 0.02, *tags, name, "w2"),
                np.zeros(w, DTYPE))
    return NsaWeights(
        w_q=normal_f32(seed, (d, d), scale, *tags, "wq"),
        w_k=normal_f32(seed, (d, w), scale, *tags, "wk"),
        w_v=normal_f32(seed, (d, w), scale, *tags, "wv"),
        w_o=normal_f32(seed, (d, d), scale, *tags, "wo"),
        gate_w=normal_f32(seed, (d, n_gates * d), scale, *tags, "gate"),
        gate_b=np.zeros(n_gates * d, DTYPE),
        compress=(rb("cmp_k"), rb("cmp_v")), n_gates=n_gates)


@dataclass
class SparseBlockWeights:
    nsa: dict            # use name -> NsaWeights
    inj_x: np.ndarray
    inj_y: np.ndarray
    gate_x: tuple        # (w [d,2d], b [2d])
    gate_y: tuple
    ln: dict             # attn_x, attn_y, ffn_x, ffn_y -> (gamma, beta)
    ffn_x: tuple         # (w1, b1, w2, b2)
    ffn_y: tuple


def init_sparse_block(seed, params, layer, scale=0.02):
    d = params.model_dim
    tag = f"sparse{layer}"

    def ffn(name):
        return (normal_f32(seed, (d, 4 * d), scale, tag, name, "w1"),
                np.zeros(4 * d, DTYPE),
                normal_f32(seed, (4 * d, d), scale, tag, name, "w2"),
                np.zeros(d, DTYPE))
    norm = (np.ones(d, DTYPE), np.zeros(d, DTYPE))
    return SparseBlockWeights(
        nsa={"v2v": init_nsa_weights(seed, params, 3, tag, "xs", scale=scale),
             "v2i": init_nsa_weights(seed, params, 2, tag, "xc", scale=scale),
             "i2i": init_nsa_weights(seed, params, 3, tag, "ys", scale=scale),
             "i2v": init_nsa_weights(seed, params, 2, tag, "yc", scale=scale)},
        inj_x=normal_f32(seed, (d, d), scale, tag, "ix"),
        inj_y=normal_f32(seed, (d, d), scale, tag, "iy"),
        gate_x=(normal_f32(seed, (d, 2 * d), scale, tag, "gx"), np.zeros(2 * d, DTYPE)),
        gate_y=(normal_f32(seed, (d, 2 * d), scale, tag, "gy"), np.zeros(2 * d, DTYPE)),
        ln={k: norm for k in ("attn_x", "attn_y", "ffn_x", "ffn_y")},
        ffn_x=ffn("fx"), ffn_y=ffn("fy"))


def ffn_forward(x, p):
    """affine-gelu-affine (`recon_pipeline.py:104-105`, `tensor_core.py:119-136`)."""
    return affine(gelu(affine(x, p[0], p[1])), p[2], p[3])


def sparse_block_forward(x, y, x_inj, y_inj, w: SparseBlockWeights, ctx,
                         params):
    """One sparse residual block (`recon_pipeline.py:461-497`).
    ctx: dict with part_vol, part_img, selections (name -> lists) and
    tables (name -> GatherTable)."""
    xe = (x.astype(ACC) + x_inj.astype(ACC)).astype(DTYPE)
    ye = (y.astype(ACC) + y_inj.astype(ACC)).astype(DTYPE)
    xh = layer_norm(xe, *w.ln["attn_x"])
    yh = layer_norm(ye, *w.ln["attn_y"])
    d = x.shape[1]
    gx = sigmoid(affine(xh, *w.gate_x))
    gy = sigmoid(affine(yh, *w.gate_y))
    pv, pi = ctx["part_vol"], ctx["part_img"]

    def use(name, q, kv, pq, pkv):
        return nsa_use(q, kv, pq, pkv, ctx["selections"][name], w.nsa[name],
                       params, table=ctx["tables"][name]).astype(ACC)
    o_x = gx[:, :d].astype(ACC) * use("v2v", xh, xh, pv, pv) \
        + gx[:, d:].astype(ACC) * use("v2i", xh, yh, pv, pi)
    o_y = gy[:, :d].astype(ACC) * use("i2i", yh, yh, pi, pi) \
        + gy[:, d:].astype(ACC) * use("i2v", yh, xh, pi, pv)
    x1 = (xe.astype(ACC) + o_x).astype(DTYPE)
    y1 = (ye.astype(ACC) + o_y).astype(DTYPE)
    x2 = (x1.astype(ACC) + ffn_forward(layer_norm(x1, *w.ln["ffn_x"]), w.ffn_x)
          .astype(ACC)).astype(DTYPE)
    y2 = (y1.astype(ACC) + ffn_forward(layer_norm(y1, *w.ln["ffn_y"]), w.ffn_y)
          .astype(ACC)).astype(DTYPE)
    return x2, y2
