"""Stage-2 sparse residual block around the four NSA uses (drop-in for the
hot-path part of `lsrm/recon_pipeline.py`).

`sparse_block_forward` keeps the reference signature and float contract: f32
in/out, f64 arithmetic in the row-wise steps, fp32 (no TF32) GEMMs and the
fp32 NSA path. `SparseBlockEngine` is the bf16 throughput path over the same
weights. It reuses `SparseLayerEngine` for the four uses, folds the use-gate
projection into each stream's fused projection GEMM, and runs injection +
LayerNorm, gate mixture + LayerNorm and the FFN residual as fused kernels
(csrc/block.cu) around bf16 cuBLAS GEMMs.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev as D
from . import _ops, fastpath
from ._native import call
from .block_partition import BlockPartition
from .engine import USE_GEOM, USES, SparseLayerEngine
from .errors import require
from .nsa_attention import NsaWeights, build_gather_table, init_nsa_weights, nsa_cross_attention
from .rng import normal_f32
from .tensor_core import DTYPE, AttentionParams

LN_EPS = 1e-5
TABLE_NAMES = ("v2v", "v2i", "i2v", "i2i")


@dataclass
class NormParams:
    """`recon_pipeline.py:60-63`."""
    gamma: np.ndarray
    beta: np.ndarray


@dataclass
class FfnWeights:
    """`recon_pipeline.py:52-57`: w1 [d, 4d], b1, w2 [4d, d], b2."""
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray


@dataclass
class SparseBlockWeights:
    """`recon_pipeline.py:379-395`."""
    nsa_x_self: NsaWeights
    nsa_x_cross: NsaWeights
    nsa_y_self: NsaWeights
    nsa_y_cross: NsaWeights
    inj_x: np.ndarray
    inj_y: np.ndarray
    gate_x_w: np.ndarray
    gate_x_b: np.ndarray
    gate_y_w: np.ndarray
    gate_y_b: np.ndarray
    ln_attn_x: NormParams
    ln_attn_y: NormParams
    ln_ffn_x: NormParams
    ln_ffn_y: NormParams
    ffn_x: FfnWeights
    ffn_y: FfnWeights

    def uses(self) -> dict:
        return {"v2v": self.nsa_x_self, "v2i": self.nsa_x_cross, "i2i": self.nsa_y_self,
                "i2v": self.nsa_y_cross}


def init_ffn(seed: int, d: int, *tags, scale: float = 0.02) -> FfnWeights:
    """`recon_pipeline.py:78-84`."""
    return FfnWeights(normal_f32(seed, (d, 4 * d), scale, *tags, "w1"),
                      np.zeros(4 * d, dtype=DTYPE),
                      normal_f32(seed, (4 * d, d), scale, *tags, "w2"),
                      np.zeros(d, dtype=DTYPE))


def init_norm(d: int) -> NormParams:
    """`recon_pipeline.py:87-88`."""
    return NormParams(np.ones(d, dtype=DTYPE), np.zeros(d, dtype=DTYPE))


def init_sparse_block(seed: int, params: AttentionParams, layer: int,
                      scale: float = 0.02) -> SparseBlockWeights:
    """`recon_pipeline.py:398-414` (same tags, so identical weights)."""
    d = params.model_dim
    tag = f"sparse{layer}"
    return SparseBlockWeights(
        nsa_x_self=init_nsa_weights(seed, params, 3, tag, "xs", scale=scale),
        nsa_x_cross=init_nsa_weights(seed, params, 2, tag, "xc", scale=scale),
        nsa_y_self=init_nsa_weights(seed, params, 3, tag, "ys", scale=scale),
        nsa_y_cross=init_nsa_weights(seed, params, 2, tag, "yc", scale=scale),
        inj_x=normal_f32(seed, (d, d), scale, tag, "ix"),
        inj_y=normal_f32(seed, (d, d), scale, tag, "iy"),
        gate_x_w=normal_f32(seed, (d, 2 * d), scale, tag, "gx"),
        gate_x_b=np.zeros(2 * d, dtype=DTYPE),
        gate_y_w=normal_f32(seed, (d, 2 * d), scale, tag, "gy"),
        gate_y_b=np.zeros(2 * d, dtype=DTYPE),
        ln_attn_x=init_norm(d), ln_attn_y=init_norm(d),
        ln_ffn_x=init_norm(d), ln_ffn_y=init_norm(d),
        ffn_x=init_ffn(seed, d, tag, "fx", scale=scale),
        ffn_y=init_ffn(seed, d, tag, "fy", scale=scale))


@dataclass
class SparseContext:
    """`recon_pipeline.py:417-430`: partitions, routed selections (or score
    budgets) and the gather tables amortised across layers."""
    part_vol: BlockPartition
    part_img: BlockPartition
    selections: dict = None
    budgets: dict = None
    tables: dict = None

    def mode(self) -> str:
        return "3d" if self.selections is not None else "score"


def build_sparse_context(part_vol: BlockPartition, part_img: BlockPartition,
                         selections: dict = None, budgets: dict = None) -> SparseContext:
    """`recon_pipeline.py:436-448`."""
    ctx = SparseContext(part_vol, part_img, selections, budgets)
    if selections is not None:
        kv_parts = {"v2v": part_vol, "v2i": part_img, "i2v": part_vol, "i2i": part_img}
        own = {"v2v": part_vol.block_of_token, "i2i": part_img.block_of_token}
        ctx.tables = {name: build_gather_table(selections[name], kv_parts[name],
                                               own_block=own.get(name))
                      for name in TABLE_NAMES}
    return ctx


# ---------------------------------------------------------------------------
# fused row / element steps (csrc/block.cu)


def _add_ln(a, b, norm: NormParams, out_dtype=torch.float32, exact=True):
    """sum = f32(a + b), LayerNorm(sum) -> (sum f32, normalised)."""
    n, d = a.shape
    s = D.empty((n, d), torch.float32)
    y = D.empty((n, d), out_dtype)
    gamma, beta = D.weight(norm.gamma), D.weight(norm.beta)   # alive across the launch
    call("lsrm_add_layer_norm", int(exact), a.data_ptr(), D.ptr(b), int(b is not None and
                                                           b.dtype == torch.bfloat16),
         n, d, gamma.data_ptr(), beta.data_ptr(), LN_EPS, s.data_ptr(),
         int(out_dtype == torch.bfloat16), y.data_ptr(), D.stream())
    return s, y


def _gate_mix_ln(exact, xe, logits, ld, gate_b, o_self, o_cross, norm: NormParams,
                 out_dtype=torch.float32):
    """x1 = f32(xe + sig(self logits) * o_self + sig(cross logits) * o_cross),
    h = LayerNorm(x1)."""
    n, d = xe.shape
    x1 = D.empty((n, d), torch.float32)
    h = D.empty((n, d), out_dtype)
    gamma, beta = D.weight(norm.gamma), D.weight(norm.beta)   # alive across the launch
    call("lsrm_gate_mix_layer_norm", int(exact), xe.data_ptr(), logits.data_ptr(), ld,
         int(logits.dtype == torch.bfloat16), gate_b.data_ptr(), o_self.data_ptr(),
         o_cross.data_ptr(), int(o_self.dtype == torch.bfloat16), n, d, x1.data_ptr(),
         gamma.data_ptr(), beta.data_ptr(), LN_EPS,
         int(out_dtype == torch.bfloat16), h.data_ptr(), D.stream())
    return x1, h


def _bias_act(exact, h, bias, act, residual=None, out=None, out_dtype=None):
    n, cols = h.shape
    out = h if out is None and out_dtype is None else out
    if out is None:
        out = D.empty((n, cols), out_dtype)
    call("lsrm_bias_act", int(exact), h.data_ptr(), int(h.dtype == torch.bfloat16), h.stride(0),
         bias.data_ptr(), n, cols, int(act), D.ptr(residual), out.data_ptr(),
         int(out.dtype == torch.bfloat16), out.stride(0), D.stream())
    return out


def ffn_forward(x, w: FfnWeights):
    """affine-gelu-affine (`recon_pipeline.py:101-102`), fp32."""
    on_dev = D.is_device(x)
    xd = D.dev(x, torch.float32)
    t = _bias_act(1, _ops.gemm(xd, D.weight(w.w1)), D.weight(w.b1), 1)
    out = _bias_act(1, _ops.gemm(t, D.weight(w.w2)), D.weight(w.b2), 0)
    return out if on_dev else D.host(out)


def _nsa_use(x_hat, kv_hat, part_q, part_kv, name, w_use, ctx: SparseContext, params):
    """`recon_pipeline.py:451-458`."""
    if ctx.selections is not None:
        return nsa_cross_attention(x_hat, kv_hat, part_q, part_kv, ctx.selections[name], w_use,
                                   params, table=ctx.tables[name])
    return nsa_cross_attention(x_hat, kv_hat, part_q, part_kv, None, w_use, params,
                               b_sel=ctx.budgets[name])


def sparse_block_forward(x, y, x_inj, y_inj, w: SparseBlockWeights, ctx: SparseContext,
                         params: AttentionParams):
    """One sparse residual block (`recon_pipeline.py:461-497`), reference
    float contract. NumPy in -> NumPy out; CUDA tensors stay on the device."""
    require(x.shape[0] > 0 and y.shape[0] > 0, "sparse block needs nonempty token streams")
    if fastpath.active():
        r = fastpath.sparse_block(x, y, x_inj, y_inj, w, ctx, params)
        if r is not None:
            return r
    on_dev = D.is_device(x)
    xd, yd, xi, yi = (D.dev(a, torch.float32) for a in (x, y, x_inj, y_inj))
    xe, xh = _add_ln(xd, xi, w.ln_attn_x)
    ye, yh = _add_ln(yd, yi, w.ln_attn_y)
    lx = _ops.gemm(xh, D.weight(w.gate_x_w))
    ly = _ops.gemm(yh, D.weight(w.gate_y_w))
    o_vv = _nsa_use(xh, xh, ctx.part_vol, ctx.part_vol, "v2v", w.nsa_x_self, ctx, params)
    o_vi = _nsa_use(xh, yh, ctx.part_vol, ctx.part_img, "v2i", w.nsa_x_cross, ctx, params)
    o_ii = _nsa_use(yh, yh, ctx.part_img, ctx.part_img, "i2i", w.nsa_y_self, ctx, params)
    o_iv = _nsa_use(yh, xh, ctx.part_img, ctx.part_vol, "i2v", w.nsa_y_cross, ctx, params)
    outs = []
    for e, lg, gb, os_, oc, ln, ffn in ((xe, lx, D.weight(w.gate_x_b), o_vv, o_vi, w.ln_ffn_x, w.ffn_x),
                                        (ye, ly, D.weight(w.gate_y_b), o_ii, o_iv, w.ln_ffn_y, w.ffn_y)):
        x1, h = _gate_mix_ln(1, e, lg, lg.stride(0), gb, os_, oc, ln)
        t = _bias_act(1, _ops.gemm(h, D.weight(ffn.w1)), D.weight(ffn.b1), 1)
        outs.append(_bias_act(1, _ops.gemm(t, D.weight(ffn.w2)), D.weight(ffn.b2), 0, residual=x1))
    return tuple(o if on_dev else D.host(o) for o in outs)


def sparse_stage_forward(x_up, y_up, weights, ctx: SparseContext, params: AttentionParams):
    """Residual stage (`recon_pipeline.py:500-512`): zero state, per-layer
    injections of the frozen inputs, inputs added back at the end."""
    if fastpath.active():
        r = fastpath.sparse_stage(x_up, y_up, weights, ctx, params)
        if r is not None:
            return r
    xf = D.dev(x_up.features, torch.float32)
    yf = D.dev(y_up.features, torch.float32)
    x, y = torch.zeros_like(xf), torch.zeros_like(yf)
    for w in weights:
        x, y = sparse_block_forward(x, y, _ops.gemm(xf, D.weight(w.inj_x)),
                                    _ops.gemm(yf, D.weight(w.inj_y)), w, ctx, params)
    xs = D.empty(tuple(xf.shape), torch.float32)
    ys = D.empty(tuple(yf.shape), torch.float32)
    for a, b, o in ((x, xf, xs), (y, yf, ys)):
        _bias_act(1, a, torch.zeros(a.shape[1], dtype=torch.float32, device=a.device), 0,
                  residual=b, out=o)
    return D.host(xs), D.host(ys)


# ---------------------------------------------------------------------------
# bf16 throughput path


class SparseBlockEngine:
    """One Stage-2 block on the bf16 engine, block-major order end to end.

    forward(x, y, x_inj, y_inj) takes f32 block-major rows and returns
    (x2, y2) f32 block-major. The four NSA uses run on `SparseLayerEngine`.
    Its fused per-stream projection GEMM also produces the two use-gate
    logits."""

    def __init__(self, part_vol: BlockPartition, part_img: BlockPartition, plan_rows: dict,
                 w: SparseBlockWeights, params: AttentionParams, pool: dict = None,
                 uses: dict = None, shard: dict = None):
        # `uses`: use -> NsaWeights, for weight objects without `.uses()` (the
        # reference's SparseBlockWeights, via the drop-in). `shard`: owned
        # occupied rows per stream (sequence parallelism; every row-local
        # step then runs on the owned tokens in the rank-local order)
        self.w, self.params = w, params
        self.layer = SparseLayerEngine(part_vol, part_img, plan_rows, uses or w.uses(), params,
                                       extra_cols={"x": w.gate_x_w, "y": w.gate_y_w}, pool=pool,
                                       shard=shard)
        # FFN weights transposed ([n, k], K contiguous) for the tcgen05 GEMM
        self.bf = {name: D.dev(np.asarray(getattr(getattr(w, f), n)).T, torch.bfloat16)
                   for name, f, n in (("fx1", "ffn_x", "w1"), ("fx2", "ffn_x", "w2"),
                                      ("fy1", "ffn_y", "w1"), ("fy2", "ffn_y", "w2"))}

    def forward(self, x, y, x_inj, y_inj):
        w, L = self.w, self.layer
        xe, xh = _add_ln(x, x_inj, w.ln_attn_x, torch.bfloat16, exact=False)
        ye, yh = _add_ln(y, y_inj, w.ln_attn_y, torch.bfloat16, exact=False)
        outs = L.forward(xh, yh)
        x1s, hs = [], []
        for s, e, gb, us, uc, ln in (
                ("x", xe, D.weight(w.gate_x_b), "v2v", "v2i", w.ln_ffn_x),
                ("y", ye, D.weight(w.gate_y_b), "i2i", "i2v", w.ln_ffn_y)):
            Y = L.buf[("Y", s)]
            lg = Y[:, L.cols[("extra", s)]:]
            x1, h = _gate_mix_ln(0, e, lg, Y.stride(0), gb, outs[us], outs[uc], ln,
                                 torch.bfloat16)
            x1s.append(x1)
            hs.append(h)
        # FFN on the tcgen05 GEMM, both streams per launch: gelu(h W1 + b1)
        # (bias + erf-gelu in the epilogue, bf16), then t W2 + b2 + x1 (bias
        # and residual in the epilogue, f32)
        ts, p1 = [], []
        for h, k1, ffn in zip(hs, ("fx1", "fy1"), (w.ffn_x, w.ffn_y)):
            t = D.empty((h.shape[0], self.bf[k1].shape[0]), torch.bfloat16)
            ts.append(t)
            p1.append(_ops.gemm_problem(h, self.bf[k1], t, bias=D.weight(ffn.b1), gelu=True))
        _ops.gemm_tc([p for p, h in zip(p1, hs) if h.shape[0]])
        res, p2 = [], []
        for t, x1, k2, ffn in zip(ts, x1s, ("fx2", "fy2"), (w.ffn_x, w.ffn_y)):
            u = D.empty(tuple(x1.shape), torch.float32)
            res.append(u)
            p2.append(_ops.gemm_problem(t, self.bf[k2], u, bias=D.weight(ffn.b2), res=x1))
        _ops.gemm_tc([p for p, t in zip(p2, ts) if t.shape[0]])
        return tuple(res)


# ---------------------------------------------------------------------------
# Stage 1: dense blocks (recon_pipeline.py:113-193; §8f rank 4)


@dataclass
class MhaWeights:
    """`recon_pipeline.py:45-49`."""
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray


@dataclass
class DenseBlockWeights:
    """`recon_pipeline.py:117-131`."""
    x_self: MhaWeights
    x_cross: MhaWeights
    y_self: MhaWeights
    y_cross: MhaWeights
    gate_x_w: np.ndarray
    gate_x_b: np.ndarray
    gate_y_w: np.ndarray
    gate_y_b: np.ndarray
    ln_attn_x: NormParams
    ln_attn_y: NormParams
    ln_ffn_x: NormParams
    ln_ffn_y: NormParams
    ffn_x: FfnWeights
    ffn_y: FfnWeights


def init_mha(seed: int, params: AttentionParams, *tags, scale: float = 0.02) -> MhaWeights:
    """`recon_pipeline.py:66-74` (same tags, so identical weights)."""
    d = params.model_dim
    kv_w = params.n_kv_heads * params.head_dim
    return MhaWeights(normal_f32(seed, (d, d), scale, *tags, "wq"),
                      normal_f32(seed, (d, kv_w), scale, *tags, "wk"),
                      normal_f32(seed, (d, kv_w), scale, *tags, "wv"),
                      normal_f32(seed, (d, d), scale, *tags, "wo"))


def init_dense_block(seed: int, params: AttentionParams, layer: int,
                     scale: float = 0.02) -> DenseBlockWeights:
    """`recon_pipeline.py:134-151`."""
    d = params.model_dim
    tag = f"dense{layer}"
    return DenseBlockWeights(
        x_self=init_mha(seed, params, tag, "xs", scale=scale),
        x_cross=init_mha(seed, params, tag, "xc", scale=scale),
        y_self=init_mha(seed, params, tag, "ys", scale=scale),
        y_cross=init_mha(seed, params, tag, "yc", scale=scale),
        gate_x_w=normal_f32(seed, (d, 2 * d), scale, tag, "gx"),
        gate_x_b=np.zeros(2 * d, dtype=DTYPE),
        gate_y_w=normal_f32(seed, (d, 2 * d), scale, tag, "gy"),
        gate_y_b=np.zeros(2 * d, dtype=DTYPE),
        ln_attn_x=init_norm(d), ln_attn_y=init_norm(d),
        ln_ffn_x=init_norm(d), ln_ffn_y=init_norm(d),
        ffn_x=init_ffn(seed, d, tag, "fx", scale=scale),
        ffn_y=init_ffn(seed, d, tag, "fy", scale=scale))


def mha_forward(q_in, kv_in, w: MhaWeights, params: AttentionParams):
    """Full multi-head attention with the output projection
    (`recon_pipeline.py:90-98`): fp32 projections, dense GQA softmax
    (`tensor_core.py:164-206`, csrc/attn_f32.cu mode 0), W_o."""
    from .errors import EmptyContextError
    from .nsa_attention import _attn
    on_dev = D.is_device(q_in)
    qd, kd = D.dev(q_in, torch.float32), D.dev(kv_in, torch.float32)
    if kd.shape[0] == 0:
        raise EmptyContextError("attention over an empty key set")
    n = int(qd.shape[0])
    hq, hkv, dh = params.n_q_heads, params.n_kv_heads, params.head_dim
    q = _ops.gemm(qd, D.weight(w.w_q)).view(n, hq, dh)
    k = _ops.gemm(kd, D.weight(w.w_k)).view(-1, hkv, dh)
    v = _ops.gemm(kd, D.weight(w.w_v)).view(-1, hkv, dh)
    o = _attn(0, q, k, v, params)
    out = _ops.gemm(o.view(n, params.model_dim), D.weight(w.w_o))
    return out if on_dev else D.host(out)


def dense_block_forward(x, y, w: DenseBlockWeights, params: AttentionParams):
    """Pre-norm residual dense block (`recon_pipeline.py:154-184`): both
    streams update from the same pre-block state. Returns (x', y')."""
    require(x.shape[0] > 0 and y.shape[0] > 0, "dense block needs nonempty token streams")
    d = params.model_dim
    require(x.shape[1] == d and y.shape[1] == d, "token width mismatch")
    on_dev = D.is_device(x)
    xd, yd = D.dev(x, torch.float32), D.dev(y, torch.float32)
    _, xh = _add_ln(xd, None, w.ln_attn_x)
    _, yh = _add_ln(yd, None, w.ln_attn_y)
    lx = _ops.gemm(xh, D.weight(w.gate_x_w))
    ly = _ops.gemm(yh, D.weight(w.gate_y_w))
    o = {"xs": mha_forward(xh, xh, w.x_self, params), "xc": mha_forward(xh, yh, w.x_cross, params),
         "ys": mha_forward(yh, yh, w.y_self, params), "yc": mha_forward(yh, xh, w.y_cross, params)}
    outs = []
    for base, lg, gb, os_, oc, ln, ffn in ((xd, lx, w.gate_x_b, o["xs"], o["xc"], w.ln_ffn_x, w.ffn_x),
                                          (yd, ly, w.gate_y_b, o["ys"], o["yc"], w.ln_ffn_y, w.ffn_y)):
        x1, h = _gate_mix_ln(1, base, lg, lg.stride(0), D.weight(gb), os_, oc, ln)
        t = _bias_act(1, _ops.gemm(h, D.weight(ffn.w1)), D.weight(ffn.b1), 1)
        outs.append(_bias_act(1, _ops.gemm(t, D.weight(ffn.w2)), D.weight(ffn.b2), 0,
                              residual=x1))
    return tuple(a if on_dev else D.host(a) for a in outs)


def dense_stage_forward(x0, y0, weights, params: AttentionParams):
    """`recon_pipeline.py:187-193`."""
    on_dev = D.is_device(x0)
    x, y = D.dev(x0, torch.float32), D.dev(y0, torch.float32)
    for w in weights:
        x, y = dense_block_forward(x, y, w, params)
    return (x, y) if on_dev else (D.host(x), D.host(y))


# ---------------------------------------------------------------------------
# feature decode (recon_pipeline.py:196-348; csrc/decode.cu)

T_SIDE = 4          # per-axis decode upsampling (recon_pipeline.py:36)
FEATURE_DIM = 32    # decoded feature channels (recon_pipeline.py:37)


@dataclass
class DecodeWeights:
    """`recon_pipeline.py:197-199`: weight [d, T^3 * d_f], bias."""
    weight: np.ndarray
    bias: np.ndarray


def init_decode(seed: int, d: int, *tags, d_f: int = FEATURE_DIM,
                scale: float = 0.02) -> DecodeWeights:
    """`recon_pipeline.py:202-206`."""
    out = (T_SIDE ** 3) * d_f
    return DecodeWeights(normal_f32(seed, (d, out), scale, *tags, "dec"),
                         np.zeros(out, dtype=DTYPE))


@dataclass
class FeatureVolume:
    """`recon_pipeline.py:271-283`; arrays may be NumPy or CUDA tensors."""
    dense: object
    sparse_index: object = None
    sparse_rows: object = None

    @property
    def s_df(self) -> int:
        return int(self.dense.shape[0])

    @property
    def s_f(self):
        return None if self.sparse_index is None else int(self.sparse_index.shape[0])


@dataclass
class DecoderHeads:
    """`recon_pipeline.py:286-289`: [(w, b, act), ...] per head."""
    z_layers: list
    s_layers: list


def init_decoder_heads(seed: int, d_f: int = FEATURE_DIM, z_channels: int = 3,
                       hidden: int = 64, scale: float = 0.02) -> DecoderHeads:
    """`recon_pipeline.py:292-301`."""
    def head(tag, out_dim, act):
        w1 = normal_f32(seed, (d_f, hidden), scale, "head", tag, "w1")
        w2 = normal_f32(seed, (hidden, out_dim), scale, "head", tag, "w2")
        return [(w1, np.zeros(hidden, dtype=DTYPE), "gelu"),
                (w2, np.zeros(out_dim, dtype=DTYPE), act)]
    return DecoderHeads(head("z", z_channels, "sigmoid"), head("s", 1, "identity"))


def _affine_dec(x, w: DecodeWeights):
    """f32(x W + b) with the reference's f64 einsum accumulation
    (`tensor_core.py:100-116`; csrc/decode.cu `lsrm_affine_exact`), so the
    decoded grid -- which the decoded-geometry voxel mask thresholds -- is
    the reference's bit for bit."""
    return affine_exact(x, w.weight, w.bias)


def affine_exact(x, weight, bias=None, act: int = 0):
    """`tensor_core.affine` (+ activation 0 identity / 1 gelu / 2 sigmoid):
    f32 storage, f64 accumulation in np.einsum's order, on the GPU."""
    xd = D.dev(x, torch.float32)
    n, din = int(xd.shape[0]), int(xd.shape[1])
    wd = D.weight(weight)
    require(int(wd.shape[0]) == din, f"affine dim mismatch: x has {din}, weight expects "
            f"{int(wd.shape[0])}")
    dout = int(wd.shape[1])
    bd = D.weight(bias) if bias is not None else None
    y = D.empty((n, dout), torch.float32)
    call("lsrm_affine_exact", xd.data_ptr(), xd.stride(0), n, din, wd.data_ptr(), D.ptr(bd),
         dout, act, y.data_ptr(), y.stride(0), D.stream())
    return y


def decode_feature_volume(x_d, w: DecodeWeights, d_f: int = FEATURE_DIM):
    """Dense feature grid [4s, 4s, 4s, d_f] from the coarse token cube
    (`recon_pipeline.py:223-231`)."""
    on_dev = D.is_device(x_d)
    xd = D.dev(x_d, torch.float32)
    n = int(xd.shape[0])
    side = round(n ** (1.0 / 3.0))
    if side ** 3 != n:
        from .errors import ConfigurationError
        raise ConfigurationError(f"{n} tokens is not a cubic grid")
    require(w.weight.shape[1] == (T_SIDE ** 3) * d_f, "decode width mismatch")
    vec = _affine_dec(xd, w)
    s = side * T_SIDE
    grid = D.empty((s, s, s, d_f), torch.float32)
    call("lsrm_decode_scatter", vec.data_ptr(), side, T_SIDE, d_f, grid.data_ptr(), D.stream())
    return grid if on_dev else D.host(grid)


def build_sparse_features(tokens, w: DecodeWeights, d_f: int = FEATURE_DIM):
    """(index [S_f^3] int64 with -1 for absent cells, rows [M, d_f]) over the
    4^3 cells of every active volume token (`recon_pipeline.py:234-268`)."""
    require(tokens.modality == "volume", "sparse decode needs volume tokens")
    on_dev = D.is_device(tokens.features)
    s_f = T_SIDE * int(tokens.grid_res[0])
    index = D.empty((s_f, s_f, s_f), torch.int64)
    n = int(tokens.count)
    rows = D.empty((n * T_SIDE ** 3, d_f), torch.float32)
    vec = _affine_dec(D.dev(tokens.features, torch.float32), w) if n else rows
    coords = D.dev(tokens.coords, torch.int64)
    call("lsrm_sparse_features", vec.data_ptr(), coords.data_ptr(), n, T_SIDE, d_f, s_f,
         index.data_ptr(), rows.data_ptr(), D.stream())
    return (index, rows) if on_dev else (D.host(index), D.host(rows))


def _points(points):
    from .errors import OutOfDomainError
    pts = D.dev(points, torch.float64).reshape(-1, 3)
    bad = (pts < 0.0) | (pts > 1.0)
    if bool(bad.any()):
        p = D.host(pts[bad.any(dim=1)][0])
        raise OutOfDomainError(f"point outside the unit cube: {p.tolist()}")
    return pts


def _decode(fv: FeatureVolume, points, heads: DecoderHeads = None, want_field=False):
    dense = D.dev(fv.dense, torch.float32)
    s_df, d_f = int(dense.shape[0]), int(dense.shape[3])
    require(s_df >= 2, "trilinear needs side >= 2")
    pts = _points(points)
    n = int(pts.shape[0])
    idx = rows = None
    s_f = 0
    if fv.sparse_index is not None:
        idx = D.dev(fv.sparse_index, torch.int64)
        rows = D.dev(fv.sparse_rows, torch.float32)
        s_f = int(idx.shape[0])
    field = D.empty((n, d_f), torch.float32) if want_field else None
    z = s = hw = None
    hidden = zc = 1
    if heads is not None:
        (zw1, zb1, _), (zw2, zb2, _) = heads.z_layers
        (sw1, sb1, _), (sw2, sb2, _) = heads.s_layers
        ws = [D.weight(a) for a in (zw1, zb1, zw2, zb2, sw1, sb1, sw2, sb2)]
        hw = (ctypes.c_void_p * 8)(*[t.data_ptr() for t in ws])
        hidden, zc = int(zw1.shape[1]), int(zw2.shape[1])
        z = D.empty((n, zc), torch.float32)
        s = D.empty((n,), torch.float32)
    call("lsrm_decode_points", dense.data_ptr(), s_df, D.ptr(idx), D.ptr(rows), s_f, d_f,
         pts.data_ptr(), n, hw, hidden, zc, D.ptr(z), D.ptr(s), D.ptr(field), D.stream())
    return z, s, field


def query_field(fv: FeatureVolume, mask, points):
    """Blended sparse/dense feature lookup (`recon_pipeline.py:304-346`)."""
    require(fv.sparse_index is not None, "feature volume has no sparse part")
    require(mask.shape[0] * T_SIDE == fv.s_f, "mask resolution does not match the sparse grid")
    on_dev = D.is_device(points)
    _, _, f = _decode(fv, points, want_field=True)
    return f if on_dev else D.host(f)


def decode_points(fv: FeatureVolume, heads: DecoderHeads, points, mask=None):
    """(z, s) at query points (`recon_pipeline.py:349-365`): the blended
    sparse query when the volume has a sparse part, else dense trilinear; z
    through the sigmoid head, s through the SDF head + bounding-sphere offset."""
    if fv.sparse_index is not None:
        require(mask is not None, "sparse field query needs the voxel mask")
        require(mask.shape[0] * T_SIDE == fv.s_f,
                "mask resolution does not match the sparse grid")
    on_dev = D.is_device(points)
    z, s, _ = _decode(fv, points, heads)
    return (z, s) if on_dev else (D.host(z), D.host(s))


def decode_point(fv: FeatureVolume, heads: DecoderHeads, p, mask=None):
    """`recon_pipeline.py:368-371`."""
    z, s = decode_points(fv, heads, np.asarray(p, np.float64).reshape(1, 3), mask)
    return z[0], float(s[0])


class SparseStageEngine:
    """The Stage-2 sparse stage (`recon_pipeline.py:500-512`) on the bf16
    engine: `depth` SparseBlockEngines over one routing, sharing their work
    buffers (layers run one after another; only the weights are per layer).
    forward(x_up, y_up) takes the fine tokens' f32 features in block-major
    order and returns the stage output x_s, y_s (f32, block-major): zero
    state, per-layer injection of the frozen inputs, inputs added at the end."""

    def __init__(self, part_vol: BlockPartition, part_img: BlockPartition, plan_rows: dict,
                 weights: list, params: AttentionParams, uses: list = None,
                 shard: dict = None):
        self.pool = {}
        uses = uses or [None] * len(weights)
        self.blocks = [SparseBlockEngine(part_vol, part_img, plan_rows, w, params, pool=self.pool,
                                         uses=u, shard=shard) for w, u in zip(weights, uses)]
        # injection weights transposed for the tcgen05 GEMM
        self.inj = [(D.dev(np.asarray(w.inj_x).T, torch.bfloat16),
                     D.dev(np.asarray(w.inj_y).T, torch.bfloat16)) for w in weights]

    def forward(self, x_up: torch.Tensor, y_up: torch.Tensor, out=None):
        """out: optional (x_s, y_s) f32 buffers to write the stage output to."""
        xb, yb = _ops.cast(x_up, torch.bfloat16), _ops.cast(y_up, torch.bfloat16)
        x, y = torch.zeros_like(x_up), torch.zeros_like(y_up)
        xi = D.empty(tuple(x_up.shape), torch.float32)
        yi = D.empty(tuple(y_up.shape), torch.float32)
        for blk, (ix, iy) in zip(self.blocks, self.inj):
            _ops.gemm_tc([_ops.gemm_problem(a, wt, o) for a, wt, o in ((xb, ix, xi), (yb, iy, yi))
                          if a.shape[0]])
            x, y = blk.forward(x, y, xi, yi)
        zero = torch.zeros(x_up.shape[1], dtype=torch.float32, device=x_up.device)
        ox, oy = out if out is not None else (None, None)
        return (_bias_act(0, x, zero, 0, residual=x_up, out=ox, out_dtype=torch.float32),
                _bias_act(0, y, zero, 0, residual=y_up, out=oy, out_dtype=torch.float32))
