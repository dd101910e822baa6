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

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev as D
from . import _ops
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


def _add_ln(a, b, norm: NormParams, out_dtype=torch.float32):
    """sum = f32(a + b), LayerNorm(sum) -> (sum f32, normalised)."""
    n, d = a.shape
    s = D.empty((n, d), torch.float32)
    y = D.empty((n, d), out_dtype)
    call("lsrm_add_layer_norm", a.data_ptr(), D.ptr(b), int(b is not None and
                                                           b.dtype == torch.bfloat16),
         n, d, D.weight(norm.gamma).data_ptr(), D.weight(norm.beta).data_ptr(), LN_EPS, s.data_ptr(),
         int(out_dtype == torch.bfloat16), y.data_ptr(), D.stream())
    return s, y


def _gate_mix_ln(exact, xe, logits, ld, gate_b, o_self, o_cross, norm: NormParams,
                 out_dtype=torch.float32):
    """x1 = f32(xe + sig(self logits) * o_self + sig(cross logits) * o_cross),
    h = LayerNorm(x1)."""
    n, d = xe.shape
    x1 = D.empty((n, d), torch.float32)
    h = D.empty((n, d), out_dtype)
    call("lsrm_gate_mix_layer_norm", int(exact), xe.data_ptr(), logits.data_ptr(), ld,
         int(logits.dtype == torch.bfloat16), gate_b.data_ptr(), o_self.data_ptr(),
         o_cross.data_ptr(), int(o_self.dtype == torch.bfloat16), n, d, x1.data_ptr(),
         D.weight(norm.gamma).data_ptr(), D.weight(norm.beta).data_ptr(), LN_EPS,
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
                 w: SparseBlockWeights, params: AttentionParams):
        self.w, self.params = w, params
        self.layer = SparseLayerEngine(part_vol, part_img, plan_rows, w.uses(), params,
                                       extra_cols={"x": w.gate_x_w, "y": w.gate_y_w})
        self.bf = {name: D.weight(getattr(getattr(w, f), n), torch.bfloat16)
                   for name, f, n in (("fx1", "ffn_x", "w1"), ("fx2", "ffn_x", "w2"),
                                      ("fy1", "ffn_y", "w1"), ("fy2", "ffn_y", "w2"))}

    def forward(self, x, y, x_inj, y_inj):
        w, L = self.w, self.layer
        xe, xh = _add_ln(x, x_inj, w.ln_attn_x, torch.bfloat16)
        ye, yh = _add_ln(y, y_inj, w.ln_attn_y, torch.bfloat16)
        outs = L.forward(xh, yh)
        res = []
        for s, e, gb, us, uc, ln, k1, k2, ffn in (
                ("x", xe, D.weight(w.gate_x_b), "v2v", "v2i", w.ln_ffn_x, "fx1", "fx2", w.ffn_x),
                ("y", ye, D.weight(w.gate_y_b), "i2i", "i2v", w.ln_ffn_y, "fy1", "fy2", w.ffn_y)):
            Y = L.buf[("Y", s)]
            lg = Y[:, L.cols[("extra", s)]:]
            x1, h = _gate_mix_ln(0, e, lg, Y.stride(0), gb, outs[us], outs[uc], ln,
                                 torch.bfloat16)
            t = _ops.gemm(h, self.bf[k1])
            _bias_act(0, t, D.weight(ffn.b1), 1)
            u = _ops.gemm(t, self.bf[k2], out_dtype=torch.float32)
            res.append(_bias_act(0, u, D.weight(ffn.b2), 0, residual=x1))
        return tuple(res)
