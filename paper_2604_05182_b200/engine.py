"""Device-resident bf16 fast path of one LSRM sparse-attention layer.

A "layer" is the four gated NSA uses of a Stage-2 block (v2v, v2i, i2i, i2v;
`lsrm/recon_pipeline.py:477-488`).  Everything stays on the GPU in the
block-major order of each modality's own partition, so that

  * every KV block is one contiguous row range (one bulk-async copy),
  * query tiles never straddle blocks (window branch + W-invariance),
  * the routed selections are expressed as occupied-row indices.

Per layer and stream, ONE bf16 GEMM (cuBLAS) computes all projections that
read that stream: the q and gate columns of its two query uses and the k/v
columns of the two uses that read it as KV.  Then per use: ResBlock
compression (fp32, csrc/compress.cu), K/V re-layout into the padded
core-matrix layout (csrc/attn_tc.cu), the fused tcgen05 three-branch
attention with the gated merge, and the W_o GEMM.

Numerics: bf16 storage, fp32 accumulation (tensor cores), fp32 softmax with
bf16 probabilities, fp32 compression.  Tolerance vs the f32/f64 reference is
stated in DESIGN.md and enforced in tests/test_gpu_engine.py.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev as D
from . import _ops
from ._native import call
from .block_partition import BlockPartition, _dev_res
from .errors import require
from .tensor_core import AttentionParams

USES = ("v2v", "v2i", "i2i", "i2v")
# (query stream, kv stream, n_gates) per use
USE_GEOM = {"v2v": ("x", "x", 3), "v2i": ("x", "y", 2), "i2i": ("y", "y", 3),
            "i2v": ("y", "x", 2)}
ROW_PAD = 16
ONES_COLS = 16   # extra V columns (1 = real key) that make P.V also emit row sums


@dataclass
class StreamMeta:
    """Device metadata of one modality in its own block-major order."""
    part: BlockPartition
    n: int
    n_blocks: int
    kv_off: torch.Tensor        # [B+1] int64 block offsets (block-major == identity)
    pad_off: torch.Tensor       # [B+1] int64 16-row padded offsets
    n_rows_pad: int
    ident: torch.Tensor         # [n] int64 arange (block-major token ids)
    pad_off_host: np.ndarray
    pad_row: torch.Tensor       # [n] int32 padded row of every (block-major) token


def stream_meta(part: BlockPartition) -> StreamMeta:
    occ = part.occupancy.astype(np.int64)
    padded = (occ + ROW_PAD - 1) // ROW_PAD * ROW_PAD
    pad_off = np.concatenate([[0], np.cumsum(padded)]).astype(np.int64)
    blk = np.repeat(np.arange(part.n_occupied), occ)
    pad_row = (pad_off[:-1][blk] + np.arange(part.n_tokens) - part.block_offsets[:-1][blk])
    return StreamMeta(part, part.n_tokens, part.n_occupied, part.dev("block_offsets"),
                      D.dev(pad_off), int(pad_off[-1]),
                      D.dev(np.arange(part.n_tokens, dtype=np.int64)), pad_off,
                      D.dev(pad_row.astype(np.int32)))


def query_tiles(part: BlockPartition, group: int, self_use: bool) -> np.ndarray:
    """[n_tiles, 4] int32 (first query, count, own kv row or -1, 0): tiles of
    128/group tokens that never straddle a query block."""
    T = 128 // group
    occ = part.occupancy.astype(np.int64)
    off = part.block_offsets.astype(np.int64)
    n_t = (occ + T - 1) // T
    rows = np.repeat(np.arange(part.n_occupied), n_t)
    k = np.arange(int(n_t.sum())) - np.repeat(np.cumsum(n_t) - n_t, n_t)
    first = off[rows] + k * T
    cnt = np.minimum(T, occ[rows] - k * T)
    own = rows if self_use else np.full_like(rows, -1)
    return np.stack([first, cnt, own, np.zeros_like(rows)], axis=1).astype(np.int32)


def block_major_rows(rows_tok, count_tok, part_q: BlockPartition, part_kv: BlockPartition,
                     self_use: bool):
    """Routed rows (token order) -> fallback-resolved rows in the query
    partition's block-major order (`nsa_attention.py:133-144`)."""
    n, kmax = int(rows_tok.shape[0]), int(rows_tok.shape[1])
    res_rows = D.empty((n, kmax), torch.int32)
    res_count = D.empty((n,), torch.int32)
    own_row = part_kv.dev("row_of_token") if self_use else None
    call("lsrm_build_gather_table", rows_tok.data_ptr(), count_tok.data_ptr(), n, kmax,
         D.ptr(own_row), 1, part_kv.dev("block_offsets").data_ptr(),
         part_kv.dev("block_token_ids").data_ptr(), 0, res_rows.data_ptr(),
         res_count.data_ptr(), None, None, None, D.stream())
    tok = part_q.dev("block_token_ids")
    return _ops.gather_rows(res_rows, tok), _ops.gather_rows(res_count.view(n, 1), tok).view(n)


class SparseLayerEngine:
    """Four gated NSA uses over device-resident, block-major bf16 streams.

    weights: dict use -> NsaWeights (reference layout, f32 host arrays).
    plan_rows: dict use -> (rows [n, kmax] int32, count [n] int32), token
    order, as produced by `block_routing.build_routing_plan(...).device_rows`.
    """

    def __init__(self, part_vol: BlockPartition, part_img: BlockPartition, plan_rows: dict,
                 weights: dict, params: AttentionParams):
        require(params.head_dim in (32, 64), "bf16 engine: head_dim must be 32 or 64")
        G = params.group_size
        require(128 % G == 0, "bf16 engine: (n_q_heads/n_kv_heads) must divide 128")
        self.params = params
        d, w = params.model_dim, params.n_kv_heads * params.head_dim
        self.d, self.w = d, w
        self.meta = {"x": stream_meta(part_vol), "y": stream_meta(part_img)}
        parts = {"x": part_vol, "y": part_img}
        # fused projection weights per stream: [q|gates] of its query uses, then
        # [k|v] of the uses that read it as KV
        self.cols = {}
        wcat = {"x": [], "y": []}
        ncol = {"x": 0, "y": 0}
        for use in USES:
            qs, _, ng = USE_GEOM[use]
            wu = weights[use]
            self.cols[(use, "q")] = ncol[qs]
            wcat[qs] += [wu.w_q, wu.gate_w]
            ncol[qs] += d + ng * d
        for use in USES:
            _, ks, _ = USE_GEOM[use]
            wu = weights[use]
            self.cols[(use, "k")] = ncol[ks]
            self.cols[(use, "v")] = ncol[ks] + w
            wcat[ks] += [wu.w_k, wu.w_v]
            ncol[ks] += 2 * w
        self.ncol = ncol
        self.w_cat = {s: D.dev(np.concatenate(wcat[s], axis=1), torch.bfloat16) for s in wcat}
        self.w_o = {u: D.dev(weights[u].w_o, torch.bfloat16) for u in USES}
        self.gate_b = {u: D.dev(weights[u].gate_b, torch.float32) for u in USES}
        self.cmp_w = {u: (_dev_res(weights[u].compress.for_k), _dev_res(weights[u].compress.for_v))
                      for u in USES}
        # per-use routing and tiles
        self.rows, self.count, self.tiles, self.kmax = {}, {}, {}, {}
        for use in USES:
            qs, ks, ng = USE_GEOM[use]
            r, c = plan_rows[use]
            rb, cb = block_major_rows(r, c, parts[qs], parts[ks], ng == 3)
            self.rows[use], self.count[use] = rb, cb
            self.kmax[use] = int(rb.shape[1])
            self.tiles[use] = D.dev(query_tiles(parts[qs], G, ng == 3))
        # work buffers
        self.buf = {}
        for s in ("x", "y"):
            m = self.meta[s]
            self.buf[("Y", s)] = D.empty((m.n, ncol[s]), torch.bfloat16)
            # zero once: padding rows (and their ones columns) are never written again
            self.buf[("k_il", s)] = D.zeros((params.n_kv_heads, m.n_rows_pad, params.head_dim),
                                            torch.bfloat16)
            self.buf[("v_il", s)] = D.zeros(
                (params.n_kv_heads, m.n_rows_pad, params.head_dim + ONES_COLS), torch.bfloat16)
            bpad = (m.n_blocks + ROW_PAD - 1) // ROW_PAD * ROW_PAD
            self.buf[("kc_il", s)] = D.empty((params.n_kv_heads, bpad, params.head_dim),
                                             torch.bfloat16)
            self.buf[("vc_il", s)] = D.empty(
                (params.n_kv_heads, bpad, params.head_dim + ONES_COLS), torch.bfloat16)
            self.buf[("kc", s)] = D.empty((m.n_blocks, w), torch.float32)
            self.buf[("vc", s)] = D.empty((m.n_blocks, w), torch.float32)
            self.buf[("scratch", s)] = D.empty((m.n, w), torch.float32)
        for use in USES:
            qs = USE_GEOM[use][0]
            self.buf[("merged", use)] = D.empty((self.meta[qs].n, d), torch.bfloat16)
            self.buf[("out", use)] = D.empty((self.meta[qs].n, d), torch.bfloat16)

    # -- pieces --------------------------------------------------------------
    def project(self, x_bm: torch.Tensor, y_bm: torch.Tensor):
        _ops.gemm(x_bm, self.w_cat["x"], out=self.buf[("Y", "x")])
        _ops.gemm(y_bm, self.w_cat["y"], out=self.buf[("Y", "y")])

    def prepare_kv(self, use: str):
        _, ks, _ = USE_GEOM[use]
        m, p = self.meta[ks], self.params
        Y = self.buf[("Y", ks)]
        ld = Y.stride(0)
        st = D.stream()
        for kind, wres in (("k", self.cmp_w[use][0]), ("v", self.cmp_w[use][1])):
            col = self.cols[(use, kind)]
            src = Y[:, col:]
            ones = ONES_COLS if kind == "v" else 0   # V gets the row-sum columns
            cmp = self.buf[(kind + "c", ks)]
            w1, b1, w2, b2 = wres
            # fused: interleaved K/V layout + fp32 ResBlock + per-block mean
            call("lsrm_kv_prepare", src.data_ptr(), ld, m.n, p.n_kv_heads, p.head_dim,
                 m.pad_row.data_ptr(), m.n_rows_pad, self.buf[(kind + "_il", ks)].data_ptr(), ones,
                 w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(),
                 self.buf[("scratch", ks)].data_ptr(), m.kv_off.data_ptr(), m.n_blocks,
                 cmp.data_ptr(), st)
            il = self.buf[(kind + "c_il", ks)]
            call("lsrm_kv_interleave", 0, cmp.data_ptr(), self.w, m.n_blocks, p.n_kv_heads,
                 p.head_dim, ones, None, None, 0, None, int(il.shape[1]), il.data_ptr(), st)

    def attend(self, use: str):
        qs, ks, ng = USE_GEOM[use]
        mq, mk, p = self.meta[qs], self.meta[ks], self.params
        Y = self.buf[("Y", qs)]
        qcol = self.cols[(use, "q")]
        q = Y[:, qcol:]
        tiles = self.tiles[use]
        call("lsrm_nsa_attention_tc", q.data_ptr(), Y.stride(0), mq.n, p.n_q_heads,
             p.n_kv_heads, p.head_dim, self.buf[("k_il", ks)].data_ptr(),
             self.buf[("v_il", ks)].data_ptr(), mk.pad_off.data_ptr(), mk.kv_off.data_ptr(),
             mk.n_rows_pad, self.buf[("kc_il", ks)].data_ptr(),
             self.buf[("vc_il", ks)].data_ptr(), mk.n_blocks, tiles.data_ptr(),
             int(tiles.shape[0]), self.rows[use].data_ptr(), self.count[use].data_ptr(),
             self.kmax[use], Y.data_ptr(), Y.stride(0), qcol + self.d,
             self.gate_b[use].data_ptr(), ng, self.buf[("merged", use)].data_ptr(), D.stream())

    def output(self, use: str):
        _ops.gemm(self.buf[("merged", use)], self.w_o[use], out=self.buf[("out", use)])

    # -- whole layer ---------------------------------------------------------
    def forward(self, x_bm: torch.Tensor, y_bm: torch.Tensor) -> dict:
        """x_bm [Nv, d], y_bm [Ni, d] bf16 (LN'd, block-major) -> dict use ->
        [Nq, d] bf16 (block-major).  Output buffers are reused across calls."""
        self.project(x_bm, y_bm)
        for use in USES:
            self.prepare_kv(use)
            self.attend(use)
            self.output(use)
        return {u: self.buf[("out", u)] for u in USES}

    # -- accounting ------------------------------------------------------------
    def attention_flops(self) -> dict:
        """Algorithmic attention-core FLOPs per use: useful
        work only (no padding, union inflation or masked keys)."""
        p = self.params
        out = {}
        for use in USES:
            qs, ks, ng = USE_GEOM[use]
            pk = self.meta[ks].part
            nq = self.meta[qs].n
            rows = D.host(self.rows[use])
            cnt = D.host(self.count[use])
            occ = pk.occupancy.astype(np.float64)
            mask = np.arange(rows.shape[1])[None, :] < cnt[:, None]
            L = np.where(mask, occ[np.clip(rows, 0, None)], 0.0).sum(axis=1)
            cmp = 4.0 * nq * p.n_q_heads * p.head_dim * pk.n_occupied
            sel = 4.0 * p.n_q_heads * p.head_dim * L.sum()
            win = 4.0 * p.n_q_heads * p.head_dim * float((occ ** 2).sum()) if ng == 3 else 0.0
            out[use] = {"cmp": cmp, "sel": sel, "win": win}
        return out

    def projection_flops(self) -> float:
        return sum(2.0 * self.meta[s].n * self.d * self.ncol[s] for s in ("x", "y")) + \
            sum(2.0 * self.meta[USE_GEOM[u][0]].n * self.d * self.d for u in USES)
