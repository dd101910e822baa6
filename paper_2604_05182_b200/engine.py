"""Device-resident bf16 fast path of one LSRM sparse-attention layer.

A "layer" is the four gated NSA uses of a Stage-2 block (v2v, v2i, i2i, i2v;
`lsrm/recon_pipeline.py:477-488`).  Everything stays on the GPU in the
block-major order of each modality's own partition, so that

  * every KV block is one contiguous row range (one bulk-async copy),
  * query tiles never straddle blocks (window branch + W-invariance),
  * the routed selections are expressed as occupied-row indices.

Per layer, ONE grouped tcgen05 GEMM launch (csrc/gemm_tc.cu) computes, for
each stream, all projections that read it: the q and gate columns of its two
query uses and the k/v columns of the two uses that read it as KV.  Then ONE launch prepares the K/V
of all four uses (interleaved layout + tensor-core ResBlock + block mean,
written straight into the compressed layout; csrc/kv_prep.cu), and per use
the fused tcgen05 three-branch attention with the gated merge
(csrc/attn_tc.cu) and the four W_o GEMMs (one grouped launch).

Sharding (block-aware sequence parallelism, seq_parallel.py): an engine can
own only a subset of each stream's blocks.  Its query side then works on the
owned tokens in a rank-local compact order (owned blocks, canonical order);
its KV side computes K/V and compression for the owned KV blocks and an
`exchange` hook (All-gather-KV) assembles the canonical global KV buffers
that every rank's attention reads — so each output row is computed from the
same inputs by the same tile regardless of the number of ranks.

Numerics: bf16 storage, fp32 accumulation (tensor cores), fp32 softmax with
bf16 probabilities, fp32 compression.  Tolerance vs the f32/f64 reference is
stated in DESIGN.md and enforced in tests/test_gpu_parity.py.
"""

from dataclasses import dataclass

import ctypes as C
import os

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
ONES_COLS = 16
# cross uses (v2i, i2v) may tile their signature-sorted tokens across query
# blocks (LSRM_CROSS_GLOBAL_TILES=1: ~5% faster attention).  Off by default: a
# row's online-softmax rescale points depend on how its keys fall into the
# tile's chunks, so tiles that mix blocks make results depend on tile-mates,
# and a sharded rank (which owns whole blocks) could not reproduce them.  With
# block tiles every output row is bit-identical for every world size W
# (the reference's serial == parallel contract, tests/test_seq_parallel.py).
CROSS_GLOBAL_TILES = os.environ.get("LSRM_CROSS_GLOBAL_TILES", "0") != "0"
# self uses tile across blocks too; their window branch then spans each tile's
# distinct own blocks (per-token own rows). Correct, measured neutral
# (1.230 -> 1.236 ms), so off.
SELF_GLOBAL_TILES = os.environ.get("LSRM_SELF_GLOBAL_TILES", "0") != "0"
# self uses keep block tiles but pool every block's partial last tile with the
# others' into full tiles (per-token own rows for the window branch).
# Correct, measured neutral (the LPT queue already hides the small items): off.
PACK_SELF_TAILS = os.environ.get("LSRM_PACK_SELF_TAILS", "0") != "0"
# self uses run cmp + sel on such tiles and the window branch in a second,
# accumulating launch (correct, measured slower: 1.23 -> 1.31 ms; off)
SPLIT_SELF_WINDOW = os.environ.get("LSRM_SPLIT_SELF_WINDOW", "0") != "0"   # extra V columns (1 = real key) that make P.V also emit row sums


def _padded(occ: np.ndarray) -> np.ndarray:
    return (occ + ROW_PAD - 1) // ROW_PAD * ROW_PAD


class KvJob(C.Structure):
    """Mirror of `lsrm_kv_job` (include/lsrm_b200.h)."""
    _fields_ = [("src", C.c_void_p), ("ld", C.c_int64), ("blk_off", C.c_void_p),
                ("pad_off", C.c_void_p), ("n_blocks", C.c_int64), ("rows_pad", C.c_int64),
                ("il", C.c_void_p), ("ones_cols", C.c_int64), ("w1", C.c_void_p),
                ("b1", C.c_void_p), ("w2", C.c_void_p), ("b2", C.c_void_p),
                ("mean_out", C.c_void_p), ("cmp_il", C.c_void_p), ("cmp_rows_pad", C.c_int64),
                ("work", C.c_void_p), ("n_work", C.c_int64), ("partial", C.c_void_p),
                ("arrive", C.c_void_p)]


class NsaUse(C.Structure):
    """Mirror of `lsrm_nsa_use` (include/lsrm_b200.h)."""
    _fields_ = [("q", C.c_void_p), ("ld_q", C.c_int64), ("nq", C.c_int64),
                ("k_il", C.c_void_p), ("v_il", C.c_void_p), ("pad_offsets", C.c_void_p),
                ("kv_offsets", C.c_void_p), ("n_kv_rows_pad", C.c_int64),
                ("kcmp_il", C.c_void_p), ("vcmp_il", C.c_void_p), ("n_blocks", C.c_int64),
                ("tiles", C.c_void_p), ("n_tiles", C.c_int64), ("rows", C.c_void_p),
                ("count", C.c_void_p), ("kmax_rows", C.c_int64), ("gate_logits", C.c_void_p),
                ("ld_gl", C.c_int64), ("gate_col0", C.c_int64), ("n_gates", C.c_int64),
                ("merged", C.c_void_p), ("perm", C.c_void_p), ("branch_first", C.c_int64),
                ("accumulate", C.c_int64), ("own_rows", C.c_void_p),
                ("branch_out", C.c_void_p), ("branch_lse", C.c_void_p)]


class PackedShard:
    """Byte layout of one rank's KV shard for one use: interleaved K
    [hkv, rows_pad, dh] bf16, V [hkv, rows_pad, dh+16] bf16, compressed K and
    V [n_blocks, w] f32 (every section a multiple of 16 bytes)."""

    def __init__(self, hkv: int, dh: int, w: int, n_rows_pad: int, n_blocks: int):
        self.rows_pad = max(int(n_rows_pad), ROW_PAD)
        self.n_blocks = max(int(n_blocks), 1)
        self.off_v = hkv * self.rows_pad * dh * 2
        self.off_kc = self.off_v + hkv * self.rows_pad * (dh + ONES_COLS) * 2
        self.off_vc = self.off_kc + self.n_blocks * w * 4
        self.total = self.off_vc + self.n_blocks * w * 4


@dataclass
class StreamMeta:
    """One modality: canonical (global) KV layout + this engine's owned shard.

    Global: block-major token order, 16-row padded block segments in ascending
    occupied-row order.  Local: the owned blocks' tokens, same order, compact.
    """
    part: BlockPartition
    n: int                      # global tokens
    n_blocks: int
    kv_off: torch.Tensor        # [B+1] int64 global block offsets
    pad_off: torch.Tensor       # [B+1] int64 global padded offsets
    pad_off_host: np.ndarray
    n_rows_pad: int
    owned: np.ndarray           # owned occupied rows (ascending)
    n_loc: int
    loc2glob: torch.Tensor      # [n_loc] int64 global block-major index of local tokens
    loc_off: torch.Tensor       # [B_loc+1] local block offsets
    loc_off_host: np.ndarray
    loc_pad_row: torch.Tensor   # [n_loc] int32 padded row in the local compact layout
    loc_pad_off_host: np.ndarray
    loc_pad_off: torch.Tensor   # [B_loc+1] int64 padded offsets in the local compact layout
    n_loc_rows_pad: int
    sharded: bool


def stream_meta(part: BlockPartition, owned=None) -> StreamMeta:
    occ = part.occupancy.astype(np.int64)
    off = part.block_offsets.astype(np.int64)
    pad_off = np.concatenate([[0], np.cumsum(_padded(occ))]).astype(np.int64)
    sharded = owned is not None
    owned = np.arange(part.n_occupied) if owned is None else np.sort(np.asarray(owned, np.int64))
    occ_l = occ[owned]
    loc_off = np.concatenate([[0], np.cumsum(occ_l)]).astype(np.int64)
    loc_pad_off = np.concatenate([[0], np.cumsum(_padded(occ_l))]).astype(np.int64)
    blk = np.repeat(np.arange(owned.size), occ_l)
    within = np.arange(int(loc_off[-1])) - loc_off[:-1][blk]
    loc2glob = off[:-1][owned][blk] + within
    loc_pad_row = loc_pad_off[:-1][blk] + within
    return StreamMeta(part, part.n_tokens, part.n_occupied, part.dev("block_offsets"),
                      D.dev(pad_off), pad_off, int(pad_off[-1]), owned, int(loc_off[-1]),
                      D.dev(loc2glob.astype(np.int64)), D.dev(loc_off), loc_off,
                      D.dev(loc_pad_row.astype(np.int32)), loc_pad_off, D.dev(loc_pad_off),
                      int(loc_pad_off[-1]), sharded)


def query_tiles(part: BlockPartition, group: int, self_use: bool, owned=None) -> np.ndarray:
    """[n_tiles, 4] int32 (first query (local index), count, own kv row or -1,
    0): tiles of 128/group tokens that never straddle a query block."""
    T = 128 // group
    rows_all = np.arange(part.n_occupied) if owned is None else np.sort(np.asarray(owned))
    occ = part.occupancy.astype(np.int64)[rows_all]
    loc_off = np.concatenate([[0], np.cumsum(occ)]).astype(np.int64)
    n_t = (occ + T - 1) // T
    idx = np.repeat(np.arange(rows_all.size), n_t)
    k = np.arange(int(n_t.sum())) - np.repeat(np.cumsum(n_t) - n_t, n_t)
    first = loc_off[idx] + k * T
    cnt = np.minimum(T, occ[idx] - k * T)
    own = rows_all[idx] if self_use else np.full(idx.size, -1)
    return np.stack([first, cnt, own, np.zeros_like(idx)], axis=1).astype(np.int32)


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
    shard: optional {"x": owned vol rows, "y": owned img rows}; `exchange`
    (seq_parallel) then fills the global KV buffers between prepare_kv and
    attend.
    extra_cols: optional {"x": W [d, m], "y": ...} appended to a stream's fused
    projection GEMM (the Stage-2 block's use gates); their output columns start
    at `self.cols[("extra", stream)]` of `buf[("Y", stream)]`.
    """

    def __init__(self, part_vol: BlockPartition, part_img: BlockPartition, plan_rows: dict,
                 weights: dict, params: AttentionParams, shard: dict = None,
                 extra_cols: dict = None, pool: dict = None):
        require(params.head_dim in (32, 64), "bf16 engine: head_dim must be 32 or 64")
        # the uses this engine runs: every use `weights` holds (a layer is all
        # four; the reference-API drop-in builds one-use engines)
        self.uses = tuple(u for u in USES if u in weights)
        require(len(self.uses) > 0, "bf16 engine: no NSA use weights given")
        G = params.group_size
        require(128 % G == 0 and G >= 4, "bf16 engine: (n_q_heads/n_kv_heads) must be in 4..128 "
                "and divide 128")
        self.params = params
        d, w = params.model_dim, params.n_kv_heads * params.head_dim
        self.d, self.w = d, w
        shard = shard or {}
        self.meta = {"x": stream_meta(part_vol, shard.get("x")),
                     "y": stream_meta(part_img, shard.get("y"))}
        self.sharded = bool(shard)
        self.exchange = None   # set by seq_parallel for sharded engines
        parts = {"x": part_vol, "y": part_img}
        # fused projection weights per stream: [q|gates] of its query uses, then
        # [k|v] of the uses that read it as KV
        # (the gate biases ride in the same GEMM's bias epilogue, so the gate
        # logits the attention reads are complete)
        self.cols = {}
        wcat = {"x": [], "y": []}
        bcat = {"x": [], "y": []}
        ncol = {"x": 0, "y": 0}
        for use in self.uses:
            qs, _, ng = USE_GEOM[use]
            wu = weights[use]
            self.cols[(use, "q")] = ncol[qs]
            wcat[qs] += [wu.w_q, wu.gate_w]
            bcat[qs] += [np.zeros(d, np.float32), np.asarray(wu.gate_b, np.float32)]
            ncol[qs] += d + ng * d
        for use in self.uses:
            _, ks, _ = USE_GEOM[use]
            wu = weights[use]
            self.cols[(use, "k")] = ncol[ks]
            self.cols[(use, "v")] = ncol[ks] + w
            wcat[ks] += [wu.w_k, wu.w_v]
            bcat[ks].append(np.zeros(2 * w, np.float32))
            ncol[ks] += 2 * w
        for s_, wx in (extra_cols or {}).items():
            self.cols[("extra", s_)] = ncol[s_]
            wcat[s_].append(np.asarray(wx, np.float32))
            bcat[s_].append(np.zeros(int(wx.shape[1]), np.float32))
            ncol[s_] += int(wx.shape[1])
        self.ncol = ncol
        # weights stored transposed ([n, k], K contiguous): both tcgen05 GEMM
        # operands K-major (csrc/gemm_tc.cu)
        self.w_cat = {s: D.dev(np.concatenate(wcat[s], axis=1).T, torch.bfloat16)
                      for s in wcat if wcat[s]}
        self.b_cat = {s: D.dev(np.concatenate(bcat[s]), torch.bfloat16) for s in bcat if bcat[s]}
        self.w_o = {u: D.dev(np.asarray(weights[u].w_o).T, torch.bfloat16) for u in self.uses}
        self.gate_b = {u: D.dev(weights[u].gate_b, torch.float32) for u in self.uses}
        self.cmp_w = {u: (_dev_res(weights[u].compress.for_k), _dev_res(weights[u].compress.for_v))
                      for u in self.uses}
        # per-use routing (local query order) and tiles
        self.rows, self.count, self.tiles, self.kmax = {}, {}, {}, {}
        for use in self.uses:
            qs, ks, ng = USE_GEOM[use]
            r, c = plan_rows[use]
            rb, cb = block_major_rows(r, c, parts[qs], parts[ks], ng == 3)
            mq = self.meta[qs]
            if mq.sharded:
                rb = _ops.gather_rows(rb, mq.loc2glob)
                cb = _ops.gather_rows(cb.view(-1, 1), mq.loc2glob).view(-1)
            self.rows[use], self.count[use] = rb, cb
            self.kmax[use] = int(rb.shape[1])
            self.tiles[use] = D.dev(query_tiles(parts[qs], G, ng == 3,
                                                mq.owned if mq.sharded else None))
        # work buffers (a `pool` shared by engines that run one after another,
        # e.g. the layers of a stage, hands out the same tensors by key)
        hkv, dh = params.n_kv_heads, params.head_dim
        self.buf = {}

        def alloc(key, shape, dtype, zero=False):
            t = pool.get(key) if pool is not None else None
            if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
                t = D.zeros(shape, dtype) if zero else D.empty(shape, dtype)
                if pool is not None:
                    pool[key] = t
            return t
        for s in ("x", "y"):
            if ncol[s]:     # a one-use engine reads one stream only for a self use
                m = self.meta[s]
                self.buf[("Y", s)] = alloc(("Y", s), (m.n_loc, ncol[s]), torch.bfloat16)
        for use in self.uses:
            qs, ks, _ = USE_GEOM[use]
            m = self.meta[ks]
            # global KV of this use (zeroed once: padding rows, their ones
            # columns and the compressed padding rows stay 0)
            for key, shape, zero in (
                    (("k_il", use), (hkv, m.n_rows_pad, dh), True),
                    (("v_il", use), (hkv, m.n_rows_pad, dh + ONES_COLS), True),
                    (("kc_il", use), (hkv, (m.n_blocks + ROW_PAD - 1) // ROW_PAD * ROW_PAD, dh),
                     True),
                    (("vc_il", use), (hkv, (m.n_blocks + ROW_PAD - 1) // ROW_PAD * ROW_PAD,
                                      dh + ONES_COLS), True),
                    (("merged", use), (self.meta[qs].n_loc, d), False),
                    (("out", use), (self.meta[qs].n_loc, d), False)):
                self.buf[key] = alloc(key, shape, torch.bfloat16, zero)
            self.buf[("kc", use)] = alloc(("kc", use), (m.n_blocks, w), torch.float32)
            self.buf[("vc", use)] = alloc(("vc", use), (m.n_blocks, w), torch.float32)
            m = self.meta[ks]
            if m.sharded:
                # rank-local compact KV shard of this use, packed in ONE buffer
                # [k_il | v_il | k_cmp | v_cmp] so the exchange sends it whole
                lay = PackedShard(hkv, dh, w, m.n_loc_rows_pad, m.owned.size)
                buf = D.zeros((lay.total,), torch.uint8)
                self.buf[("packed", use)] = buf
                self.buf[("k_loc", use)] = buf[:lay.off_v].view(torch.bfloat16).view(
                    hkv, lay.rows_pad, dh)
                self.buf[("v_loc", use)] = buf[lay.off_v:lay.off_kc].view(torch.bfloat16).view(
                    hkv, lay.rows_pad, dh + ONES_COLS)
                self.buf[("kc_loc", use)] = buf[lay.off_kc:lay.off_vc].view(torch.float32).view(
                    lay.n_blocks, w)
                self.buf[("vc_loc", use)] = buf[lay.off_vc:].view(torch.float32).view(
                    lay.n_blocks, w)
        self._build_kv_jobs()
        self._build_attention_queue()

    def _build_kv_jobs(self):
        """Device array of `lsrm_kv_job`: K and V of every use (one launch)."""
        p = self.params
        jobs, self._job_refs = [], []
        job_stream = []          # KV stream of each job (per-stream launches)
        max_blocks = 0
        for use in self.uses:
            _, ks, _ = USE_GEOM[use]
            m = self.meta[ks]
            if not m.n_loc:
                continue
            Y = self.buf[("Y", ks)]
            for kind, wres in (("k", self.cmp_w[use][0]), ("v", self.cmp_w[use][1])):
                src = Y[:, self.cols[(use, kind)]:]
                w1, b1, w2, b2 = wres
                w1, w2 = w1.to(torch.bfloat16).contiguous(), w2.to(torch.bfloat16).contiguous()
                self._job_refs += [w1, w2]
                if m.sharded:   # rank-local compact shard; means go to the packed buffer
                    il = self.buf[(kind + "_loc", use)]
                    blk, pad, nb = m.loc_off, m.loc_pad_off, m.owned.size
                    mean, cmp_il = self.buf[(kind + "c_loc", use)], None
                else:           # global layout; compressed rows straight to the kernel layout
                    il = self.buf[(kind + "_il", use)]
                    blk, pad, nb = m.kv_off, m.pad_off, m.n_blocks
                    mean, cmp_il = None, self.buf[(kind + "c_il", use)]
                occ = np.diff(m.loc_off_host)
                nsub = (occ + 127) // 128   # 128-token sub-tiles (kv_prep.cu kSub)
                # work code = (block << 12) | 128-token sub-tile (kv_prep.cu kSubBits)
                require(int(nsub.max(initial=0)) <= 1 << 12 and nb < 1 << 19,
                        f"kv_prepare: blocks of up to {128 << 12} tokens and fewer than "
                        f"{1 << 19} occupied blocks are supported (got {int(occ.max(initial=0))} "
                        f"tokens, {nb} blocks)")
                work = np.concatenate([(b << 12) + np.arange(k) for b, k in enumerate(nsub)])
                work_d = D.dev(work.astype(np.int32))
                partial = D.empty((work.size, self.w), torch.float32)
                arrive = D.zeros((max(nb, 1),), torch.int32)
                jobs.append(KvJob(src.data_ptr(), Y.stride(0), blk.data_ptr(), pad.data_ptr(), nb,
                                  int(il.shape[1]), il.data_ptr(),
                                  ONES_COLS if kind == "v" else 0, w1.data_ptr(), b1.data_ptr(),
                                  w2.data_ptr(), b2.data_ptr(), D.ptr(mean), D.ptr(cmp_il),
                                  int(cmp_il.shape[1]) if cmp_il is not None else 0,
                                  work_d.data_ptr(), work.size, partial.data_ptr(),
                                  arrive.data_ptr()))
                self._job_refs += [src, il, blk, pad, mean, cmp_il, work_d, partial, arrive]
                max_blocks = max(max_blocks, int(work.size))
                job_stream.append((ks, int(work.size)))

        def pack(sel):
            js = [j for j, (ks, _) in zip(jobs, job_stream) if ks in sel]
            mb = max([nb for ks, nb in job_stream if ks in sel], default=0)
            raw = b"".join(C.string_at(C.addressof(j), C.sizeof(j)) for j in js)
            return (D.dev(np.frombuffer(raw, dtype=np.uint8).copy()) if js else None, len(js), mb)
        self.kv_jobs, self.n_kv_jobs, self.kv_max_blocks = pack(("x", "y"))
        # per KV stream (sharded engines start a stream's exchanges while the
        # other stream is still being projected)
        self.kv_jobs_of = {s: pack((s,)) for s in ("x", "y")}

    def _build_attention_queue(self):
        """The four uses' attention as heaviest-first item queues. An item is
        (use, tile, kv head); its cost is the keys it streams: compressed rows
        + the padded union of its tokens' selected blocks + (window) its own
        block.

        Tokens are sorted by selection signature before tiling, so a tile's
        tokens share most of their selected blocks. Only the window branch
        ties a tile to one query block, so (SPLIT_SELF_WINDOW) the cmp and sel
        branches of every use run on tiles of the signature order across
        blocks in launch A, and the self uses' window branch runs on block
        tiles in launch B, which adds its gated output to A's."""
        p = self.params
        hkv = p.n_kv_heads
        T = 128 // p.group_size
        queues = {"A": ([], [], []), "B": ([], [], [])}   # uses, costs, codes

        def add(qname, use, tiles, rows_h, cnt_h, perm, n_gates, br_first, accum,
                own_rows=None):
            qs, ks, _ = USE_GEOM[use]
            mq, mk = self.meta[qs], self.meta[ks]
            Y = self.buf[("Y", qs)]
            qcol = self.cols[(use, "q")]
            rows = np.ascontiguousarray(rows_h if perm is None else rows_h[perm])
            cnt = np.ascontiguousarray(cnt_h if perm is None else cnt_h[perm])
            perm_d = D.dev(perm.astype(np.int32)) if perm is not None else None
            rows_d, cnt_d = D.dev(rows), D.dev(cnt)
            own_d = D.dev(own_rows.astype(np.int32)) if own_rows is not None else None
            self._job_refs += [t for t in (perm_d, rows_d, cnt_d, tiles, own_d) if t is not None]
            uses, costs, codes = queues[qname]
            ui = len(uses)
            uses.append(NsaUse(
                Y[:, qcol:].data_ptr(), Y.stride(0), mq.n_loc,
                self.buf[("k_il", use)].data_ptr(), self.buf[("v_il", use)].data_ptr(),
                mk.pad_off.data_ptr(), mk.kv_off.data_ptr(), mk.n_rows_pad,
                self.buf[("kc_il", use)].data_ptr(), self.buf[("vc_il", use)].data_ptr(),
                mk.n_blocks, tiles.data_ptr(), int(tiles.shape[0]), rows_d.data_ptr(),
                cnt_d.data_ptr(), self.kmax[use], Y.data_ptr(), Y.stride(0),
                qcol + self.d, n_gates, self.buf[("merged", use)].data_ptr(), D.ptr(perm_d),
                br_first, accum, D.ptr(own_d)))
            th = D.host(tiles)
            padlen = np.diff(mk.pad_off_host)
            cmp_rows = (mk.n_blocks + ROW_PAD - 1) // ROW_PAD * ROW_PAD
            for t, (first, tc, own, _) in enumerate(th):
                c = int(padlen[own]) if (own >= 0 and n_gates == 3) else 0
                if own_rows is not None:   # the tile's distinct own blocks
                    c += int(padlen[np.unique(own_rows[first:first + tc])].sum())
                if br_first == 0:
                    r = rows[first:first + tc].ravel()
                    r = np.unique(r[r >= 0])
                    c += cmp_rows + int(padlen[r].sum())
                for h in range(hkv):
                    costs.append(c)
                    codes.append((ui << 28) | (t * hkv + h))

        for use in self.uses:
            qs, ks, ng = USE_GEOM[use]
            mq = self.meta[qs]
            rows_h = D.host(self.rows[use])
            cnt_h = D.host(self.count[use])
            blk = np.repeat(np.arange(mq.loc_off_host.size - 1), np.diff(mq.loc_off_host))
            key = np.sort(np.where(rows_h >= 0, rows_h, np.iinfo(np.int32).max), axis=1)
            sig = tuple(key[:, j] for j in reversed(range(key.shape[1])))
            across = not mq.sharded and (SPLIT_SELF_WINDOW if ng == 3 else CROSS_GLOBAL_TILES)
            if ng == 3 and not mq.sharded and PACK_SELF_TAILS and not SELF_GLOBAL_TILES:
                # block tiles (signature order inside each block), except that
                # each block's partial last tile is pooled with the other
                # blocks' into full tiles; the window branch follows each
                # token's own block (per-token own rows)
                order = np.lexsort(sig + (blk,))
                occ = np.diff(mq.loc_off_host).astype(np.int64)
                full = (occ // T) * T
                pos_in_blk = np.arange(order.size) - np.repeat(mq.loc_off_host[:-1], occ)
                is_full = pos_in_blk < np.repeat(full, occ)
                perm = np.concatenate([order[is_full], order[~is_full]])
                n_q = int(rows_h.shape[0])
                first = np.arange(0, n_q, T, dtype=np.int64)
                tiles = D.dev(np.stack([first, np.minimum(T, n_q - first),
                                        np.full_like(first, -1), np.zeros_like(first)],
                                       axis=1).astype(np.int32))
                add("A", use, tiles, rows_h, cnt_h, perm, 3, 0, 0, own_rows=blk[perm])
            elif ng == 3 and not mq.sharded and SELF_GLOBAL_TILES and not SPLIT_SELF_WINDOW:
                # signature order across blocks (own block as the minor key);
                # the window branch follows each token's own block
                perm = np.lexsort((blk,) + sig)
                n_q = int(rows_h.shape[0])
                first = np.arange(0, n_q, T, dtype=np.int64)
                tiles = D.dev(np.stack([first, np.minimum(T, n_q - first),
                                        np.full_like(first, -1), np.zeros_like(first)],
                                       axis=1).astype(np.int32))
                add("A", use, tiles, rows_h, cnt_h, perm, 3, 0, 0, own_rows=blk[perm])
            elif across:
                perm = np.lexsort(sig)
                n_q = int(rows_h.shape[0])
                first = np.arange(0, n_q, T, dtype=np.int64)
                tiles = D.dev(np.stack([first, np.minimum(T, n_q - first),
                                        np.full_like(first, -1), np.zeros_like(first)],
                                       axis=1).astype(np.int32))
                add("A", use, tiles, rows_h, cnt_h, perm, 2, 0, 0)
                if ng == 3:   # window branch on block tiles, added to A's output
                    add("B", use, self.tiles[use], rows_h, cnt_h, None, 3, 2, 1)
            else:
                add("A", use, self.tiles[use], rows_h, cnt_h, np.lexsort(sig + (blk,)), ng, 0, 0)

        self.attn_queues = []
        for qname in ("A", "B"):
            uses, costs, codes = queues[qname]
            if not uses:
                continue
            costs, codes = np.asarray(costs, np.int64), np.asarray(codes, np.int64)
            order = codes[np.lexsort((codes, -costs))].astype(np.int32)
            self.attn_queues.append(((NsaUse * len(uses))(*uses), len(uses), D.dev(order),
                                     D.zeros((1,), torch.int32)))

    def attend_all(self):
        """The four uses' fused attention: persistent launches over LPT queues
        (A: every use's cmp + sel (+ window when not split); B: the self uses'
        window branch, accumulating into A's output)."""
        p = self.params
        for uses, n_uses, order, counter in self.attn_queues:
            call("lsrm_nsa_attention_tc_multi", C.cast(uses, C.c_void_p), n_uses,
                 p.n_q_heads, p.n_kv_heads, p.head_dim, order.data_ptr(),
                 int(order.shape[0]), counter.data_ptr(), D.stream())

    # -- pieces --------------------------------------------------------------
    def project(self, x_loc: torch.Tensor, y_loc: torch.Tensor, streams=("x", "y")):
        """The streams' fused projections (q | gate logits + bias | k | v)
        as ONE grouped tcgen05 GEMM launch."""
        probs = [_ops.gemm_problem(a, self.w_cat[s], self.buf[("Y", s)], bias=self.b_cat[s])
                 for s, a in (("x", x_loc), ("y", y_loc))
                 if s in streams and self.meta[s].n_loc and self.ncol[s]]
        if probs:
            _ops.gemm_tc(probs)

    def prepare_kv(self, stream: str = None):
        """K/V of all four uses in one launch, or of the uses whose KV side is
        `stream` (owned KV blocks when sharded; unsharded engines write the
        global buffers, compressed rows included)."""
        jobs, n, mb = (self.kv_jobs, self.n_kv_jobs, self.kv_max_blocks) if stream is None \
            else self.kv_jobs_of[stream]
        if n:
            p = self.params
            call("lsrm_kv_prepare_jobs", jobs.data_ptr(), n, mb, p.n_kv_heads, p.head_dim,
                 D.stream())

    def finish_kv(self, use: str):
        """Compressed rows (global, canonical order) -> interleaved layout."""
        _, ks, _ = USE_GEOM[use]
        m, p = self.meta[ks], self.params
        st = D.stream()
        for kind in ("k", "v"):
            ones = ONES_COLS if kind == "v" else 0
            cmp, il = self.buf[(kind + "c", use)], self.buf[(kind + "c_il", use)]
            call("lsrm_kv_interleave", 0, cmp.data_ptr(), self.w, m.n_blocks, p.n_kv_heads,
                 p.head_dim, ones, None, None, 0, None, int(il.shape[1]), il.data_ptr(), st)

    def attend(self, use: str):
        qs, ks, ng = USE_GEOM[use]
        mq, mk, p = self.meta[qs], self.meta[ks], self.params
        tiles = self.tiles[use]
        if int(tiles.shape[0]) == 0:
            return
        Y = self.buf[("Y", qs)]
        qcol = self.cols[(use, "q")]
        q = Y[:, qcol:]
        call("lsrm_nsa_attention_tc", q.data_ptr(), Y.stride(0), mq.n_loc, p.n_q_heads,
             p.n_kv_heads, p.head_dim, self.buf[("k_il", use)].data_ptr(),
             self.buf[("v_il", use)].data_ptr(), mk.pad_off.data_ptr(), mk.kv_off.data_ptr(),
             mk.n_rows_pad, self.buf[("kc_il", use)].data_ptr(),
             self.buf[("vc_il", use)].data_ptr(), mk.n_blocks, tiles.data_ptr(),
             int(tiles.shape[0]), self.rows[use].data_ptr(), self.count[use].data_ptr(),
             self.kmax[use], Y.data_ptr(), Y.stride(0), qcol + self.d,
             None, ng, self.buf[("merged", use)].data_ptr(), D.stream())   # bias: in the GEMM

    def output(self, use: str):
        if self.buf[("merged", use)].shape[0]:
            _ops.gemm_tc([_ops.gemm_problem(self.buf[("merged", use)], self.w_o[use],
                                            self.buf[("out", use)])])

    def output_all(self):
        """The four uses' W_o projections as ONE grouped tcgen05 GEMM launch."""
        probs = [_ops.gemm_problem(self.buf[("merged", u)], self.w_o[u], self.buf[("out", u)])
                 for u in self.uses if self.buf[("merged", u)].shape[0]]
        if probs:
            _ops.gemm_tc(probs)

    # -- whole layer ---------------------------------------------------------
    def forward(self, x_loc: torch.Tensor, y_loc: torch.Tensor) -> dict:
        """x_loc [Nv_loc, d], y_loc [Ni_loc, d] bf16 (LN'd; block-major, or the
        rank-local compact order when sharded) -> dict use -> [Nq_loc, d] bf16.
        Output buffers are reused across calls."""
        if self.sharded:
            return self.forward_overlapped(x_loc, y_loc)
        self.project(x_loc, y_loc)
        self.prepare_kv()
        self.attend_all()
        self.output_all()
        return {u: self.buf[("out", u)] for u in self.uses}

    def forward_local(self, x_loc: torch.Tensor, y_loc: torch.Tensor):
        """Sharded phase 1: projections and this rank's KV shards of all uses."""
        self.project(x_loc, y_loc)
        self.prepare_kv()

    def forward_exchange(self) -> dict:
        """Sharded phase 2: launch all four All-gather-KV exchanges, then per
        use wait + place, then attend."""
        require(self.exchange is not None, "sharded engine needs an exchange (seq_parallel)")
        handles = {use: self.exchange(self, use) for use in self.uses}
        return self._finish_exchange(handles)

    def _finish_exchange(self, handles) -> dict:
        for use in self.uses:
            handles[use]()          # wait + place into the canonical layout
            self.finish_kv(use)
        self.attend_all()
        self.output_all()
        return {u: self.buf[("out", u)] for u in self.uses}

    def uses_with_kv(self, stream: str):
        return [u for u in self.uses if USE_GEOM[u][1] == stream]

    def forward_overlapped(self, x_loc: torch.Tensor, y_loc: torch.Tensor) -> dict:
        """Sharded layer with the exchange overlapped: project + prepare the
        x stream's KV, start the exchanges of the uses that read it (v2v,
        i2v; the transport runs them on its own stream), then project +
        prepare the y stream while they are in flight, start v2i / i2i, and
        only then wait, place and attend (`lsrm/seq_parallel.py:298-311`:
        window attention and compression are local; only KV moves)."""
        require(self.exchange is not None, "sharded engine needs an exchange (seq_parallel)")
        handles = {}
        for s in ("x", "y"):
            self.project(x_loc, y_loc, streams=(s,))
            self.prepare_kv(s)
            for use in self.uses_with_kv(s):
                handles[use] = self.exchange(self, use)
        return self._finish_exchange(handles)

    def capture(self, x_bm: torch.Tensor, y_bm: torch.Tensor):
        """Record one layer (all ~30 launches) as a CUDA graph over fixed
        input/output buffers; `replay()` then re-runs it with one launch."""
        require(not self.sharded, "CUDA-graph capture is for the single-GPU engine")
        self._gx, self._gy = x_bm, y_bm
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):          # warm up outside capture
            self.forward(x_bm, y_bm)
        torch.cuda.current_stream().wait_stream(st)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.forward(x_bm, y_bm)
        return self.graph

    def replay(self) -> dict:
        self.graph.replay()
        return {u: self.buf[("out", u)] for u in self.uses}

    # -- accounting ------------------------------------------------------------
    def attention_flops(self) -> dict:
        """Algorithmic attention-core FLOPs per use for this engine's queries
        (SURVEY.md §8d): useful work only (no padding, union inflation or
        masked keys)."""
        p = self.params
        out = {}
        for use in self.uses:
            qs, ks, ng = USE_GEOM[use]
            pk = self.meta[ks].part
            mq = self.meta[qs]
            nq = mq.n_loc
            rows = D.host(self.rows[use])
            cnt = D.host(self.count[use])
            occ = pk.occupancy.astype(np.float64)
            mask = np.arange(rows.shape[1])[None, :] < cnt[:, None]
            L = np.where(mask, occ[np.clip(rows, 0, None)], 0.0).sum(axis=1)
            cmp = 4.0 * nq * p.n_q_heads * p.head_dim * pk.n_occupied
            sel = 4.0 * p.n_q_heads * p.head_dim * L.sum()
            qocc = mq.part.occupancy.astype(np.float64)[mq.owned]
            win = 4.0 * p.n_q_heads * p.head_dim * float((qocc ** 2).sum()) if ng == 3 else 0.0
            out[use] = {"cmp": cmp, "sel": sel, "win": win}
        return out

    def projection_flops(self) -> float:
        return sum(2.0 * self.meta[s].n_loc * self.d * self.ncol[s] for s in ("x", "y")) + \
            sum(2.0 * self.meta[USE_GEOM[u][0]].n_loc * self.d * self.d for u in self.uses)
