"""Spatial block partition and per-block KV compression on the GPU
(drop-in for `lsrm/block_partition.py:22-192`).

Block ids are global and stable: volume (bi*Sb + bj)*Sb + bk, image
view*Sb^2 + bv*Sb + bu; occupied blocks ascend; tokens inside a block ascend.
The partition arrays are small integer metadata: they are returned on the
host (reference API) and mirrored once on the device (`part.dev(...)`).
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev as D
from ._native import call, lib
from .errors import require
from .rng import normal_f32

BLOCK = 8


@dataclass
class BlockPartition:
    modality: str
    block_size: int
    block_grid: tuple
    n_blocks_total: int
    block_of_token: np.ndarray
    occupied_ids: np.ndarray
    block_offsets: np.ndarray
    block_token_ids: np.ndarray
    occupancy: np.ndarray
    block_centers: np.ndarray
    block_views: np.ndarray
    _dev_cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def n_occupied(self) -> int:
        return int(self.occupied_ids.size)

    @property
    def n_tokens(self) -> int:
        return int(self.block_of_token.size)

    def row_of_block(self) -> dict:
        return {int(b): i for i, b in enumerate(self.occupied_ids)}

    def tokens_in_row(self, row: int) -> np.ndarray:
        return self.block_token_ids[self.block_offsets[row]:self.block_offsets[row + 1]]

    def row_of_token(self) -> np.ndarray:
        """Occupied-row index of every token (int32)."""
        if "row_of_token" not in self._dev_cache:
            rows = np.empty(self.n_tokens, np.int32)
            rows[self.block_token_ids] = np.repeat(
                np.arange(self.n_occupied, dtype=np.int32), self.occupancy)
            self._dev_cache["row_of_token"] = rows
        return self._dev_cache["row_of_token"]

    def dev(self, name: str) -> torch.Tensor:
        """Device mirror of a metadata array (cached)."""
        key = ("dev", name, torch.cuda.current_device())
        if key not in self._dev_cache:
            arr = self.row_of_token() if name == "row_of_token" else getattr(self, name)
            self._dev_cache[key] = D.dev(np.ascontiguousarray(arr))
        return self._dev_cache[key]


def partition(tokens, block_size: int = BLOCK) -> BlockPartition:
    """Group tokens by floor-divided coords; blocks never span views
    (`block_partition.py:54-105`)."""
    if tokens.modality == "volume":
        side = tokens.grid_res[0]
        require(side % block_size == 0, f"grid side {side} not divisible by block {block_size}")
        sb = side // block_size
        g = (side, side, side)
        grid, total, mod = (sb, sb, sb), sb ** 3, 0
    else:
        n_views, rows_f, _ = tokens.grid_res
        require(rows_f % block_size == 0,
                f"grid side {rows_f} not divisible by block {block_size}")
        sb = rows_f // block_size
        g = (n_views, rows_f, rows_f)
        grid, total, mod = (n_views, sb, sb), n_views * sb * sb, 1
    n = tokens.count
    coords = D.dev(tokens.coords, torch.int64)
    bot = D.empty((n,), torch.int64)
    tok = D.empty((n,), torch.int64)
    occ_ids = D.empty((total,), torch.int64)
    offs = D.empty((total + 1,), torch.int64)
    occ = D.empty((total,), torch.int64)
    ncols = 3 if mod == 0 else 2
    centers = D.empty((total, ncols), torch.float64)
    views = D.empty((total,), torch.int64)
    ws_bytes = lib().lsrm_partition_workspace(n, total)
    ws = D.empty((ws_bytes,), torch.uint8)
    b_out = np.zeros(1, np.int64)
    call("lsrm_partition", mod, coords.data_ptr(), n, g[0], g[1], g[2], block_size,
         bot.data_ptr(), tok.data_ptr(), occ_ids.data_ptr(), offs.data_ptr(), occ.data_ptr(),
         centers.data_ptr(), views.data_ptr() if mod else None, b_out.ctypes.data,
         ws.data_ptr(), ws_bytes, D.stream())
    B = int(b_out[0])
    part = BlockPartition(
        modality=tokens.modality, block_size=block_size, block_grid=grid,
        n_blocks_total=total, block_of_token=D.host(bot), occupied_ids=D.host(occ_ids[:B]),
        block_offsets=D.host(offs[:B + 1]), block_token_ids=D.host(tok),
        occupancy=D.host(occ[:B]), block_centers=D.host(centers[:B]),
        block_views=D.host(views[:B]) if mod else np.zeros(0, np.int64))
    dv = torch.cuda.current_device()
    for name, t in (("block_of_token", bot), ("block_token_ids", tok),
                    ("occupied_ids", occ_ids[:B]), ("block_offsets", offs[:B + 1]),
                    ("occupancy", occ[:B]), ("block_centers", centers[:B].contiguous())):
        part._dev_cache[("dev", name, dv)] = t
    return part


# ---------------------------------------------------------------------------
# compressed KV


@dataclass
class ResBlockParams:
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray


@dataclass
class CompressWeights:
    for_k: ResBlockParams
    for_v: ResBlockParams


def init_res_block(seed, width, *tags, scale=0.02) -> ResBlockParams:
    return ResBlockParams(
        w1=normal_f32(seed, (width, width), scale, *tags, "w1"),
        b1=np.zeros(width, np.float32),
        w2=normal_f32(seed, (width, width), scale, *tags, "w2"),
        b2=np.zeros(width, np.float32))


def init_compress_weights(seed, width, *tags) -> CompressWeights:
    return CompressWeights(init_res_block(seed, width, *tags, "cmp_k"),
                           init_res_block(seed, width, *tags, "cmp_v"))


def _dev_res(p: ResBlockParams):
    return [D.weight(a) for a in (p.w1, p.b1, p.w2, p.b2)]


def compress_rows(x, ld, n, width, params, part: BlockPartition, src_bf16=False, out=None,
                  scratch=None):
    """Device-level compression of one [n, width] row set (strided view)."""
    w1, b1, w2, b2 = params if isinstance(params, (list, tuple)) else _dev_res(params)
    B = part.n_occupied
    out = D.empty((B, width), torch.float32) if out is None else out
    scratch = D.empty((n, width), torch.float32) if scratch is None else scratch
    call("lsrm_compress_block", int(src_bf16), x.data_ptr(), ld, n, width, w1.data_ptr(),
         b1.data_ptr(), w2.data_ptr(), b2.data_ptr(), part.dev("block_token_ids").data_ptr(),
         part.dev("block_offsets").data_ptr(), B, out.data_ptr(), scratch.data_ptr(),
         D.stream())
    return out


def res_block(x, p: ResBlockParams):
    """x + W2·gelu(W1·x + b1) + b2 per row, f64 inside, f32 out
    (`block_partition.py:112-124`).  x [N, w] -> [N, w]."""
    on_dev = D.is_device(x)
    xd = D.dev(x, torch.float32)
    n, width = (int(s) for s in xd.shape)
    if n == 0:
        return xd.clone() if on_dev else np.zeros((0, width), np.float32)
    scratch = D.empty((n, width), torch.float32)
    one = D.empty((1, width), torch.float32)
    ids = torch.arange(n, dtype=torch.int64, device=xd.device)
    offs = D.dev(np.array([0, n], np.int64))
    w1, b1, w2, b2 = _dev_res(p)
    call("lsrm_compress_block", 0, xd.data_ptr(), width, n, width, w1.data_ptr(), b1.data_ptr(),
         w2.data_ptr(), b2.data_ptr(), ids.data_ptr(), offs.data_ptr(), 1, one.data_ptr(),
         scratch.data_ptr(), D.stream())
    return scratch if on_dev else D.host(scratch)


def compress_block_kv(k, v, part: BlockPartition, w: CompressWeights):
    """Per-token ResBlock then the in-block mean in ascending token order
    (`block_partition.py:147-167`).  k, v [N, h_kv, d_h] -> [B, h_kv, d_h]."""
    on_dev = D.is_device(k)
    n, h_kv, d_h = (int(s) for s in k.shape)
    require(tuple(v.shape) == tuple(k.shape), "k and v shapes must match")
    require(n == part.n_tokens, "partition does not index these tokens")
    if n == 0:
        z = np.zeros((0, h_kv, d_h), np.float32)
        return (D.dev(z), D.dev(z)) if on_dev else (z, z.copy())
    width = h_kv * d_h
    outs = []
    for t, p in ((k, w.for_k), (v, w.for_v)):
        x = D.dev(t, torch.float32).reshape(n, width)
        o = compress_rows(x, width, n, width, p, part).reshape(-1, h_kv, d_h)
        outs.append(o if on_dev else D.host(o))
    return outs[0], outs[1]


def occupancy_stats(part: BlockPartition) -> dict:
    """Host-side summary (`block_partition.py:170-192`)."""
    occ = part.occupancy
    if occ.size == 0:
        return {"total_tokens": 0, "occupied_blocks": 0, "min": 0, "max": 0, "mean": 0.0,
                "max_over_mean": 0.0, "gini": 0.0, "histogram": {}}
    mean = float(occ.mean())
    s = np.sort(occ).astype(np.float64)
    n = occ.size
    gini = float(2.0 * np.sum(np.arange(1, n + 1) * s) / (n * s.sum()) - (n + 1.0) / n)
    vals, freq = np.unique(occ, return_counts=True)
    return {"total_tokens": int(occ.sum()), "occupied_blocks": int(n), "min": int(occ.min()),
            "max": int(occ.max()), "mean": mean, "max_over_mean": float(occ.max() / mean),
            "gini": gini, "histogram": {int(a): int(b) for a, b in zip(vals, freq)}}
