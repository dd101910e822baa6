"""Spatial block partition and per-block KV compression (TEST INFRASTRUCTURE ONLY).

Restates `lsrm/block_partition.py:22-167`.
"""

from dataclasses import dataclass

import numpy as np

from .numerics import ACC, DTYPE, affine, gelu

BLOCK = 8


@dataclass
class Partition:
    """Fields mirror `BlockPartition` (`block_partition.py:22-51`)."""
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

    @property
    def n_occupied(self):
        return int(self.occupied_ids.size)

    @property
    def n_tokens(self):
        return int(self.block_of_token.size)

    def row_of_block(self):
        return {int(b): r for r, b in enumerate(self.occupied_ids)}

    def tokens_in_row(self, r):
        return self.block_token_ids[self.block_offsets[r]:self.block_offsets[r + 1]]


def partition_tokens(modality, coords, grid_res, block_size=BLOCK):
    """Global block id per token, stable (block id, token id) order, occupied
    ids ascending, offsets, occupancy and block centers
    (`block_partition.py:54-105`).  coords [N,3] int: (i,j,k) for volume,
    (view,u,v) for image."""
    coords = np.asarray(coords, np.int64)
    n = coords.shape[0]
    if modality == "volume":
        side = grid_res[0]
        sb = side // block_size
        b = coords // block_size
        bid = (b[:, 0] * sb + b[:, 1]) * sb + b[:, 2]
        grid, total = (sb, sb, sb), sb ** 3
    else:
        nv, side, _ = grid_res
        sb = side // block_size
        bid = (coords[:, 0] * sb * sb + (coords[:, 2] // block_size) * sb
               + coords[:, 1] // block_size)
        grid, total = (nv, sb, sb), nv * sb * sb
    order = np.argsort(bid, kind="stable")          # == lexsort((arange, bid))
    occ_ids, starts, counts = np.unique(bid[order], return_index=True,
                                        return_counts=True)
    offsets = np.append(starts, n).astype(np.int64)
    half = block_size / 2.0
    if modality == "volume":
        bi, bj, bk = occ_ids // (sb * sb), (occ_ids // sb) % sb, occ_ids % sb
        centers = np.stack([(block_size * bi + half) / side,
                            (block_size * bj + half) / side,
                            (block_size * bk + half) / side], axis=-1)
        views = np.zeros(0, np.int64)
    else:
        views = occ_ids // (sb * sb)
        rem = occ_ids % (sb * sb)
        centers = np.stack([block_size * (rem % sb) + half,
                            block_size * (rem // sb) + half], axis=-1)
    return Partition(modality, block_size, grid, total, bid.astype(np.int64),
                     occ_ids.astype(np.int64), offsets, order.astype(np.int64),
                     counts.astype(np.int64), centers.reshape(-1, 3 if modality == "volume" else 2),
                     views.astype(np.int64))


def res_block(x, w1, b1, w2, b2):
    """x + affine(gelu(affine(x, w1, b1)), w2, b2) (`block_partition.py:141-144`)."""
    h = affine(gelu(affine(x, w1, b1)), w2, b2)
    return (np.asarray(x, ACC) + h.astype(ACC)).astype(DTYPE)


def compress_block_kv(k, v, part: Partition, cw):
    """Residual transform per token then the per-block mean in ascending token
    order (`block_partition.py:147-167`).  cw = ((w1,b1,w2,b2) for k,
    (w1,b1,w2,b2) for v)."""
    n, h, dh = k.shape
    if n == 0:
        z = np.zeros((0, h, dh), DTYPE)
        return z, z.copy()
    outs = []
    for t, p in ((k, cw[0]), (v, cw[1])):
        r = res_block(t.reshape(n, h * dh), *p).astype(ACC)[part.block_token_ids]
        # sequential sum inside each block, in ascending token order
        s = np.add.reduceat(r, part.block_offsets[:-1], axis=0)
        outs.append((s / part.occupancy[:, None]).astype(DTYPE).reshape(-1, h, dh))
    return outs[0], outs[1]
