"""Foreground pruning, informative-voxel mask and fine-token compaction
(TEST INFRASTRUCTURE ONLY).

Restates `lsrm/tokenizer.py:180-313` and the analytic SDFs it consumes
(`lsrm/camera_geometry.py:190-205`).  SDF nodes are dicts:
{"kind": "sphere", "center", "radius"} | {"kind": "box", "center",
"half_sizes"} | {"kind": "union", "parts": [...]} (the scene-json schema,
`camera_geometry.py:352-361`).
"""

from dataclasses import dataclass

import numpy as np

from .numerics import DTYPE


@dataclass
class TokenSet:
    modality: str
    features: np.ndarray
    coords: np.ndarray
    grid_res: tuple

    @property
    def count(self):
        return int(self.features.shape[0])


def _norm3(a):
    # np.linalg.norm over a length-3 axis: sqrt((a0^2 + a1^2) + a2^2)
    return np.sqrt(np.add.reduce(a * a, axis=-1))


def eval_sdf(node, pts):
    """`camera_geometry.py:190-205`."""
    kind = node["kind"]
    if kind == "sphere":
        return _norm3(pts - np.asarray(node["center"], np.float64)) - float(node["radius"])
    if kind == "box":
        q = np.abs(pts - np.asarray(node["center"], np.float64)) \
            - np.asarray(node["half_sizes"], np.float64)
        return _norm3(np.maximum(q, 0.0)) + np.minimum(q.max(axis=-1), 0.0)
    if kind == "union":
        return np.stack([eval_sdf(p, pts) for p in node["parts"]]).min(axis=0)
    raise ValueError(kind)


def foreground_patch_mask(alpha, patch=8):
    """any(alpha > 0.5) per patch (`tokenizer.py:200-208`)."""
    h, w = alpha.shape
    return (np.asarray(alpha).reshape(h // patch, patch, w // patch, patch)
            > 0.5).any(axis=(1, 3))


def informative_voxel_mask(sdf, s_vol, tau=None, t_side=4):
    """Eq. 11 over the t_side^3 cell-center samples of each voxel
    (`tokenizer.py:211-239`)."""
    tau = 1.0 / s_vol if tau is None else tau
    fine = t_side * s_vol
    line = (np.arange(fine) + 0.5) / fine
    yy, zz = np.meshgrid(line, line, indexing="ij")
    mask = np.zeros((s_vol,) * 3, bool)
    for i in range(s_vol):
        pts = np.empty((t_side, fine, fine, 3))
        pts[..., 0] = line[t_side * i:t_side * (i + 1)][:, None, None]
        pts[..., 1] = yy[None]
        pts[..., 2] = zz[None]
        s = eval_sdf(sdf, pts.reshape(-1, 3)).reshape(
            t_side, s_vol, t_side, s_vol, t_side)
        ax = (0, 2, 4)
        mask[i] = (np.abs(s).min(axis=ax) <= tau) | \
            (s.min(axis=ax) * s.max(axis=ax) <= 0.0)
    return mask


def factorized_pos_embed(tables, coords):
    """f32(((0 + t0[c0]) + t1[c1]) [+ t2[c2]]) summed in f64 (`tokenizer.py:180-193`)."""
    coords = np.asarray(coords, np.int64)
    acc = np.zeros((coords.shape[0], tables[0].shape[1]))
    for ax, t in enumerate(tables):
        acc += t.astype(np.float64)[coords[:, ax]]
    return acc.astype(DTYPE)


def upsample_select_tokens(x_d, y_d, vol_mask, img_mask, pe_vol, pe_img,
                           factor_vol=6, factor_img=3):
    """Compaction of mask-true fine cells with parent replication plus the
    fine positional embedding (`tokenizer.py:255-313`).  Volume order is
    lexicographic (i,j,k); image order is view-major raster (row outer),
    stored as (view, u=col, v=row)."""
    s = vol_mask.shape[0]
    sc = s // factor_vol
    vc = np.argwhere(vol_mask)
    par = vc // factor_vol
    pidx = (par[:, 0] * sc + par[:, 1]) * sc + par[:, 2]
    vfeat = (x_d[pidx].astype(np.float64)
             + factorized_pos_embed(pe_vol, vc).astype(np.float64)).astype(DTYPE)
    x_up = TokenSet("volume", vfeat, vc.astype(np.int64), (s, s, s))

    nv, rows, _ = img_mask.shape
    sic = rows // factor_img
    yv = y_d.reshape(nv, sic, sic, -1)
    feats, coords = [], []
    for view in range(nv):
        rc = np.argwhere(img_mask[view])
        if rc.size == 0:
            continue
        p = rc // factor_img
        f = (yv[view, p[:, 0], p[:, 1]].astype(np.float64)
             + factorized_pos_embed(pe_img, rc[:, ::-1]).astype(np.float64))
        feats.append(f.astype(DTYPE))
        coords.append(np.column_stack([np.full(len(rc), view), rc[:, 1], rc[:, 0]]))
    if feats:
        yf, ycrd = np.concatenate(feats), np.concatenate(coords).astype(np.int64)
    else:
        yf, ycrd = np.zeros((0, x_d.shape[1]), DTYPE), np.zeros((0, 3), np.int64)
    return x_up, TokenSet("image", yf, ycrd, (nv, rows, rows))
