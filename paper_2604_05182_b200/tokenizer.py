"""Foreground pruning, informative-voxel mask and fine-token compaction on the
GPU (drop-in for `lsrm/tokenizer.py:32-66,180-313`).

Inputs/outputs follow the reference API (NumPy in -> NumPy out); passing CUDA
tensors keeps everything device-resident (CUDA in -> CUDA out).  Masks and
compaction are bit-exact with the reference (integer order, exact f64 compares,
same f64 add order for features); see kernels in csrc/tokens.cu.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev as D
from ._native import call, lib
from .sdf import DeviceField, sdf_primitives  # noqa: F401 (re-export)
from .sdf import ptr as sdf_ptr
from .errors import ConfigurationError, require

PATCH = 8


@dataclass
class TokenSet:
    """`lsrm/tokenizer.py:32-66`.  features [N,d] f32, coords [N,3] int64:
    (i,j,k) volume or (view,u,v) image; NumPy or CUDA tensors."""
    modality: str
    features: object
    coords: object
    grid_res: tuple
    validate: bool = True

    def __post_init__(self):
        require(self.modality in ("volume", "image"), f"bad modality {self.modality!r}")
        if not D.is_device(self.features):
            self.features = np.asarray(self.features, dtype=np.float32)
        if not D.is_device(self.coords):
            self.coords = np.asarray(self.coords, dtype=np.int64)
        require(self.features.ndim == 2, "features must be [N, d]")
        require(tuple(self.coords.shape) == (self.features.shape[0], 3), "coords must be [N, 3]")
        self.grid_res = tuple(int(g) for g in self.grid_res)
        if self.validate and self.coords.shape[0] and not D.is_device(self.coords):
            c = self.coords
            require(c.min() >= 0, "negative token coord")
            for ax in range(3):
                require(int(c[:, ax].max()) < self.grid_res[ax],
                        f"token coord axis {ax} exceeds grid {self.grid_res}")
            keys = (c[:, 0] * self.grid_res[1] + c[:, 1]) * self.grid_res[2] + c[:, 2]
            require(np.unique(keys).size == keys.size, "duplicate token coords")

    @property
    def count(self) -> int:
        return int(self.features.shape[0])

    @property
    def dim(self) -> int:
        return int(self.features.shape[1])


@dataclass
class PosEmbed:
    """Per-axis 1-D tables summed per token (`tokenizer.py:157-177`)."""
    tables: tuple

    @property
    def side(self):
        return int(self.tables[0].shape[0])

    @property
    def dim(self):
        return int(self.tables[0].shape[1])


def init_pos_embed(seed, n_axes, side, d, scale=0.02, label="pos"):
    from .rng import normal_f32
    return PosEmbed(tuple(normal_f32(seed, (side, d), scale, label, f"axis{ax}")
                          for ax in range(n_axes)))


def _ret(t, like_device):
    return t if like_device else D.host(t)


def foreground_patch_mask(alpha, patch: int = PATCH):
    """[H,W] (or [V,H,W]) alpha -> bool patch mask: any(alpha > 0.5)
    (`tokenizer.py:200-208`)."""
    on_dev = D.is_device(alpha)
    require(alpha.ndim in (2, 3), "alpha must be [H, W]")
    a = D.dev(alpha, torch.float32)
    squeeze = a.ndim == 2
    if squeeze:
        a = a[None]
    v, h, w = a.shape
    if h % patch or w % patch:
        raise ConfigurationError(f"alpha {h}x{w} not divisible by patch {patch}")
    m = D.empty((v, h // patch, w // patch), torch.uint8)
    call("lsrm_foreground_mask", a.data_ptr(), v, h, w, patch, m.data_ptr(), D.stream())
    m = m.bool()
    if squeeze:
        m = m[0]
    return _ret(m, on_dev)


def informative_voxel_mask(field, s_vol: int, tau: float = None, t_side: int = 4,
                           as_device: bool = False):
    """[S,S,S] bool, Eq. 11 over t_side^3 cell-center samples per voxel
    (`tokenizer.py:211-239`).  `field`: the analytic scene (reference
    SdfField or scene-json dict), the decoded coarse volume
    (`sdf.decoded_sdf_field`, evaluated in-kernel), or any callable field
    (`callable_field(fn)`: fn is called on the GPU-generated sample points of
    each x-slab batch, in the reference's layout; the reduction runs on the
    GPU)."""
    require(s_vol >= 1 and t_side >= 1, "bad mask resolution")
    if tau is None:
        tau = 1.0 / s_vol
    require(tau > 0, "tau must be positive")
    f = DeviceField(field)
    m = D.zeros((s_vol, s_vol, s_vol), torch.uint8)
    st = D.stream()
    if not f.opaque:
        call("lsrm_voxel_mask_field", sdf_ptr(f.desc), s_vol, float(tau), t_side, 0, s_vol,
             m.data_ptr(), st)
        return _ret(m.bool(), as_device)
    fine = t_side * s_vol
    per_slab = t_side * fine * fine
    step = max(1, (1 << 22) // per_slab)
    for i0 in range(0, s_vol, step):
        i1 = min(s_vol, i0 + step)
        pts = D.empty(((i1 - i0) * per_slab, 3), torch.float64)
        call("lsrm_voxel_sample_points", s_vol, t_side, i0, i1, pts.data_ptr(), st)
        vals = f.eval_host(pts)
        call("lsrm_voxel_mask_field", sdf_ptr(f.values_desc(vals)), s_vol, float(tau), t_side,
             i0, i1, m.data_ptr(), st)
    return _ret(m.bool(), as_device)


def _compact_scan(kind, mask_u8, n_views, s_fine, factor):
    """Mask scan: cell list of the set cells in the returned workspace and
    their count (one host readback: the output size is data-dependent)."""
    n_cells = mask_u8.numel()
    ws_bytes = lib().lsrm_compact_workspace(n_cells)
    ws = D.empty((ws_bytes,), torch.uint8)
    n_out = np.zeros(1, np.int64)
    nptr = n_out.ctypes.data
    st = D.stream()
    if kind == "volume":
        call("lsrm_compact_volume", mask_u8.data_ptr(), s_fine, factor, None, 0, None, None,
             None, None, None, 0, nptr, ws.data_ptr(), ws_bytes, st)
    else:
        call("lsrm_compact_image", mask_u8.data_ptr(), n_views, s_fine, factor, None, 0, None,
             None, None, None, 0, nptr, ws.data_ptr(), ws_bytes, st)
    return ws, n_cells, int(n_out[0])


def _compact_rows(kind, ws, n_cells, n, parents, d, tables, n_views, s_fine, factor,
                  coords, feats):
    """Coords + features of the n scanned cells (no rescan, no host sync)."""
    if n:
        tp = [t.data_ptr() for t in tables] + [None] * (3 - len(tables))
        call("lsrm_compact_rows", 0 if kind == "volume" else 1, ws.data_ptr(), n_cells, n,
             n_views, s_fine, factor, parents.data_ptr(), d, tp[0], tp[1], tp[2],
             coords.data_ptr(), feats.data_ptr(), D.stream())


def _compact(kind, mask_u8, parents, d, tables, n_views, s_fine, factor):
    ws, n_cells, n = _compact_scan(kind, mask_u8, n_views, s_fine, factor)
    coords = D.empty((n, 3), torch.int64)
    feats = D.empty((n, d), torch.float32)
    _compact_rows(kind, ws, n_cells, n, parents, d, tables, n_views, s_fine, factor, coords,
                  feats)
    return coords, feats


def upsample_select_tokens(x_d, y_d, vol_mask, img_mask, pe_fine_vol, pe_fine_img,
                           factor_vol: int = 6, factor_img: int = 3):
    """Fine active tokens: mask-true cells take their parent coarse feature
    plus the fine positional embedding (`tokenizer.py:255-313`).  Volume in
    lexicographic (i,j,k) order; image view-major raster, coords (view,u,v)."""
    on_dev = D.is_device(x_d)
    s_fine = int(vol_mask.shape[0])
    require(tuple(vol_mask.shape) == (s_fine,) * 3, "vol mask not cubic")
    require(s_fine % factor_vol == 0, "volume mask not divisible by factor")
    sc = s_fine // factor_vol
    require(x_d.shape[0] == sc ** 3, f"x_d has {x_d.shape[0]} tokens, expected {sc ** 3}")
    require(pe_fine_vol.side == s_fine, "fine volume pos-embed side mismatch")
    n_views, rows_f, cols_f = (int(s) for s in img_mask.shape)
    require(rows_f == cols_f, "image mask must be square")
    require(rows_f % factor_img == 0, "image mask not divisible by factor")
    sic = rows_f // factor_img
    require(y_d.shape[0] == n_views * sic ** 2,
            f"y_d has {y_d.shape[0]} tokens, expected {n_views * sic ** 2}")
    require(pe_fine_img.side == rows_f, "fine image pos-embed side mismatch")
    d = int(x_d.shape[1])
    xd = D.dev(x_d, torch.float32)
    yd = D.dev(y_d, torch.float32)
    vm = D.dev(vol_mask).to(torch.uint8).contiguous()
    im = D.dev(img_mask).to(torch.uint8).contiguous()
    # positional tables are weights: uploaded once per array (device cache)
    tv = [D.dev(t, torch.float32) if D.is_device(t) else D.weight(t) for t in pe_fine_vol.tables]
    ti = [D.dev(t, torch.float32) if D.is_device(t) else D.weight(t) for t in pe_fine_img.tables]
    vc, vf = _compact("volume", vm, xd, d, tv, 1, s_fine, factor_vol)
    ic, ifeat = _compact("image", im, yd, d, ti, n_views, rows_f, factor_img)
    if not on_dev:
        vc, vf, ic, ifeat = (D.host(t) for t in (vc, vf, ic, ifeat))
    x_up = TokenSet("volume", vf, vc, (s_fine,) * 3, validate=False)
    y_up = TokenSet("image", ifeat, ic, (n_views, rows_f, cols_f), validate=False)
    return x_up, y_up
