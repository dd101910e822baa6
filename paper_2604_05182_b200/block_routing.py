"""3D-aware spatial routing on the GPU (drop-in for `lsrm/block_routing.py`).

Volume KV blocks are ranked by center distance; image KV blocks by the
two-stage rule (per-view 2D shortlist of b_i blocks, pooled, ranked by min 3D
distance to the block's token points).  The kernels (csrc/routing.cu) are f64
with no FMA contraction and exact lexicographic (distance, row) selection, so
the lists equal the reference's bit for bit, tie order included.
"""

import struct
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _dev as D
from . import _ops
from ._native import call
from .block_partition import BlockPartition
from .errors import require
from .nsa_attention import Selection, write_selection

QUERY_CHUNK = 512
PLAN_TABLE_ORDER = ("v2v", "v2i", "i2v", "i2i")


@dataclass
class RoutingBudgets:
    b_i: int = 16
    b_v2v: int = 8
    b_v2i: int = 8
    b_i2v: int = 8
    b_i2i: int = 8


@dataclass
class TokenCoords3D:
    points: np.ndarray
    miss: np.ndarray

    def __post_init__(self):
        self.points = np.asarray(self.points, dtype=np.float64)
        self.miss = np.asarray(self.miss, dtype=bool)
        require(self.points.ndim == 2 and self.points.shape[1] == 3, "token points must be [N,3]")
        require(self.miss.shape == (self.points.shape[0],), "miss flags must be [N]")
        if self.points.size:
            require(float(self.points.min()) >= 0.0 and float(self.points.max()) <= 1.0,
                    "token points must lie in the unit cube")


@dataclass
class RoutingPlan:
    tables: dict
    budgets: RoutingBudgets
    fallback_queries: dict = dc_field(default_factory=dict)
    device_rows: dict = dc_field(default_factory=dict, repr=False)   # name -> (rows, count)


def volume_token_coords(tokens) -> TokenCoords3D:
    """Voxel centers (c + 0.5) / S (`block_routing.py:67-70`)."""
    side = tokens.grid_res[0]
    c = tokens.coords if not D.is_device(tokens.coords) else D.host(tokens.coords)
    return TokenCoords3D((c.astype(np.float64) + 0.5) / side, np.zeros(tokens.count, bool))


LAPLACE_BETA = 0.02   # camera_geometry.py:19


def image_token_coords(tokens, cameras, field, beta: float = LAPLACE_BETA) -> TokenCoords3D:
    """Surface point of each image token's patch-center ray
    (`block_routing.py:73-108`): 128-sample Laplace opacity march
    (`camera_geometry.py:264-302`) on the GPU, f64, warp per ray; rays with
    no opacity peak fall back to their cube-entry point, rays missing the cube
    to the clamped closest approach to the cube center, both flagged in
    `miss`.  `field` as in `informative_voxel_mask`: analytic, the decoded
    coarse volume (in-kernel), or any callable field (called on the
    GPU-generated sample points of the rays that enter the cube)."""
    from .sdf import DeviceField, ptr as sdf_ptr
    n_views, rows_f, _ = tokens.grid_res
    require(len(cameras) == n_views, "camera count != view count")
    require(beta > 0, "beta must be positive")
    wh = []
    for cam in cameras:
        size = getattr(cam, "image_size", None)
        if size is None and isinstance(cam, (tuple, list)) and len(cam) > 3:
            size = cam[3]
        wh.append(size if size is not None else (8 * rows_f, 8 * rows_f))
    n = tokens.count
    coords = D.dev(tokens.coords, torch.int64)
    cams = D.dev(pack_cameras(cameras))
    whd = D.dev(np.asarray(wh, np.int32).reshape(-1, 2))
    f = DeviceField(field)
    pts = D.empty((max(n, 1), 3), torch.float64)
    miss = D.empty((max(n, 1),), torch.uint8)
    st = D.stream()
    desc = f.desc
    if f.opaque and n:
        samples = D.empty((n * 128, 3), torch.float64)
        span = D.empty((n,), torch.uint8)
        call("lsrm_ray_sample_points", coords.data_ptr(), n, cams.data_ptr(), whd.data_ptr(),
             n_views, rows_f, samples.data_ptr(), span.data_ptr(), st)
        live = span.bool().repeat_interleave(128)
        vals = torch.zeros((n * 128,), dtype=torch.float64, device=samples.device)
        if bool(live.any()):
            vals[live] = f.eval_host(samples[live])
        desc = f.values_desc(vals)
    if n:
        call("lsrm_image_token_points_field", coords.data_ptr(), n, cams.data_ptr(),
             whd.data_ptr(), n_views, rows_f, sdf_ptr(desc), float(beta), pts.data_ptr(),
             miss.data_ptr(), st)
    return TokenCoords3D(D.host(pts)[:n], D.host(miss)[:n].astype(bool))


def pack_cameras(cameras) -> np.ndarray:
    """[V, 21] f64 rows K(9) R(9) t(3) from reference Camera objects or
    (K, R, t) tuples."""
    rows = []
    for cam in cameras:
        if isinstance(cam, (tuple, list)):
            K, R, t = cam[:3]
        else:
            K, R, t = cam.intrinsics, cam.rotation, cam.translation
        rows.append(np.concatenate([np.asarray(K, np.float64).ravel(),
                                    np.asarray(R, np.float64).ravel(),
                                    np.asarray(t, np.float64).ravel()]))
    return np.asarray(rows, np.float64).reshape(-1, 21)


def _rows_to_selection(rows, count, part: BlockPartition) -> Selection:
    r = D.host(rows)
    c = D.host(count)
    ids = part.occupied_ids
    return Selection([ids[r[i, :c[i]]] for i in range(r.shape[0])])


def route_volume_rows(points, part: BlockPartition, budget: int):
    """Device result: (rows [nq, budget] int32, count [nq] int32)."""
    pts = D.dev(points, torch.float64)
    nq = int(pts.shape[0])
    rows = D.empty((nq, max(budget, 1)), torch.int32)
    count = D.zeros((nq,), torch.int32)
    if nq and part.n_occupied:
        call("lsrm_route_volume", pts.data_ptr(), nq, part.dev("block_centers").data_ptr(),
             part.n_occupied, budget, rows.data_ptr(), count.data_ptr(), D.stream())
    else:
        rows.fill_(-1)
    return rows, count


class ImageSide:
    """Per-(image partition, token points, cameras) device state of the image
    router: block-major token points SoA [3, Ni], per-block bounding boxes
    (`lsrm_block_bounds`), packed cameras and per-view row ranges.  Built once
    and shared by every query set routed against the same image side (v2i and
    i2i of a plan)."""

    def __init__(self, part: BlockPartition, token_points, cameras):
        tp = token_points.points if isinstance(token_points, TokenCoords3D) else token_points
        cams = pack_cameras(cameras)
        self.n_views = int(cams.shape[0])
        vrs = np.searchsorted(part.block_views, np.arange(self.n_views + 1)).astype(np.int64)
        self.max_view_rows = int(np.diff(vrs).max()) if vrs.size > 1 else 0
        self.cams, self.vrs = D.dev(cams), D.dev(vrs)
        # block-major token points, SoA [3, Ni] (coalesced loads in the kernel)
        self.tp = _ops.gather_rows(D.dev(tp, torch.float64),
                                   part.dev("block_token_ids")).t().contiguous()
        self.bounds = D.empty((part.n_occupied, 6), torch.float64)
        if part.n_occupied:
            call("lsrm_block_bounds", self.tp.data_ptr(), int(self.tp.shape[1]),
                 part.dev("block_offsets").data_ptr(), part.n_occupied,
                 self.bounds.data_ptr(), D.stream())


def route_image_rows(points, cameras, part: BlockPartition, token_points, b_i: int,
                     budget: int, side: ImageSide = None):
    pts = D.dev(points, torch.float64)
    nq = int(pts.shape[0])
    rows = D.empty((nq, max(budget, 1)), torch.int32)
    count = D.zeros((nq,), torch.int32)
    if nq == 0 or part.n_occupied == 0:
        rows.fill_(-1)
        return rows, count
    side = side or ImageSide(part, token_points, cameras)
    call("lsrm_route_image", pts.data_ptr(), nq, side.cams.data_ptr(), side.n_views,
         side.vrs.data_ptr(), part.dev("block_centers").data_ptr(), part.n_occupied,
         side.tp.data_ptr(), side.bounds.data_ptr(), part.dev("block_offsets").data_ptr(), b_i,
         budget, side.max_view_rows, rows.data_ptr(), count.data_ptr(), D.stream())
    return rows, count


def _route_points_to_volume(points, part: BlockPartition, budget: int) -> Selection:
    """`block_routing.py:134-143`."""
    return _rows_to_selection(*route_volume_rows(points, part, budget), part)


def route_to_volume_blocks(p, vol_part: BlockPartition, budget: int) -> np.ndarray:
    """`block_routing.py:124-131`."""
    return _route_points_to_volume(np.asarray(p, np.float64).reshape(1, 3), vol_part,
                                   budget).lists[0]


def _route_points_to_image(points, cameras, img_part: BlockPartition, img_coords3d,
                           b_i: int, budget: int) -> Selection:
    """`block_routing.py:183-220`."""
    return _rows_to_selection(*route_image_rows(points, cameras, img_part, img_coords3d,
                                                b_i, budget), img_part)


def route_to_image_blocks(p, cameras, img_part, img_coords3d, b_i, budget) -> np.ndarray:
    """`block_routing.py:223-230`."""
    return _route_points_to_image(np.asarray(p, np.float64).reshape(1, 3), cameras,
                                  img_part, img_coords3d, b_i, budget).lists[0]


def build_routing_plan(vol_coords, img_coords, part_vol, part_img, cameras,
                       budgets: RoutingBudgets, host_lists: bool = True) -> RoutingPlan:
    """All four query->KV tables (`block_routing.py:237-258`); the device rows
    are kept on the plan for the fused attention path."""
    vp = vol_coords.points if isinstance(vol_coords, TokenCoords3D) else vol_coords
    ip = img_coords.points if isinstance(img_coords, TokenCoords3D) else img_coords
    side = ImageSide(part_img, ip, cameras) if part_img.n_occupied else None
    dev_rows = {
        "v2v": route_volume_rows(vp, part_vol, budgets.b_v2v),
        "i2v": route_volume_rows(ip, part_vol, budgets.b_i2v),
        "v2i": route_image_rows(vp, cameras, part_img, ip, budgets.b_i, budgets.b_v2i, side),
        "i2i": route_image_rows(ip, cameras, part_img, ip, budgets.b_i, budgets.b_i2i, side),
    }
    parts = {"v2v": part_vol, "i2v": part_vol, "v2i": part_img, "i2i": part_img}
    tables, fallback = {}, {}
    if host_lists:
        for name in ("v2v", "i2v", "v2i", "i2i"):
            tables[name] = _rows_to_selection(*dev_rows[name], parts[name])
            empty = [i for i, l in enumerate(tables[name].lists) if len(l) == 0]
            if empty:
                fallback[name] = empty
    plan = RoutingPlan(tables, budgets, fallback)
    plan.device_rows = dev_rows
    return plan


def write_plan(path, plan: RoutingPlan) -> None:
    """`block_routing.py:284-290`: four tables in fixed order."""
    with open(path, "wb") as fh:
        fh.write(struct.pack("<I", len(PLAN_TABLE_ORDER)))
        for name in PLAN_TABLE_ORDER:
            write_selection(fh, plan.tables[name])
