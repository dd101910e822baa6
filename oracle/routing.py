"""3D-aware spatial router (TEST INFRASTRUCTURE ONLY).

Restates `lsrm/block_routing.py:115-258`.  All distance arithmetic keeps the
reference's f64 elementary-operation order (NumPy never contracts to FMA), so
the block lists — including tie order — are reproduced exactly.
"""

from dataclasses import dataclass, field

import numpy as np

from .partition import Partition

QUERY_CHUNK = 512
PATCH_PX = 8.0


@dataclass
class RoutingPlan:
    tables: dict
    budgets: dict
    fallback_queries: dict = field(default_factory=dict)


def route_volume(points, part: Partition, budget):
    """Nearest `budget` occupied block centers, ties to lower block id
    (`block_routing.py:115-143`)."""
    pts = np.asarray(points, np.float64)
    if part.n_occupied == 0:
        return [np.zeros(0, np.int64) for _ in range(pts.shape[0])]
    c = part.block_centers
    out = []
    for lo in range(0, pts.shape[0], QUERY_CHUNK):
        p = pts[lo:lo + QUERY_CHUNK]
        dx = p[:, 0, None] - c[None, :, 0]
        dy = p[:, 1, None] - c[None, :, 1]
        dz = p[:, 2, None] - c[None, :, 2]
        d2 = dx * dx + dy * dy + dz * dz
        for r in np.argsort(d2, axis=1, kind="stable")[:, :budget]:
            out.append(part.occupied_ids[r])
    return out


def project(points, K, R, t):
    """Pinhole projection with the reference's scalar order
    (`block_routing.py:150-163`, `camera_geometry.py:52-74`)."""
    dx = points[:, 0] - t[0]
    dy = points[:, 1] - t[1]
    dz = points[:, 2] - t[2]
    xc = R[0, 0] * dx + R[1, 0] * dy + R[2, 0] * dz
    yc = R[0, 1] * dx + R[1, 1] * dy + R[2, 1] * dz
    zc = R[0, 2] * dx + R[1, 2] * dy + R[2, 2] * dz
    with np.errstate(divide="ignore", invalid="ignore"):
        u = K[0, 0] * (xc / zc) + K[0, 2]
        v = K[1, 1] * (yc / zc) + K[1, 2]
    return u, v, zc


def _block_min_d2(points, part: Partition, token_points):
    """[Nq,B] min squared distance to each block's token points
    (`block_routing.py:166-180`)."""
    tp = np.asarray(token_points, np.float64)[part.block_token_ids]
    out = np.empty((points.shape[0], part.n_occupied))
    for lo in range(0, points.shape[0], QUERY_CHUNK):
        p = points[lo:lo + QUERY_CHUNK]
        dx = p[:, 0, None] - tp[None, :, 0]
        dy = p[:, 1, None] - tp[None, :, 1]
        dz = p[:, 2, None] - tp[None, :, 2]
        out[lo:lo + QUERY_CHUNK] = np.minimum.reduceat(
            dx * dx + dy * dy + dz * dz, part.block_offsets[:-1], axis=1)
    return out


def route_image(points, cameras, part: Partition, token_points, b_i, budget):
    """Two-stage image rule (`block_routing.py:183-220`): per visible view a
    stable top-b_i 2D shortlist of block centers (patch units), pooled, then
    ranked by min 3D distance to the block's token points; take
    min(budget, n_candidates).  cameras: list of (K, R, t) f64 arrays."""
    pts = np.asarray(points, np.float64)
    n = pts.shape[0]
    if part.n_occupied == 0 or n == 0:
        return [np.zeros(0, np.int64) for _ in range(n)]
    cand = np.zeros((n, part.n_occupied), bool)
    for view, (K, R, t) in enumerate(cameras):
        rows = np.flatnonzero(part.block_views == view)
        if rows.size == 0:
            continue
        u, v, z = project(pts, K, R, t)
        vis = z > 0.0
        if not vis.any():
            continue
        cu = part.block_centers[rows, 0]
        cv = part.block_centers[rows, 1]
        du = (u[vis] / PATCH_PX)[:, None] - cu[None, :]
        dv = (v[vis] / PATCH_PX)[:, None] - cv[None, :]
        short = np.argsort(du * du + dv * dv, axis=1, kind="stable")[:, :b_i]
        cand[np.flatnonzero(vis)[:, None], rows[short]] = True
    rank = np.where(cand, _block_min_d2(pts, part, token_points), np.inf)
    order = np.argsort(rank, axis=1, kind="stable")
    ncand = cand.sum(axis=1)
    return [part.occupied_ids[order[i, :min(budget, int(ncand[i]))]]
            for i in range(n)]


def build_routing_plan(vol_points, img_points, part_vol, part_img, cameras,
                       budgets):
    """The four tables, reused by every sparse layer (`block_routing.py:237-258`).
    budgets: dict with b_i, b_v2v, b_v2i, b_i2v, b_i2i."""
    tables = {
        "v2v": route_volume(vol_points, part_vol, budgets["b_v2v"]),
        "i2v": route_volume(img_points, part_vol, budgets["b_i2v"]),
        "v2i": route_image(vol_points, cameras, part_img, img_points,
                           budgets["b_i"], budgets["b_v2i"]),
        "i2i": route_image(img_points, cameras, part_img, img_points,
                           budgets["b_i"], budgets["b_i2i"]),
    }
    fb = {k: [i for i, l in enumerate(v) if len(l) == 0] for k, v in tables.items()}
    return RoutingPlan(tables, dict(budgets), {k: v for k, v in fb.items() if v})
