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


# ---------------------------------------------------------------------------
# router input producer: image-token surface points (the step before K8)

N_MARCH = 128          # camera_geometry.py:18
LAPLACE_BETA = 0.02    # camera_geometry.py:19
NO_PEAK_MARGIN = 3.0   # camera_geometry.py:20


def ray_cube_intersection(o, d):
    """Slab method against [0,1]^3 (`camera_geometry.py:236-252`)."""
    t0, t1 = -np.inf, np.inf
    for ax in range(3):
        if abs(d[ax]) < 1e-12:
            if o[ax] < 0.0 or o[ax] > 1.0:
                return None
            continue
        a = (0.0 - o[ax]) / d[ax]
        b = (1.0 - o[ax]) / d[ax]
        t0 = max(t0, min(a, b))
        t1 = min(t1, max(a, b))
    if t1 <= t0 or t1 <= 0.0:
        return None
    return max(t0, 0.0), t1


def surface_peak(scene, o, d, beta=LAPLACE_BETA):
    """Opacity peak of one ray (`camera_geometry.py:264-302`): 128 mid-segment
    samples between cube entry and exit, Laplace density, peak of
    transmittance x alpha.  None if the ray misses the cube or min s > 3 beta."""
    from .tokens import eval_sdf
    d = d / np.linalg.norm(d)
    span = ray_cube_intersection(o, d)
    if span is None:
        return None, d
    t0, t1 = span
    step = (t1 - t0) / N_MARCH
    ts = t0 + (np.arange(N_MARCH) + 0.5) * step
    pts = o[None, :] + ts[:, None] * d[None, :]
    s = eval_sdf(scene, pts)
    if s.min() > NO_PEAK_MARGIN * beta:
        return None, d
    psi = np.where(s >= 0.0, 0.5 * np.exp(-s / beta), 1.0 - 0.5 * np.exp(s / beta))
    alpha = 1.0 - np.exp(-(psi / beta) * step)
    trans = np.concatenate([[1.0], np.cumprod(1.0 - alpha)[:-1]])
    return pts[int(np.argmax(trans * alpha))], d


def image_token_coords(coords, cameras, image_size, rows_f, scene, beta=LAPLACE_BETA):
    """Surface point per image token's patch-center ray, with cube-entry /
    closest-approach fallbacks and miss flags (`block_routing.py:73-108`).
    coords [N,3] (view, u=col, v=row); cameras [(K, R, t)]; image_size (W, H)."""
    n = coords.shape[0]
    pts = np.zeros((n, 3), np.float64)
    miss = np.zeros(n, bool)
    W, H = image_size
    for i in range(n):
        view, u, v = (int(c) for c in coords[i])
        K, R, t = cameras[view]
        px = ((u + 0.5) * (W / rows_f), (v + 0.5) * (H / rows_f))
        d_cam = np.array([(px[0] - K[0, 2]) / K[0, 0], (px[1] - K[1, 2]) / K[1, 1], 1.0])
        d = R @ d_cam
        d /= np.linalg.norm(d)
        o = np.asarray(t, np.float64)
        peak, dn = surface_peak(scene, o, d, beta)
        if peak is not None:
            p = np.asarray(peak)
        else:
            miss[i] = True
            span = ray_cube_intersection(o, dn)
            if span is not None:
                p = o + span[0] * dn
            else:
                t_near = float(np.dot(np.array([0.5, 0.5, 0.5]) - o, dn))
                p = o + max(t_near, 0.0) * dn
        pts[i] = np.clip(p, 0.0, 1.0)
    return pts, miss
