"""Synthetic BASELINE workloads, built without the reference.

Every config is generated on the GPU with this package's own kernels from the
reference's fixture recipe (`tests/test_acceptance.py:293-322` of the
reference): orbit cameras, the informative-voxel mask (plus C4's seeded
fully occupied blocks), silhouettes -> foreground patches, compaction and the
image-token surface points.  The tests pin the result against fixtures the
real reference produced (`tests/golden/workload_<cfg>.npz`,
`tests/test_workload_gen.py`); the package itself never reads them.
Features, positional tables and weights come from the same tagged Philox
streams the reference uses (`rng.py`), so the GPU path and the CPU oracle see
identical inputs.
"""

from dataclasses import dataclass

import numpy as np

from .block_routing import RoutingBudgets
from .nsa_attention import init_nsa_weights
from .rng import stream
from .tensor_core import AttentionParams
from .tokenizer import init_pos_embed

# BASELINE.json configs: C1 tiny (desk heads, fp32), C3 fine stage, C4 skewed,
# C5 scaled context (~20x object tokens, 18 views; "raise the
# object radius or S with the same recipe"; generated on the GPU)
CONFIGS = {
    "c1": {"params": (8, 1, 8), "dtype": "f32", "views": 4, "s_vol": 32, "s_img": 96},
    "c3": {"params": (32, 2, 32), "dtype": "bf16", "views": 16, "s_vol": 96, "s_img": 96},
    "c4": {"params": (32, 2, 32), "dtype": "bf16", "views": 16, "s_vol": 96, "s_img": 96,
           "skew": 12},
    "c5": {"params": (32, 2, 32), "dtype": "bf16", "views": 18, "s_vol": 408, "s_img": 288},
}
# the fixture scene (tests/test_acceptance.py:299-300 of the reference)
SCENE = {"kind": "union", "parts": [
    {"kind": "sphere", "center": [0.42, 0.5, 0.55], "radius": 0.18},
    {"kind": "box", "center": [0.6, 0.45, 0.4], "half_sizes": [0.12, 0.12, 0.12]}]}
CUBE_CENTER = np.array([0.5, 0.5, 0.5])
USE_TAGS = {"v2v": (3, "xs"), "v2i": (2, "xc"), "i2i": (3, "ys"), "i2v": (2, "yc")}


@dataclass
class Workload:
    name: str
    views: int
    s_vol: int
    s_img: int
    factor_vol: int
    factor_img: int
    vol_mask: np.ndarray      # [S,S,S] bool
    img_mask: np.ndarray      # [V,S,S] bool
    cameras: list             # [(K, R, t)] f64
    img_points: np.ndarray    # [Ni,3] f64 surface points (image_token_coords)
    n_vol: int
    n_img: int


def look_at_camera(eye, target, image_size, focal, world_up=(0.0, 0.0, 1.0)):
    """(K, R, t, (W, H)) of a pinhole camera at eye looking at target,
    principal point at the image center (`camera_geometry.py:110-126`)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    up = np.asarray(world_up, dtype=np.float64)
    if abs(np.dot(fwd, up)) > 0.999:
        up = np.array([1.0, 0.0, 0.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd], axis=1)
    W, H = image_size
    K = np.array([[focal, 0.0, W / 2.0], [0.0, focal, H / 2.0], [0.0, 0.0, 1.0]])
    return (K, R, eye, (int(W), int(H)))


def orbit_cameras(count, radius, elevation_deg, image_size, fov_deg=50.0, phase=0.0):
    """Ring of cameras around the cube center (`camera_geometry.py:129-144`)."""
    import math
    focal = 0.5 * image_size[0] / math.tan(math.radians(fov_deg) / 2.0)
    el = math.radians(elevation_deg)
    cams = []
    for k in range(count):
        az = phase + 2.0 * math.pi * k / count
        eye = CUBE_CENTER + radius * np.array([math.cos(az) * math.cos(el),
                                               math.sin(az) * math.cos(el), math.sin(el)])
        cams.append(look_at_camera(eye, CUBE_CENTER, image_size, focal))
    return cams


def skew_blocks(vol_mask: np.ndarray, skew: int) -> np.ndarray:
    """C4's load-balance stress: `skew` seeded 8^3 volume blocks made fully
    occupied (stream(0, "skew"), the recipe of tests/golden/make_golden.py)."""
    vol_mask = np.array(vol_mask, dtype=bool, copy=True)
    g = stream(0, "skew")
    sb = vol_mask.shape[0] // 8
    for b in g.choice(sb ** 3, size=skew, replace=False):
        i, j, k = b // (sb * sb), (b // sb) % sb, b % sb
        vol_mask[8 * i:8 * i + 8, 8 * j:8 * j + 8, 8 * k:8 * k + 8] = True
    return vol_mask


def generate_workload(name: str, views: int, s_vol: int, s_img: int, skew: int = 0) -> Workload:
    """The fixture recipe (tests/golden/make_golden.py) on the GPU: orbit
    cameras, the informative-voxel mask, silhouettes -> foreground patches,
    compaction and the image-token surface points, all with this package's
    kernels (bit-exact with the reference for masks and coords)."""
    from . import _dev as D
    from .block_routing import LAPLACE_BETA, image_token_coords
    from .camera_geometry import silhouettes
    from .tokenizer import foreground_patch_mask, informative_voxel_mask, upsample_select_tokens
    cams = orbit_cameras(views, 1.7, 20.0, (8 * s_img, 8 * s_img))
    vol_mask = informative_voxel_mask(SCENE, s_vol)
    if skew:
        vol_mask = skew_blocks(D.host(vol_mask) if D.is_device(vol_mask) else vol_mask, skew)
    img_mask = foreground_patch_mask(silhouettes(SCENE, cams, as_device=True))
    img_mask = D.host(img_mask) if D.is_device(img_mask) else img_mask
    fv = 6 if s_vol % 6 == 0 else 4
    fi = 3
    d = 8   # features do not affect coords; image points depend on coords only
    g = stream(0, "hot")
    x_d = g.standard_normal(((s_vol // fv) ** 3, d)).astype(np.float32)
    y_d = g.standard_normal((views * (s_img // fi) ** 2, d)).astype(np.float32)
    x_up, y_up = upsample_select_tokens(D.dev(x_d), D.dev(y_d), vol_mask, img_mask,
                                        init_pos_embed(6, 3, s_vol, d, label="v"),
                                        init_pos_embed(6, 2, s_img, d, label="i"), fv, fi)
    ic = image_token_coords(y_up, cams, SCENE, LAPLACE_BETA)
    return Workload(name, views, s_vol, s_img, fv, fi, np.asarray(vol_mask, bool),
                    np.asarray(img_mask, bool), [c[:3] for c in cams], ic.points,
                    int(x_up.count), int(y_up.count))


def load_workload(name: str) -> Workload:
    """The named BASELINE config, generated on the GPU (cached per process)."""
    if name not in _CACHE:
        c = CONFIGS[name]
        _CACHE[name] = generate_workload(name, c["views"], c["s_vol"], c["s_img"],
                                         c.get("skew", 0))
    return _CACHE[name]


_CACHE = {}


def coarse_inputs(wl: Workload, d: int, seed: int = 0):
    """x_d, y_d ~ N(0,1) and the fine positional tables (SURVEY §8d recipe)."""
    g = stream(seed, "hot")
    x_d = g.standard_normal(((wl.s_vol // wl.factor_vol) ** 3, d)).astype(np.float32)
    y_d = g.standard_normal((wl.views * (wl.s_img // wl.factor_img) ** 2, d)).astype(np.float32)
    pe_v = init_pos_embed(6, 3, wl.s_vol, d, label="v")
    pe_i = init_pos_embed(6, 2, wl.s_img, d, label="i")
    return x_d, y_d, pe_v, pe_i


def nsa_use_weights(params: AttentionParams, seed: int = 0, layer: int = 0) -> dict:
    """The four NsaWeights of sparse block `layer` (`recon_pipeline.py:394-410`)."""
    tag = f"sparse{layer}"
    return {u: init_nsa_weights(seed, params, ng, tag, t) for u, (ng, t) in USE_TAGS.items()}


def params_of(name: str) -> AttentionParams:
    return AttentionParams(*CONFIGS[name]["params"])


def default_budgets() -> RoutingBudgets:
    return RoutingBudgets()
