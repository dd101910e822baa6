"""Synthetic BASELINE workloads, built without the reference.

The scene-dependent inputs (masks, cameras, image-token surface points) were
produced once by the REAL reference geometry and committed as fixtures
(`tests/golden/workload_<cfg>.npz`, script `tests/golden/make_golden.py`).
Features, positional tables and weights are regenerated here from the same
tagged Philox streams the reference uses (`rng.py`), so the GPU path and the
CPU oracle see identical inputs.
"""

import os
from dataclasses import dataclass

import numpy as np

from .block_routing import RoutingBudgets
from .nsa_attention import init_nsa_weights
from .rng import stream
from .tensor_core import AttentionParams
from .tokenizer import init_pos_embed

FIXTURE_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "tests", "golden")

# BASELINE.json configs: C1 tiny (desk heads, fp32), C3 fine stage, C4 skewed
CONFIGS = {
    "c1": {"params": (8, 1, 8), "dtype": "f32"},
    "c3": {"params": (32, 2, 32), "dtype": "bf16"},
    "c4": {"params": (32, 2, 32), "dtype": "bf16"},
}
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


def load_workload(name: str) -> Workload:
    z = np.load(os.path.join(FIXTURE_DIR, f"workload_{name}.npz"))
    s, si, v = int(z["s_vol"]), int(z["s_img"]), int(z["views"])
    vm = np.unpackbits(z["vol_mask"])[: s ** 3].astype(bool).reshape(s, s, s)
    im = np.unpackbits(z["img_mask"])[: v * si * si].astype(bool).reshape(v, si, si)
    cams = [(z["cam_K"][i], z["cam_R"][i], z["cam_t"][i]) for i in range(v)]
    return Workload(name, v, s, si, int(z["factor_vol"]), int(z["factor_img"]), vm, im, cams,
                    z["img_points"], int(z["n_vol"]), int(z["n_img"]))


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
