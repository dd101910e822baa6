"""Test-side reader of the reference-made workload fixtures
(`tests/golden/workload_<cfg>.npz`, written by `tests/golden/make_golden.py`
with the real reference's geometry).  The package generates the same
workloads itself on the GPU (`workloads.load_workload`); the tests use these
fixtures as the reference's ground truth."""

import os

import numpy as np

from paper_2604_05182_b200.workloads import Workload

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_workload(name: str) -> Workload:
    z = np.load(os.path.join(GOLDEN, f"workload_{name}.npz"))
    s, si, v = int(z["s_vol"]), int(z["s_img"]), int(z["views"])
    vm = np.unpackbits(z["vol_mask"])[: s ** 3].astype(bool).reshape(s, s, s)
    im = np.unpackbits(z["img_mask"])[: v * si * si].astype(bool).reshape(v, si, si)
    cams = [(z["cam_K"][i], z["cam_R"][i], z["cam_t"][i]) for i in range(v)]
    return Workload(name, v, s, si, int(z["factor_vol"]), int(z["factor_img"]), vm, im, cams,
                    z["img_points"], int(z["n_vol"]), int(z["n_img"]))
