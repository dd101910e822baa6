"""The GPU workload generator (workloads.generate_workload, every config) must
reproduce the reference-made fixtures: cameras bit-exact on the CPU; masks,
token counts and image-token surface points on the GPU."""

import numpy as np
import pytest

from paper_2604_05182_b200.workloads import orbit_cameras

from fixtures import load_workload


@pytest.mark.parametrize("name,views,s_img", [("c1", 4, 96), ("c3", 16, 96)])
def test_orbit_cameras_bit_exact(name, views, s_img):
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, f"workload_{name}.npz"))
    cams = orbit_cameras(views, 1.7, 20.0, (8 * s_img, 8 * s_img))
    for i, (K, R, t, _) in enumerate(cams):
        assert np.array_equal(K, z["cam_K"][i])
        assert np.array_equal(R, z["cam_R"][i])
        assert np.array_equal(t, z["cam_t"][i])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c3", "c4"])
def test_generated_workload_matches_fixture(cuda, name):
    """The package's own workloads (what build_instance and bench.py use) are
    the reference-made fixtures: masks (C4 skew blocks included) and token
    counts bit-exact, surface points within 1e-12."""
    from paper_2604_05182_b200 import workloads as W
    ref = load_workload(name)
    got = W.load_workload(name)
    assert np.array_equal(got.vol_mask, ref.vol_mask)
    assert np.array_equal(got.img_mask, ref.img_mask)
    assert (got.n_vol, got.n_img) == (ref.n_vol, ref.n_img)
    assert np.max(np.abs(got.img_points - ref.img_points)) <= 1e-12
