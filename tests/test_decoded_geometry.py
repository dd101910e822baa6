"""The coarse-to-fine path on DECODED geometry (the paper's contribution 1;
BASELINE config 2): the reference runner with geometry_source="decoded"
(`runner.py:301-335`) scores voxel informativeness and marches the
image-token rays on the SDF decoded from the coarse stage.

Golden: `tests/golden/ref_decoded.npz` + `ref_decoded_messages.csv`, made by
`make_golden.py decoded` from the reference's own `run_pipeline` at the
golden-run config (tests/goldens/config.json + scene.json, workers 2).

Bars: decoded grid, voxel mask, compaction coords, routing tables and the
message log bit-exact; surface points as the analytic march (miss flags
identical, >= 99% within 1e-12); stage outputs and probes <= 1e-5.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, unflat

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dec():
    return golden("ref_decoded.npz")


def _heads(z):
    from paper_2604_05182_b200.recon_pipeline import init_decoder_heads
    h = init_decoder_heads(int(z["seed"]))
    (w1, b1, _), (w2, b2, _) = h.s_layers
    for a, key in ((w1, "s_w1"), (b1, "s_b1"), (w2, "s_w2"), (b2, "s_b2")):
        assert np.array_equal(a, z[key]), key      # same tagged init as the reference
    return h


def _fine_cams(z):
    return [(z["cam_K"][i], z["cam_R"][i], z["cam_t"][i], tuple(int(v) for v in z["cam_wh"][i]))
            for i in range(z["cam_K"].shape[0])]


def test_decoded_grid_bit_exact(cuda, dec):
    """decode_feature_volume with the reference's f64 einsum affine."""
    import paper_2604_05182_b200 as L
    w = L.init_decode(int(dec["seed"]), int(dec["d"]), "dec_coarse")
    grid = L.decode_feature_volume(dec["x_d"], w)
    assert np.array_equal(grid, dec["dense_grid"])


def test_decoded_voxel_mask_bit_exact(cuda, dec):
    """Eq. 11 on the decoded SDF, evaluated in-kernel (DecodedSdf) and through
    the opaque-callable path (the reference runner's lambda shape)."""
    import paper_2604_05182_b200 as L
    heads = _heads(dec)
    s = int(dec["s_vol_fine"])
    field = L.decoded_sdf_field(dec["dense_grid"], heads)
    got = L.informative_voxel_mask(field, s)
    want = dec["vol_mask"]
    print(f"decoded mask: {int(want.sum())} / {want.size} voxels, "
          f"{int((got != want).sum())} differ")
    assert np.array_equal(got, want)
    fv = L.FeatureVolume(dec["dense_grid"])
    opaque = L.callable_field(lambda p: L.decode_points(fv, heads, p)[1].astype(np.float64))
    assert np.array_equal(L.informative_voxel_mask(opaque, s), want)


def test_opaque_callable_matches_analytic(cuda):
    """A pure-NumPy callable field (the oracle's analytic SDF) through the
    host-evaluated path gives the analytic in-kernel mask and march."""
    import oracle as O
    import paper_2604_05182_b200 as L
    from fixtures import load_workload
    scene = {"kind": "union", "parts": [
        {"kind": "sphere", "center": [0.42, 0.5, 0.55], "radius": 0.18},
        {"kind": "box", "center": [0.6, 0.45, 0.4], "half_sizes": [0.12, 0.12, 0.12]}]}
    opaque = L.callable_field(lambda p: O.eval_sdf(scene, p))
    assert np.array_equal(L.informative_voxel_mask(opaque, 32), L.informative_voxel_mask(scene, 32))
    wl = load_workload("c1")
    ic = np.argwhere(wl.img_mask)
    coords = np.stack([ic[:, 0], ic[:, 2], ic[:, 1]], 1).astype(np.int64)[::7]

    class _T:
        pass
    t = _T()
    t.coords, t.grid_res, t.count = coords, tuple(wl.img_mask.shape), coords.shape[0]
    a = L.image_token_coords(t, wl.cameras, scene)
    b = L.image_token_coords(t, wl.cameras, opaque)
    assert np.array_equal(a.miss, b.miss)
    assert np.max(np.abs(a.points - b.points)) <= 1e-12


def _tokens_and_plan(dec):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.tokenizer import init_pos_embed
    seed, d = int(dec["seed"]), int(dec["d"])
    sv, si = int(dec["s_vol_fine"]), int(dec["s_img_fine"])
    pe_v = init_pos_embed(seed, 3, sv, d, label="pos_vol_fine")
    pe_i = init_pos_embed(seed, 2, si, d, label="pos_img_fine")
    x_up, y_up = L.upsample_select_tokens(dec["x_d"], dec["y_d"], dec["vol_mask"],
                                          dec["img_mask"], pe_v, pe_i, int(dec["factor_vol"]),
                                          int(dec["factor_img"]))
    assert np.array_equal(x_up.coords, dec["x_coords"])
    assert np.array_equal(y_up.coords, dec["y_coords"])
    field = L.decoded_sdf_field(dec["dense_grid"], _heads(dec))
    ic = L.image_token_coords(y_up, _fine_cams(dec), field)
    pv, pi = L.partition(x_up), L.partition(y_up)
    b = [int(v) for v in dec["budgets"]]
    bud = L.RoutingBudgets(b_i=b[0], b_v2v=b[1], b_v2i=b[2], b_i2v=b[3], b_i2i=b[4])
    plan = L.build_routing_plan(L.volume_token_coords(x_up), ic, pv, pi, _fine_cams(dec), bud)
    return x_up, y_up, ic, pv, pi, plan


def test_decoded_surface_points_and_plan(cuda, dec):
    x_up, y_up, ic, pv, pi, plan = _tokens_and_plan(dec)
    err = np.max(np.abs(ic.points - dec["img_points"]), axis=1)
    exact = float(np.mean(err <= 1e-12))
    print(f"decoded march: {err.size} rays, {100 * exact:.1f}% within 1e-12, "
          f"max err {err.max():.2e}")
    assert np.array_equal(ic.miss, dec["img_miss"])
    assert exact >= 0.99 and err.max() <= np.sqrt(3.0) / 128
    for name in ("v2v", "v2i", "i2v", "i2i"):
        want = unflat(dec[f"plan_{name}"], dec[f"plan_{name}_len"])
        got = plan.tables[name].lists
        bad = [i for i, (a, b) in enumerate(zip(got, want)) if not np.array_equal(a, b)]
        assert not bad, (name, len(bad))


def test_decoded_pipeline_stage_and_messages(cuda, dec, tmp_path):
    """Tokens, routing, the sparse stage (fp32 reference API, serial and the
    W = 2 sharded stage's message log) and the probe decode of the decoded
    run vs the reference."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.recon_pipeline import init_sparse_block
    x_up, y_up, ic, pv, pi, plan = _tokens_and_plan(dec)
    seed, d = int(dec["seed"]), int(dec["d"])
    hq, hkv = (int(v) for v in dec["heads"])
    params = L.AttentionParams(hq, hkv, d // hq)
    depth = int(dec["depth_sparse"])
    ws = [init_sparse_block(seed, params, layer) for layer in range(depth)]
    ctx = L.build_sparse_context(pv, pi, selections=plan.tables)
    x_s, y_s = L.sparse_stage_forward(x_up, y_up, ws, ctx, params)
    ex = float(np.max(np.abs(x_s.astype(np.float64) - dec["x_s"])))
    ey = float(np.max(np.abs(y_s.astype(np.float64) - dec["y_s"])))
    print(f"decoded stage: max|dx| {ex:.2e} max|dy| {ey:.2e}")
    assert ex <= 1e-5 and ey <= 1e-5
    _, _, topo = L.parallel_sparse_stage(x_up, y_up, ws, ctx, params, int(dec["workers"]))
    out = tmp_path / "messages.csv"
    L.message_log_to_csv(topo.message_log, out)
    with open(os.path.join(GOLDEN, "ref_decoded_messages.csv"), "rb") as fh:
        assert out.read_bytes() == fh.read()
    # probe decode on the blended sparse/dense field (runner.py:353-359)
    heads = _heads(dec)
    xs_tok = L.TokenSet("volume", x_s, x_up.coords, x_up.grid_res)
    idx, rows = L.build_sparse_features(xs_tok, L.init_decode(seed, d, "dec_fine"))
    fv = L.FeatureVolume(dec["dense_grid"], idx, rows)
    z, s = L.decode_points(fv, heads, dec["probe"], mask=dec["vol_mask"])
    ez = float(np.max(np.abs(z - dec["probe_z"])))
    es = float(np.max(np.abs(s - dec["probe_s"])))
    print(f"probes: max|dz| {ez:.2e} max|ds| {es:.2e}; checksum s "
          f"{float(np.sum(s, dtype=np.float64)):.10f} vs {float(np.sum(dec['probe_s'], dtype=np.float64)):.10f}")
    assert ez <= 1e-5 and es <= 1e-5
