"""The consumers either side of the sparse stage on the
GPU, pinned to the REAL reference's outputs (tests/golden/make_stage1.py ->
ref_stage1.npz): one Stage-1 dense block (`recon_pipeline.py:154-184`), the
dense coarse feature grid, the sparse fine features and the blended field
query + decoder heads (`recon_pipeline.py:223-365`).  C1 geometry and inputs.
"""

import numpy as np
import pytest

from conftest import golden
from paper_2604_05182_b200.workloads import coarse_inputs
from fixtures import load_workload

FLOAT_TOL = 1e-5      # the reference's own golden tolerance
DECODE_RTOL = 1e-6    # f64 decode arithmetic, f32 outputs


@pytest.fixture(scope="module")
def ref():
    return golden("ref_stage1.npz")


def test_fixture_shapes(ref):
    assert tuple(ref["grid_shape"]) == (32, 32, 32, 32)
    assert ref["probe_z"].shape == (2048, 3) and ref["probe_s"].shape == (2048,)
    assert np.all((ref["probe"] >= 0) & (ref["probe"] <= 1))


def _c1():
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import _dev as D
    wl = load_workload("c1")
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 64)
    x_up, _ = L.upsample_select_tokens(D.dev(x_d), D.dev(y_d), wl.vol_mask, wl.img_mask,
                                       pe_v, pe_i, wl.factor_vol, wl.factor_img)
    return wl, x_d, y_d, x_up


def _close(got, want, rtol):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want)) / max(1.0, float(np.max(np.abs(want)))))


@pytest.mark.gpu
def test_dense_block_matches_reference(cuda, ref):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.recon_pipeline import dense_block_forward, init_dense_block
    _, x_d, y_d, _ = _c1()
    params = L.AttentionParams(8, 1, 8)
    x2, y2 = dense_block_forward(x_d, y_d, init_dense_block(0, params, 0), params)
    assert _close(x2[::8], ref["dense_x"], FLOAT_TOL) <= FLOAT_TOL
    assert _close(y2[::8], ref["dense_y"], FLOAT_TOL) <= FLOAT_TOL


@pytest.mark.gpu
def test_decode_grid_sparse_features_and_probes(cuda, ref):
    from paper_2604_05182_b200.recon_pipeline import (FeatureVolume, build_sparse_features,
                                                      decode_feature_volume, decode_points,
                                                      init_decode, init_decoder_heads,
                                                      query_field)
    wl, x_d, _, x_up = _c1()
    grid = decode_feature_volume(x_d, init_decode(0, 64, "dec_coarse"))
    assert grid.shape == tuple(ref["grid_shape"])
    assert _close(grid.ravel()[::97], ref["grid_sample"], DECODE_RTOL) <= DECODE_RTOL
    index, rows = build_sparse_features(x_up, init_decode(0, 64, "dec_fine"))
    index, rows = index.cpu().numpy(), rows.cpu().numpy()
    assert int((index >= 0).sum()) == int(ref["index_count"][0])
    assert int(index[index >= 0].sum()) == int(ref["index_sum"][0])
    assert np.array_equal(index.ravel()[::1009], ref["index_sample"])
    assert rows.shape == tuple(ref["rows_shape"])
    assert _close(rows[::61], ref["rows_sample"], DECODE_RTOL) <= DECODE_RTOL
    heads = init_decoder_heads(0)
    fv = FeatureVolume(grid, index, rows)
    z, s = decode_points(fv, heads, ref["probe"], mask=wl.vol_mask)
    assert _close(z, ref["probe_z"], DECODE_RTOL) <= DECODE_RTOL
    assert _close(s, ref["probe_s"], DECODE_RTOL) <= DECODE_RTOL
    z2, s2 = decode_points(FeatureVolume(grid), heads, ref["probe"])
    assert _close(z2, ref["probe_dense_z"], DECODE_RTOL) <= DECODE_RTOL
    assert _close(s2, ref["probe_dense_s"], DECODE_RTOL) <= DECODE_RTOL
    f = query_field(fv, wl.vol_mask, ref["probe"][:4])
    assert f.shape == (4, 32)


@pytest.mark.gpu
def test_decode_rejects_points_outside_the_cube(cuda):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.recon_pipeline import (FeatureVolume, decode_points,
                                                      init_decoder_heads)
    fv = FeatureVolume(np.zeros((4, 4, 4, 32), np.float32))
    with pytest.raises(L.OutOfDomainError):
        decode_points(fv, init_decoder_heads(0), np.array([[0.5, 1.2, 0.5]]))


# ---------------------------------------------------------------------------
# LSRMGV1 golden-vector files (tensor_core.py:255-311), host-side format


def test_goldens_reader_and_writer_match_reference_bytes(tmp_path):
    import os
    from conftest import GOLDEN
    from paper_2604_05182_b200.tensor_core import read_goldens, write_goldens
    path = os.path.join(GOLDEN, "ref_goldens_small.bin")
    ts = read_goldens(path)
    # the writer's ascontiguousarray turns a 0-d scalar into shape (1,)
    assert [t.shape for t in ts] == [(3, 5), (4, 3), (7,), (1,), (2, 0, 3)]
    out = tmp_path / "g.bin"
    write_goldens(out, ts)
    assert out.read_bytes() == open(path, "rb").read()


@pytest.mark.parametrize("mutate,offset", [
    (lambda b: b"XSRMGV1\x00" + b[8:], 0),          # bad magic
    (lambda b: b[:10], 8),                           # truncated count
    (lambda b: b[:-4], None),                        # truncated payload
    (lambda b: b + b"\x00", None),                   # trailing bytes
])
def test_goldens_reader_rejects_malformed_files(tmp_path, mutate, offset):
    import os
    from conftest import GOLDEN
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.tensor_core import read_goldens
    blob = open(os.path.join(GOLDEN, "ref_goldens_small.bin"), "rb").read()
    p = tmp_path / "bad.bin"
    p.write_bytes(mutate(blob))
    with pytest.raises(L.GoldenFormatError) as ei:
        read_goldens(p)
    if offset is not None:
        assert ei.value.byte_offset == offset


def test_goldens_reader_rejects_rank_above_16(tmp_path):
    import struct
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.tensor_core import read_goldens
    p = tmp_path / "r.bin"
    p.write_bytes(b"LSRMGV1\x00" + struct.pack("<II", 1, 17))
    with pytest.raises(L.GoldenFormatError, match="rank 17"):
        read_goldens(p)
