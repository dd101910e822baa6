"""Golden vectors for the consumers either side of the sparse stage
(SURVEY.md §8f rank 4): one Stage-1 dense block and the feature decode
(dense grid, sparse fine features, blended field query + decoder heads).

Run in the build container only (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_stage1.py

Inputs are the C1 coarse tokens (`rng.stream(0, "hot")`, as ref_c1) and the
C1 compacted volume tokens; outputs are subsampled to keep the fixture small.
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import lsrm  # noqa: E402
from lsrm import rng  # noqa: E402
from lsrm.recon_pipeline import (FeatureVolume, build_sparse_features,  # noqa: E402
                                 decode_feature_volume, decode_points, dense_block_forward,
                                 init_decode, init_decoder_heads, init_dense_block)
from lsrm.tokenizer import init_pos_embed  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROW_STEP = 8          # dense-block output rows kept
GRID_STEP = 97        # dense feature grid entries kept (flattened)
ROWS_STEP = 61        # sparse feature rows kept
N_PROBE = 2048


def main():
    wl = np.load(os.path.join(HERE, "workload_c1.npz"))
    s_vol, s_img, views = int(wl["s_vol"]), int(wl["s_img"]), int(wl["views"])
    vol_mask = np.unpackbits(wl["vol_mask"])[: s_vol ** 3].astype(bool).reshape((s_vol,) * 3)
    img_mask = np.unpackbits(wl["img_mask"])[: views * s_img ** 2].astype(bool).reshape(
        views, s_img, s_img)
    params = lsrm.AttentionParams(8, 1, 8)
    d = params.model_dim
    g = rng.stream(0, "hot")
    x_d = g.standard_normal((8 ** 3, d)).astype(np.float32)
    y_d = g.standard_normal((4 * 32 ** 2, d)).astype(np.float32)
    out = {}
    w = init_dense_block(0, params, 0)
    x2, y2 = dense_block_forward(x_d, y_d, w, params)
    out["dense_x"], out["dense_y"] = x2[::ROW_STEP], y2[::ROW_STEP]
    # decode: coarse dense grid from the coarse volume tokens, sparse fine
    # features from the compacted C1 volume tokens, then the probe query
    dec_c, dec_f = init_decode(0, d, "dec_coarse"), init_decode(0, d, "dec_fine")
    heads = init_decoder_heads(0)
    grid = decode_feature_volume(x_d, dec_c)
    out["grid_shape"] = np.array(grid.shape)
    out["grid_sample"] = grid.ravel()[::GRID_STEP]
    pe_v = init_pos_embed(6, 3, 32, d, label="v")
    pe_i = init_pos_embed(6, 2, 96, d, label="i")
    x_up, _ = lsrm.upsample_select_tokens(x_d, y_d, vol_mask, img_mask, pe_v, pe_i, 4, 3)
    index, rows = build_sparse_features(x_up, dec_f)
    out["index_count"] = np.array([(index >= 0).sum()])
    out["index_sum"] = np.array([index[index >= 0].sum()])
    out["index_sample"] = index.ravel()[::1009]
    out["rows_shape"] = np.array(rows.shape)
    out["rows_sample"] = rows[::ROWS_STEP]
    fv = FeatureVolume(grid, index, rows)
    probe = rng.stream(0, "probe").random((N_PROBE, 3))
    # half the probes near the occupied region so every corner mix occurs
    near = (x_up.coords[rng.stream(0, "probe_tok").integers(0, x_up.count, N_PROBE // 2)]
            + rng.stream(0, "probe_off").random((N_PROBE // 2, 3))) / 32.0
    probe[: N_PROBE // 2] = np.clip(near, 0.0, 1.0)
    z, s = decode_points(fv, heads, probe, mask=vol_mask)
    out["probe"], out["probe_z"], out["probe_s"] = probe, z, s
    z2, s2 = decode_points(FeatureVolume(grid), heads, probe)
    out["probe_dense_z"], out["probe_dense_s"] = z2, s2
    np.savez_compressed(os.path.join(HERE, "ref_stage1.npz"), **out)
    # an LSRMGV1 file written by the reference's own writer
    from lsrm.tensor_core import write_goldens
    write_goldens(os.path.join(HERE, "ref_goldens_small.bin"),
                  [x2[:3, :5], z[:4], s[:7], np.float32(2.5), np.zeros((2, 0, 3), np.float32)])
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
