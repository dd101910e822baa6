"""Pin the CPU oracle (oracle/) against fixtures produced by the REAL reference
(tests/golden/make_golden.py).  Integer/index outputs must be bit-exact;
float outputs within the reference's own tolerances."""

import csv
import os

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, golden, unflat
from paper_2604_05182_b200.workloads import coarse_inputs
from fixtures import load_workload

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


@pytest.fixture(scope="module")
def c1_instance(ref_c1):
    wl = load_workload("c1")
    params = O.AttentionParams(8, 1, 8)
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 64)
    x_up, y_up = O.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v.tables,
                                          pe_i.tables, wl.factor_vol, wl.factor_img)
    pv = O.partition_tokens("volume", x_up.coords, x_up.grid_res)
    pi = O.partition_tokens("image", y_up.coords, y_up.grid_res)
    return dict(wl=wl, params=params, x_d=x_d, y_d=y_d, x_up=x_up, y_up=y_up, pv=pv, pi=pi)


def test_rng_matches_reference(ref_c1, c1_instance):
    assert np.array_equal(c1_instance["x_d"][:64], ref_c1["x_d_head"])
    assert np.array_equal(c1_instance["y_d"][:64], ref_c1["y_d_head"])


def test_compaction_bit_exact(ref_c1, c1_instance):
    assert np.array_equal(c1_instance["x_up"].coords, ref_c1["x_coords"])
    assert np.array_equal(c1_instance["y_up"].coords, ref_c1["y_coords"])
    assert np.array_equal(c1_instance["x_up"].features.view(np.uint32),
                          ref_c1["x_up"].view(np.uint32))
    assert np.array_equal(c1_instance["y_up"].features.view(np.uint32),
                          ref_c1["y_up"].view(np.uint32))


def test_voxel_mask_bit_exact(ref_c1):
    from fixtures import load_workload
    scene = {"kind": "union", "parts": [
        {"kind": "sphere", "center": [0.42, 0.5, 0.55], "radius": 0.18},
        {"kind": "box", "center": [0.6, 0.45, 0.4], "half_sizes": [0.12, 0.12, 0.12]}]}
    m = O.informative_voxel_mask(scene, 32)
    want = np.unpackbits(ref_c1["mask32"])[:32 ** 3].astype(bool).reshape(32, 32, 32)
    assert np.array_equal(m, want)
    wl = load_workload("c1")
    assert np.array_equal(m, wl.vol_mask)


def test_partition_bit_exact(ref_c1, c1_instance):
    for tag, p in (("pv", c1_instance["pv"]), ("pi", c1_instance["pi"])):
        assert np.array_equal(p.block_of_token, ref_c1[f"{tag}_block_of_token"])
        assert np.array_equal(p.occupied_ids, ref_c1[f"{tag}_occupied"])
        assert np.array_equal(p.block_offsets, ref_c1[f"{tag}_offsets"])
        assert np.array_equal(p.block_token_ids, ref_c1[f"{tag}_token_ids"])
        assert np.array_equal(p.occupancy, ref_c1[f"{tag}_occupancy"])
        assert np.array_equal(p.block_centers, ref_c1[f"{tag}_centers"])


def test_routing_plan_bit_exact(ref_c1, c1_instance):
    wl = c1_instance["wl"]
    vpts = (c1_instance["x_up"].coords.astype(np.float64) + 0.5) / wl.s_vol
    plan = O.build_routing_plan(vpts, wl.img_points, c1_instance["pv"], c1_instance["pi"],
                                wl.cameras, dict(b_i=16, b_v2v=8, b_v2i=8, b_i2v=8, b_i2i=8))
    for name in ("v2v", "v2i", "i2v", "i2i"):
        want = unflat(ref_c1[f"plan_{name}"], ref_c1[f"plan_{name}_len"])
        got = plan.tables[name]
        assert len(got) == len(want)
        assert all(np.array_equal(a, b) for a, b in zip(got, want)), name


def test_gather_table_lengths(ref_c1, c1_instance):
    pv, pi = c1_instance["pv"], c1_instance["pi"]
    parts = {"v2v": pv, "i2v": pv, "v2i": pi, "i2i": pi}
    for name in ("v2v", "v2i", "i2v", "i2i"):
        lists = unflat(ref_c1[f"plan_{name}"], ref_c1[f"plan_{name}_len"])
        own = parts[name].block_of_token if name in ("v2v", "i2i") else None
        tab = O.build_gather_table(lists, parts[name], own_block=own)
        assert np.array_equal(tab.lengths, ref_c1[f"table_{name}_len"])


@pytest.mark.parametrize("seed", range(3))
def test_sel_win_small(ref_small, seed):
    r = ref_small
    params = O.AttentionParams(4, 2, 8)
    coords = r[f"s{seed}_coords"]
    part = O.partition_tokens("volume", coords, (16, 16, 16))
    q, k, v = r[f"s{seed}_q"], r[f"s{seed}_k"], r[f"s{seed}_v"]
    lists = unflat(r[f"s{seed}_sel"], r[f"s{seed}_sel_len"])
    got = O.sel_attention(q, k, v, part, lists, params, own_block=part.block_of_token)
    assert np.max(np.abs(got.astype(np.float64) - r[f"s{seed}_out_sel"])) < 1e-6
    tab = O.build_gather_table(lists, part, own_block=part.block_of_token)
    assert np.array_equal(tab.lengths, r[f"s{seed}_tab_len"])
    w = O.win_attention(q, k, v, part, params)
    assert np.max(np.abs(w.astype(np.float64) - r[f"s{seed}_out_win"])) < 1e-6


def test_nsa_uses_c1(ref_c1, c1_instance):
    """The four gated NSA uses at C1 (desk heads 8/1/8, d=64), 1e-5."""
    params = c1_instance["params"]
    x_up, y_up = c1_instance["x_up"], c1_instance["y_up"]
    pv, pi = c1_instance["pv"], c1_instance["pi"]
    d = 64
    ones, zeros = np.ones(d, np.float32), np.zeros(d, np.float32)
    xh = O.layer_norm(x_up.features, ones, zeros)
    yh = O.layer_norm(y_up.features, ones, zeros)
    blk = O.init_sparse_block(0, params, 0)
    parts = {"v2v": (xh, xh, pv, pv), "v2i": (xh, yh, pv, pi), "i2i": (yh, yh, pi, pi),
             "i2v": (yh, xh, pi, pv)}
    for name, (xq, xkv, pq, pkv) in parts.items():
        lists = unflat(ref_c1[f"plan_{name}"], ref_c1[f"plan_{name}_len"])
        got = O.nsa_use(xq, xkv, pq, pkv, lists, blk.nsa[name], params)
        assert np.max(np.abs(got.astype(np.float64) - ref_c1[f"use_{name}"])) < 1e-5, name


def test_sparse_block_c1(ref_c1, c1_instance):
    params = c1_instance["params"]
    x_up, y_up = c1_instance["x_up"], c1_instance["y_up"]
    pv, pi = c1_instance["pv"], c1_instance["pi"]
    blk = O.init_sparse_block(0, params, 0)
    sels = {n: unflat(ref_c1[f"plan_{n}"], ref_c1[f"plan_{n}_len"]) for n in
            ("v2v", "v2i", "i2v", "i2i")}
    own = {"v2v": pv.block_of_token, "i2i": pi.block_of_token}
    kvp = {"v2v": pv, "v2i": pi, "i2v": pv, "i2i": pi}
    tables = {n: O.build_gather_table(sels[n], kvp[n], own_block=own.get(n)) for n in sels}
    ctx = {"part_vol": pv, "part_img": pi, "selections": sels, "tables": tables}
    xi = O.affine(x_up.features, blk.inj_x)
    yi = O.affine(y_up.features, blk.inj_y)
    x2, y2 = O.sparse_block_forward(np.zeros_like(xi), np.zeros_like(yi), xi, yi, blk, ctx,
                                    params)
    assert np.max(np.abs(x2.astype(np.float64) - ref_c1["block_x"])) < 1e-5
    assert np.max(np.abs(y2.astype(np.float64) - ref_c1["block_y"])) < 1e-5


def test_shard_blocks_and_message_log(ref_c1, c1_instance):
    pv, pi = c1_instance["pv"], c1_instance["pi"]
    for W in (2, 3, 8):
        topo = O.shard_blocks(pv, pi, W)
        assert np.array_equal(topo.loads, ref_c1[f"shard{W}_loads"])
        want_v = unflat(ref_c1[f"shard{W}_vol"], ref_c1[f"shard{W}_vol_len"])
        want_i = unflat(ref_c1[f"shard{W}_img"], ref_c1[f"shard{W}_img_len"])
        assert all(np.array_equal(a, b) for a, b in zip(topo.vol_rows, want_v))
        assert all(np.array_equal(a, b) for a, b in zip(topo.img_rows, want_i))


def _golden_run_log():
    z = golden("ref_goldenrun.npz")
    xc, yc = z["x_coords"], z["y_coords"]
    pv = O.partition_tokens("volume", xc, tuple(z["x_grid"]))
    pi = O.partition_tokens("image", yc, tuple(z["y_grid"]))
    W, d, width, depth = int(z["workers"]), int(z["d"]), int(z["width"]), int(z["depth"])
    topo = O.shard_blocks(pv, pi, W)
    n_x = xc.shape[0]
    aligned = [np.concatenate([topo.vol_tokens[w], topo.img_tokens[w] + n_x]) for w in range(W)]
    naive = O.naive_contiguous_shards(n_x + yc.shape[0], W)
    O.all_to_all_accounting(naive, aligned, topo, "dispatch", 4 * d + O.seqpar.TOKEN_COORD_BYTES)
    for m in range(depth):
        for name, kv_is_vol, is_self in (("v2v", True, True), ("v2i", False, False),
                                         ("i2i", False, True), ("i2v", True, False)):
            toks = topo.vol_tokens if kv_is_vol else topo.img_tokens
            rows = topo.vol_rows if kv_is_vol else topo.img_rows
            O.all_gather_kv_accounting([t.size for t in toks], [r.size for r in rows], width,
                                       topo, f"layer{m}/{name}")
            if is_self:
                for w in range(W):
                    topo.message_log.append((f"layer{m}/{name}/win", "window", w, w, 0))
    O.all_to_all_accounting(aligned, naive, topo, "return", 4 * d + O.seqpar.TOKEN_COORD_BYTES)
    return topo.message_log


def test_golden_run_messages_csv_byte_identical():
    """The reference's committed golden run (tests/goldens/reference/messages.csv)."""
    log = _golden_run_log()
    with open(os.path.join(GOLDEN, "ref_goldenrun_messages.csv")) as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == ["phase", "kind", "src", "dst", "bytes"]
    want = [(r[0], r[1], int(r[2]), int(r[3]), int(r[4])) for r in rows[1:]]
    assert log == want


def test_c1_parallel_message_log(ref_c1, c1_instance):
    """Message log of the reference's 3-worker parallel stage at C1."""
    pv, pi = c1_instance["pv"], c1_instance["pi"]
    topo = O.shard_blocks(pv, pi, 3)
    n_x = pv.n_tokens
    aligned = [np.concatenate([topo.vol_tokens[w], topo.img_tokens[w] + n_x]) for w in range(3)]
    naive = O.naive_contiguous_shards(n_x + pi.n_tokens, 3)
    O.all_to_all_accounting(naive, aligned, topo, "dispatch", 4 * 64 + 12)
    for name, kv_is_vol, is_self in (("v2v", True, True), ("v2i", False, False),
                                     ("i2i", False, True), ("i2v", True, False)):
        toks = topo.vol_tokens if kv_is_vol else topo.img_tokens
        rows = topo.vol_rows if kv_is_vol else topo.img_rows
        O.all_gather_kv_accounting([t.size for t in toks], [r.size for r in rows], 8, topo,
                                   f"layer0/{name}")
        if is_self:
            for w in range(3):
                topo.message_log.append((f"layer0/{name}/win", "window", w, w, 0))
    O.all_to_all_accounting(aligned, naive, topo, "return", 4 * 64 + 12)
    got = ["%s,%s,%d,%d,%d" % r for r in topo.message_log]
    assert got == list(ref_c1["par3_log"])
