"""Generate the committed golden fixtures by running the REAL reference.

Run in the build container only (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `lsrm` 0.1.0 from /root/reference/pkg/src and writes
  workload_<cfg>.npz  -- synthetic-scene inputs per BASELINE config (masks,
                         cameras, image-token surface points); built with the
                         reference's own geometry (orbit_cameras,
                         silhouette_alpha, informative_voxel_mask,
                         image_token_coords) per SURVEY.md §8d.
  ref_c1.npz          -- reference outputs at C1 for pinning the oracle and
                         the CUDA path (partition, routing plan, compaction,
                         the four NSA uses and their branches, one sparse
                         block, shard/message log).
  ref_small.npz       -- reference attention outputs on small random sets
                         (the reference tests' small_params geometry).
  ref_goldenrun.npz   -- token coords of the reference's golden run
                         (tests/goldens/config.json + scene.json) whose
                         message log must reproduce messages.csv.
Lists of ragged int arrays are stored flattened with a lengths array.
"""

import os
import shutil
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import lsrm  # noqa: E402
from lsrm import rng  # noqa: E402
from lsrm.block_routing import RoutingBudgets  # noqa: E402
from lsrm.camera_geometry import LAPLACE_BETA  # noqa: E402
from lsrm.nsa_attention import (combine_nsa_branches, nsa_gates)  # noqa: E402
from lsrm.recon_pipeline import (init_sparse_block,  # noqa: E402
                                 sparse_block_forward)
from lsrm.tensor_core import affine  # noqa: E402
from lsrm.tokenizer import init_pos_embed  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# SURVEY.md §8d fixture recipe (tests/test_acceptance.py:293-322 pattern)
SCENE = {"kind": "union", "parts": [
    {"kind": "sphere", "center": [0.42, 0.5, 0.55], "radius": 0.18},
    {"kind": "box", "center": [0.6, 0.45, 0.4], "half_sizes": [0.12, 0.12, 0.12]}]}
CONFIGS = {
    "c1": dict(views=4, s_vol=32, s_img=96, skew=0),
    "c3": dict(views=16, s_vol=96, s_img=96, skew=0),
    "c4": dict(views=16, s_vol=96, s_img=96, skew=12),
}


def flat(lists):
    lens = np.array([len(x) for x in lists], np.int64)
    vals = (np.concatenate([np.asarray(x, np.int64) for x in lists])
            if len(lists) else np.zeros(0, np.int64))
    return vals.astype(np.int64), lens


def field():
    return lsrm.union_field(lsrm.sphere_field((0.42, 0.5, 0.55), 0.18),
                            lsrm.box_field((0.6, 0.45, 0.4), (0.12, 0.12, 0.12)))


def workload(name, views, s_vol, s_img, skew):
    f = field()
    cams = lsrm.orbit_cameras(views, 1.7, 20.0, (8 * s_img, 8 * s_img))
    vol_mask = lsrm.informative_voxel_mask(f, s_vol)
    mask_pure = vol_mask.copy()
    if skew:
        g = rng.stream(0, "skew")
        sb = s_vol // 8
        for b in g.choice(sb ** 3, size=skew, replace=False):
            i, j, k = b // (sb * sb), (b // sb) % sb, b % sb
            vol_mask[8 * i:8 * i + 8, 8 * j:8 * j + 8, 8 * k:8 * k + 8] = True
    alphas = [lsrm.silhouette_alpha(f, c) for c in cams]
    img_mask = np.stack([lsrm.foreground_patch_mask(a) for a in alphas])
    fv = 6 if s_vol % 6 == 0 else 4
    fi = 3
    d = 8  # features do not affect coords; image points depend on coords only
    g = rng.stream(0, "hot")
    x_d = g.standard_normal(((s_vol // fv) ** 3, d)).astype(np.float32)
    y_d = g.standard_normal((views * (s_img // fi) ** 2, d)).astype(np.float32)
    x_up, y_up = lsrm.upsample_select_tokens(
        x_d, y_d, vol_mask, img_mask, init_pos_embed(6, 3, s_vol, d, label="v"),
        init_pos_embed(6, 2, s_img, d, label="i"), fv, fi)
    ic = lsrm.image_token_coords(y_up, cams, f, LAPLACE_BETA)
    out = dict(
        views=views, s_vol=s_vol, s_img=s_img, skew=skew, factor_vol=fv,
        factor_img=fi,
        vol_mask=np.packbits(vol_mask.ravel()),
        vol_mask_pure=np.packbits(mask_pure.ravel()),
        img_mask=np.packbits(img_mask.ravel()),
        cam_K=np.stack([c.intrinsics for c in cams]),
        cam_R=np.stack([c.rotation for c in cams]),
        cam_t=np.stack([c.translation for c in cams]),
        img_points=ic.points, img_miss=ic.miss,
        n_vol=x_up.count, n_img=y_up.count)
    if name == "c1":
        # alpha of view 0 pins foreground_patch_mask (float input)
        out["alpha0"] = np.packbits(alphas[0].ravel() > 0.5)
    np.savez_compressed(os.path.join(HERE, f"workload_{name}.npz"), **out)
    print(name, x_up.count, y_up.count)
    return cams, f, vol_mask, img_mask, ic


def ref_c1(cams, f, vol_mask, img_mask, ic):
    c = CONFIGS["c1"]
    params = lsrm.AttentionParams(8, 1, 8)
    d = params.model_dim
    g = rng.stream(0, "hot")
    fv = 4
    x_d = g.standard_normal(((c["s_vol"] // fv) ** 3, d)).astype(np.float32)
    y_d = g.standard_normal((c["views"] * (c["s_img"] // 3) ** 2, d)).astype(np.float32)
    pe_v = init_pos_embed(6, 3, c["s_vol"], d, label="v")
    pe_i = init_pos_embed(6, 2, c["s_img"], d, label="i")
    x_up, y_up = lsrm.upsample_select_tokens(x_d, y_d, vol_mask, img_mask,
                                             pe_v, pe_i, fv, 3)
    pv, pi = lsrm.partition(x_up), lsrm.partition(y_up)
    vc = lsrm.volume_token_coords(x_up)
    plan = lsrm.build_routing_plan(vc, ic, pv, pi, cams, RoutingBudgets())
    ctx = lsrm.build_sparse_context(pv, pi, selections=plan.tables)
    w = init_sparse_block(0, params, 0)
    x0 = np.zeros_like(x_up.features)
    y0 = np.zeros_like(y_up.features)
    xi = affine(x_up.features, w.inj_x)
    yi = affine(y_up.features, w.inj_y)
    x2, y2 = sparse_block_forward(x0, y0, xi, yi, w, ctx, params)
    out = dict(x_d_head=x_d[:64], y_d_head=y_d[:64], x_up=x_up.features, x_coords=x_up.coords,
               y_up=y_up.features, y_coords=y_up.coords, block_x=x2, block_y=y2,
               mask32=np.packbits(lsrm.informative_voxel_mask(f, 32).ravel()))
    for tag, p in (("pv", pv), ("pi", pi)):
        out[f"{tag}_block_of_token"] = p.block_of_token
        out[f"{tag}_occupied"] = p.occupied_ids
        out[f"{tag}_offsets"] = p.block_offsets
        out[f"{tag}_token_ids"] = p.block_token_ids
        out[f"{tag}_occupancy"] = p.occupancy
        out[f"{tag}_centers"] = p.block_centers
    for name, sel in plan.tables.items():
        out[f"plan_{name}"], out[f"plan_{name}_len"] = flat(sel.lists)
        out[f"table_{name}_len"] = ctx.tables[name].lengths
    # the four NSA uses on (LN'd) inputs with individual branch outputs
    xh = lsrm.layer_norm(x_up.features, np.ones(d, np.float32), np.zeros(d, np.float32))
    yh = lsrm.layer_norm(y_up.features, np.ones(d, np.float32), np.zeros(d, np.float32))
    uses = {"v2v": (xh, xh, pv, pv, w.nsa_x_self), "v2i": (xh, yh, pv, pi, w.nsa_x_cross),
            "i2i": (yh, yh, pi, pi, w.nsa_y_self), "i2v": (yh, xh, pi, pv, w.nsa_y_cross)}
    for name, (xq, xkv, pq, pkv, wu) in uses.items():
        o = lsrm.nsa_cross_attention(xq, xkv, pq, pkv, plan.tables[name], wu,
                                     params, table=ctx.tables[name])
        out[f"use_{name}"] = o
        n = xq.shape[0]
        q = affine(xq, wu.w_q).reshape(n, 8, 8)
        k = affine(xkv, wu.w_k).reshape(-1, 1, 8)
        v = affine(xkv, wu.w_v).reshape(-1, 1, 8)
        kc, vc_ = lsrm.compress_block_kv(k, v, pkv, wu.compress)
        out[f"kcmp_{name}"], out[f"vcmp_{name}"] = kc, vc_
        out[f"cmp_{name}"] = lsrm.cmp_attention(q, kc, vc_, params)
        own = pkv.block_of_token if wu.n_gates == 3 else None
        out[f"sel_{name}"] = lsrm.sel_attention(q, k, v, pkv, plan.tables[name],
                                                params, own_block=own)
        if wu.n_gates == 3:
            out[f"win_{name}"] = lsrm.win_attention(q, k, v, pq, pkv, params)
        out[f"gates_{name}_head"] = np.stack(nsa_gates(xq, wu))[:, :64]
        sc = lsrm.score_topk_blocks(q, kc, 4, params, pkv.occupied_ids)
        out[f"score_{name}"], out[f"score_{name}_len"] = flat(sc.lists)
    # sharding and the message log of the simulated parallel stage (1 layer)
    for W in (2, 3, 8):
        topo = lsrm.shard_blocks(pv, pi, W)
        out[f"shard{W}_loads"] = topo.loads
        out[f"shard{W}_vol"], out[f"shard{W}_vol_len"] = flat(topo.vol_rows)
        out[f"shard{W}_img"], out[f"shard{W}_img_len"] = flat(topo.img_rows)
    ctx_s = lsrm.build_sparse_context(pv, pi, selections=plan.tables)
    xs_p, ys_p, topo = lsrm.parallel_sparse_stage(x_up, y_up, [w], ctx_s, params, 3)
    out["par3_dev"] = np.array([np.abs(xs_p.astype(np.float64) - (x2 + x_up.features)).max()])
    out["par3_log"] = np.array(["%s,%s,%d,%d,%d" % r for r in topo.message_log])
    np.savez_compressed(os.path.join(HERE, "ref_c1.npz"), **out)


def ref_small():
    out = {}
    params = lsrm.AttentionParams(4, 2, 8)
    for seed in range(3):
        gt = rng.stream(seed, "test", "fix", "vol")
        coords = np.argwhere(gt.random((16, 16, 16)) < 0.05)
        feats = gt.standard_normal((coords.shape[0], 4)).astype(np.float32)
        toks = lsrm.TokenSet("volume", feats, coords, (16, 16, 16))
        part = lsrm.partition(toks)
        n = toks.count
        g = rng.stream(seed, "t_nsa")
        q = g.standard_normal((n, 4, 8)).astype(np.float32)
        k = g.standard_normal((n, 2, 8)).astype(np.float32)
        v = g.standard_normal((n, 2, 8)).astype(np.float32)
        g2 = rng.stream(seed, "t_sel_pick")
        lists = []
        for i in range(n):
            take = int(g2.integers(0 if i % 7 == 0 else 1, part.n_occupied + 1))
            rows = g2.choice(part.n_occupied, size=take, replace=False)
            lists.append(part.occupied_ids[rows])
        sel = lsrm.Selection(lists)
        own = part.block_of_token
        out[f"s{seed}_coords"] = coords
        out[f"s{seed}_q"], out[f"s{seed}_k"], out[f"s{seed}_v"] = q, k, v
        out[f"s{seed}_sel"], out[f"s{seed}_sel_len"] = flat(lists)
        out[f"s{seed}_out_sel"] = lsrm.sel_attention(q, k, v, part, sel, params, own_block=own)
        out[f"s{seed}_out_win"] = lsrm.win_attention(q, k, v, part, part, params)
        tab = lsrm.build_gather_table(sel, part, own_block=own)
        out[f"s{seed}_tab_ids"], out[f"s{seed}_tab_len"] = tab.ids, tab.lengths
    np.savez_compressed(os.path.join(HERE, "ref_small.npz"), **out)


def ref_goldenrun():
    import json
    gdir = "/root/reference/pkg/tests/goldens"
    cfg = lsrm.config_from_json(json.load(open(os.path.join(gdir, "config.json"))))
    cams, f = lsrm.scene_from_json(json.load(open(os.path.join(gdir, "scene.json"))))
    res = lsrm.run_pipeline(cfg, cams, f)
    np.savez_compressed(
        os.path.join(HERE, "ref_goldenrun.npz"),
        x_coords=res["x_up"].coords, x_grid=np.array(res["x_up"].grid_res),
        y_coords=res["y_up"].coords, y_grid=np.array(res["y_up"].grid_res),
        d=cfg.d, workers=cfg.workers, depth=cfg.depth_sparse, width=cfg.n_kv_heads * (cfg.d // cfg.n_q_heads))
    shutil.copy(os.path.join(gdir, "reference", "messages.csv"),
                os.path.join(HERE, "ref_goldenrun_messages.csv"))


def ref_decoded():
    """The reference's coarse-to-fine path with geometry_source="decoded"
    (`runner.py:301-335`) at the golden-run config: the decoded coarse SDF
    drives the informative-voxel mask and the image-token surface points."""
    import dataclasses
    import json
    gdir = "/root/reference/pkg/tests/goldens"
    cfg = lsrm.config_from_json(json.load(open(os.path.join(gdir, "config.json"))))
    cfg = dataclasses.replace(cfg, geometry_source="decoded")
    cams, f = lsrm.scene_from_json(json.load(open(os.path.join(gdir, "scene.json"))))
    res = lsrm.run_pipeline(cfg, cams, f)
    w = res["weights"]
    fv_coarse = lsrm.FeatureVolume(res["dense_grid"])
    from lsrm.camera_geometry import callable_field
    geo = callable_field(
        lambda pts: lsrm.decode_points(fv_coarse, w.heads, pts)[1].astype(np.float64))
    ic = lsrm.image_token_coords(res["y_up"], res["fine_cams"], geo, LAPLACE_BETA)
    (sw1, sb1, _), (sw2, sb2, _) = w.heads.s_layers
    plan = res["plan"]
    out = dict(
        seed=cfg.seed, d=cfg.d, heads=np.array([cfg.n_q_heads, cfg.n_kv_heads]),
        s_vol_fine=cfg.s_vol_fine, s_img_fine=cfg.s_img_fine,
        factor_vol=cfg.factor_vol, factor_img=cfg.factor_img, workers=cfg.workers,
        depth_sparse=cfg.depth_sparse,
        budgets=np.array([cfg.budgets.b_i, cfg.budgets.b_v2v, cfg.budgets.b_v2i,
                          cfg.budgets.b_i2v, cfg.budgets.b_i2i]),
        x_d=res["x_d"], y_d=res["y_d"], dense_grid=res["dense_grid"],
        s_w1=sw1, s_b1=sb1, s_w2=sw2, s_b2=sb2,
        vol_mask=res["vol_mask"], img_mask=res["img_mask"],
        cam_K=np.stack([c.intrinsics for c in res["fine_cams"]]),
        cam_R=np.stack([c.rotation for c in res["fine_cams"]]),
        cam_t=np.stack([c.translation for c in res["fine_cams"]]),
        cam_wh=np.array([c.image_size for c in res["fine_cams"]]),
        x_coords=res["x_up"].coords, y_coords=res["y_up"].coords,
        img_points=ic.points, img_miss=ic.miss,
        x_s=res["x_s"], y_s=res["y_s"],
        probe=res["probe"], probe_z=res["probe_z"], probe_s=res["probe_s"])
    for name, selx in plan.tables.items():
        out[f"plan_{name}"], out[f"plan_{name}_len"] = flat(selx.lists)
    np.savez_compressed(os.path.join(HERE, "ref_decoded.npz"), **out)
    lsrm.message_log_to_csv(res["topology"].message_log,
                            os.path.join(HERE, "ref_decoded_messages.csv"))
    print("decoded", int(res["vol_mask"].sum()), res["x_up"].count, res["y_up"].count)


if __name__ == "__main__":
    which = sys.argv[1:] or ["work", "small", "goldenrun", "decoded"]
    if "decoded" in which:
        ref_decoded()
    if "small" in which:
        ref_small()
    if "goldenrun" in which:
        ref_goldenrun()
    if "work" in which:
        c1 = workload("c1", **CONFIGS["c1"])
        ref_c1(*c1)
        workload("c3", **CONFIGS["c3"])
        workload("c4", **CONFIGS["c4"])
