"""GPU parity of the CUDA path against the reference fixtures and the CPU oracle.

Bit-exact: masks, compaction (coords AND features), partition, routing lists
(tie order included), gather-table lengths.  Floating point: the fp32 path
within 1e-5 max-abs of the reference (its own bound); the bf16
tcgen05 path within rel-L2 <= 1e-2 and max-abs <= 2e-2 * max|ref| of the
f64 oracle on the same bf16-rounded inputs.
"""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import unflat

pytestmark = [pytest.mark.gpu, pytest.mark.filterwarnings("ignore::RuntimeWarning")]

SCENE = {"kind": "union", "parts": [
    {"kind": "sphere", "center": [0.42, 0.5, 0.55], "radius": 0.18},
    {"kind": "box", "center": [0.6, 0.45, 0.4], "half_sizes": [0.12, 0.12, 0.12]}]}


@pytest.fixture(scope="module")
def c1(cuda, ref_c1):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import coarse_inputs
    from fixtures import load_workload
    wl = load_workload("c1")
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 64)
    x_up, y_up = L.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v, pe_i,
                                          wl.factor_vol, wl.factor_img)
    pv, pi = L.partition(x_up), L.partition(y_up)
    return dict(wl=wl, x_up=x_up, y_up=y_up, pv=pv, pi=pi, x_d=x_d, y_d=y_d, pe_v=pe_v,
                pe_i=pe_i)


def test_masks_bit_exact(cuda, ref_c1):
    import paper_2604_05182_b200 as L
    from fixtures import load_workload
    m32 = L.informative_voxel_mask(SCENE, 32)
    want = np.unpackbits(ref_c1["mask32"])[:32 ** 3].astype(bool).reshape(32, 32, 32)
    assert np.array_equal(m32, want)
    z = np.load("tests/golden/workload_c3.npz")
    m96 = L.informative_voxel_mask(SCENE, 96)
    want96 = np.unpackbits(z["vol_mask_pure"])[:96 ** 3].astype(bool).reshape(96, 96, 96)
    assert np.array_equal(m96, want96)
    wl = load_workload("c1")
    alpha = np.unpackbits(np.load("tests/golden/workload_c1.npz")["alpha0"])[:768 * 768]
    alpha = alpha.reshape(768, 768).astype(np.float32)
    fg = L.foreground_patch_mask(alpha)
    assert np.array_equal(fg, wl.img_mask[0])
    assert np.array_equal(fg, O.foreground_patch_mask(alpha))
    # odd patch size goes through the generic kernel
    assert np.array_equal(L.foreground_patch_mask(alpha, patch=6),
                          O.foreground_patch_mask(alpha, patch=6))


def test_compaction_bit_exact_c1(c1, ref_c1):
    assert np.array_equal(c1["x_up"].coords, ref_c1["x_coords"])
    assert np.array_equal(c1["y_up"].coords, ref_c1["y_coords"])
    assert np.array_equal(c1["x_up"].features.view(np.uint32), ref_c1["x_up"].view(np.uint32))
    assert np.array_equal(c1["y_up"].features.view(np.uint32), ref_c1["y_up"].view(np.uint32))


def test_compaction_and_partition_c3(cuda):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import coarse_inputs
    from fixtures import load_workload
    wl = load_workload("c3")
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 1024)
    x_up, y_up = L.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v, pe_i,
                                          wl.factor_vol, wl.factor_img)
    ox, oy = O.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v.tables,
                                      pe_i.tables, wl.factor_vol, wl.factor_img)
    assert x_up.count == wl.n_vol == 16815 and y_up.count == wl.n_img == 10318
    assert np.array_equal(x_up.coords, ox.coords) and np.array_equal(y_up.coords, oy.coords)
    assert np.array_equal(x_up.features.view(np.uint32), ox.features.view(np.uint32))
    assert np.array_equal(y_up.features.view(np.uint32), oy.features.view(np.uint32))
    for tok, mod in ((x_up, "volume"), (y_up, "image")):
        got = L.partition(tok)
        want = O.partition_tokens(mod, tok.coords, tok.grid_res)
        for f in ("block_of_token", "occupied_ids", "block_offsets", "block_token_ids",
                  "occupancy", "block_centers"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), f


def test_partition_bit_exact_c1(c1, ref_c1):
    for tag, p in (("pv", c1["pv"]), ("pi", c1["pi"])):
        assert np.array_equal(p.block_of_token, ref_c1[f"{tag}_block_of_token"])
        assert np.array_equal(p.occupied_ids, ref_c1[f"{tag}_occupied"])
        assert np.array_equal(p.block_offsets, ref_c1[f"{tag}_offsets"])
        assert np.array_equal(p.block_token_ids, ref_c1[f"{tag}_token_ids"])
        assert np.array_equal(p.occupancy, ref_c1[f"{tag}_occupancy"])
        assert np.array_equal(p.block_centers, ref_c1[f"{tag}_centers"])


def _plan(c, wl):
    import paper_2604_05182_b200 as L
    return L.build_routing_plan(L.volume_token_coords(c["x_up"]), wl.img_points, c["pv"],
                                c["pi"], wl.cameras, L.RoutingBudgets())


def test_routing_bit_exact_c1(c1, ref_c1):
    plan = _plan(c1, c1["wl"])
    for name in ("v2v", "v2i", "i2v", "i2i"):
        want = unflat(ref_c1[f"plan_{name}"], ref_c1[f"plan_{name}_len"])
        got = plan.tables[name].lists
        assert len(got) == len(want)
        bad = [i for i, (a, b) in enumerate(zip(got, want)) if not np.array_equal(a, b)]
        assert not bad, (name, len(bad), bad[:5])


def test_routing_bit_exact_c3(cuda):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import coarse_inputs
    from fixtures import load_workload
    wl = load_workload("c3")
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 8)
    x_up, y_up = L.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v, pe_i,
                                          wl.factor_vol, wl.factor_img)
    c = dict(x_up=x_up, pv=L.partition(x_up), pi=L.partition(y_up))
    plan = _plan(c, wl)
    opv = O.partition_tokens("volume", x_up.coords, x_up.grid_res)
    opi = O.partition_tokens("image", y_up.coords, y_up.grid_res)
    vpts = (x_up.coords.astype(np.float64) + 0.5) / wl.s_vol
    want = O.build_routing_plan(vpts, wl.img_points, opv, opi, wl.cameras,
                                dict(b_i=16, b_v2v=8, b_v2i=8, b_i2v=8, b_i2i=8))
    for name in ("v2v", "v2i", "i2v", "i2i"):
        got = plan.tables[name].lists
        bad = [i for i, (a, b) in enumerate(zip(got, want.tables[name]))
               if not np.array_equal(a, b)]
        assert not bad, (name, len(bad))


def test_gather_table_c1(c1, ref_c1):
    import paper_2604_05182_b200 as L
    parts = {"v2v": c1["pv"], "i2v": c1["pv"], "v2i": c1["pi"], "i2i": c1["pi"]}
    for name in ("v2v", "v2i", "i2v", "i2i"):
        sel = L.Selection(unflat(ref_c1[f"plan_{name}"], ref_c1[f"plan_{name}_len"]))
        own = parts[name].block_of_token if name in ("v2v", "i2i") else None
        tab = L.build_gather_table(sel, parts[name], own_block=own)
        assert np.array_equal(tab.lengths, ref_c1[f"table_{name}_len"])
        otab = O.build_gather_table(sel.lists, O.partition_tokens(
            parts[name].modality, (c1["x_up"] if name[2] == "v" else c1["y_up"]).coords,
            (c1["x_up"] if name[2] == "v" else c1["y_up"]).grid_res), own_block=own)
        w = min(tab.ids.shape[1], otab.ids.shape[1])
        assert np.array_equal(tab.ids[:, :w] * tab.valid[:, :w], otab.ids[:, :w] * otab.valid[:, :w])


@pytest.mark.parametrize("seed", range(3))
def test_fp32_branches_small(cuda, ref_small, seed):
    import paper_2604_05182_b200 as L
    r = ref_small
    params = L.AttentionParams(4, 2, 8)
    coords = r[f"s{seed}_coords"]
    toks = L.TokenSet("volume", np.zeros((coords.shape[0], 4), np.float32), coords, (16,) * 3)
    part = L.partition(toks)
    q, k, v = r[f"s{seed}_q"], r[f"s{seed}_k"], r[f"s{seed}_v"]
    sel = L.Selection(unflat(r[f"s{seed}_sel"], r[f"s{seed}_sel_len"]))
    got = L.sel_attention(q, k, v, part, sel, params, own_block=part.block_of_token)
    err = np.max(np.abs(got.astype(np.float64) - r[f"s{seed}_out_sel"]))
    assert err < 1e-5, err
    w = L.win_attention(q, k, v, part, part, params)
    assert np.max(np.abs(w.astype(np.float64) - r[f"s{seed}_out_win"])) < 1e-5
    # caller-built GatherTable (explicit token ids) path
    tab = L.GatherTable(r[f"s{seed}_tab_ids"], r[f"s{seed}_tab_ids"] >= 0, r[f"s{seed}_tab_len"])
    g2 = L.sel_attention(q, k, v, part, None, params, table=tab)
    assert np.max(np.abs(g2.astype(np.float64) - r[f"s{seed}_out_sel"])) < 1e-5


def test_fp32_nsa_uses_c1(c1, ref_c1):
    """The four gated NSA uses at C1 (fp32 path) vs the reference, 1e-5."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import nsa_use_weights
    params = L.AttentionParams(8, 1, 8)
    ws = nsa_use_weights(params)
    d = 64
    ones, zeros = np.ones(d, np.float32), np.zeros(d, np.float32)
    xh = O.layer_norm(c1["x_up"].features, ones, zeros)
    yh = O.layer_norm(c1["y_up"].features, ones, zeros)
    pv, pi = c1["pv"], c1["pi"]
    uses = {"v2v": (xh, xh, pv, pv), "v2i": (xh, yh, pv, pi), "i2i": (yh, yh, pi, pi),
            "i2v": (yh, xh, pi, pv)}
    for name, (xq, xkv, pq, pkv) in uses.items():
        sel = L.Selection(unflat(ref_c1[f"plan_{name}"], ref_c1[f"plan_{name}_len"]))
        got = L.nsa_cross_attention(xq, xkv, pq, pkv, sel, ws[name], params)
        err = np.max(np.abs(got.astype(np.float64) - ref_c1[f"use_{name}"]))
        assert err < 1e-5, (name, err)
        # branch-level parity
        n = xq.shape[0]
        qq = O.affine(xq, ws[name].w_q).reshape(n, 8, 8)
        kk = O.affine(xkv, ws[name].w_k).reshape(-1, 1, 8)
        vv = O.affine(xkv, ws[name].w_v).reshape(-1, 1, 8)
        kc, vc = L.compress_block_kv(kk, vv, pkv, ws[name].compress)
        assert np.max(np.abs(kc - ref_c1[f"kcmp_{name}"])) < 1e-6
        assert np.max(np.abs(vc - ref_c1[f"vcmp_{name}"])) < 1e-6
        cm = L.cmp_attention(qq, ref_c1[f"kcmp_{name}"], ref_c1[f"vcmp_{name}"], params)
        assert np.max(np.abs(cm.astype(np.float64) - ref_c1[f"cmp_{name}"])) < 1e-5
        sc = L.score_topk_blocks(qq, ref_c1[f"kcmp_{name}"], 4, params, pkv.occupied_ids)
        want = unflat(ref_c1[f"score_{name}"], ref_c1[f"score_{name}_len"])
        bad = [i for i, (a, b) in enumerate(zip(sc.lists, want)) if not np.array_equal(a, b)]
        assert not bad, (name, len(bad))   # index output: bit-exact, tie order included


def test_fp32_nsa_uses_score_mode_c1(c1):
    """Score-mode routing (`recon_pipeline.py:457-458`: b_sel instead of a
    3D selection) through the whole use, vs the oracle's score-mode use."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import nsa_use_weights
    params = L.AttentionParams(8, 1, 8)
    ws = nsa_use_weights(params)
    ows = {n: O.NsaWeights(w.w_q, w.w_k, w.w_v, w.w_o, w.gate_w, w.gate_b,
                           ((w.compress.for_k.w1, w.compress.for_k.b1, w.compress.for_k.w2,
                             w.compress.for_k.b2),
                            (w.compress.for_v.w1, w.compress.for_v.b1, w.compress.for_v.w2,
                             w.compress.for_v.b2)), w.n_gates) for n, w in ws.items()}
    d = 64
    ones, zeros = np.ones(d, np.float32), np.zeros(d, np.float32)
    xh = O.layer_norm(c1["x_up"].features, ones, zeros)
    yh = O.layer_norm(c1["y_up"].features, ones, zeros)
    pv, pi = c1["pv"], c1["pi"]
    opv = O.partition_tokens("volume", c1["x_up"].coords, c1["x_up"].grid_res)
    opi = O.partition_tokens("image", c1["y_up"].coords, c1["y_up"].grid_res)
    uses = {"v2v": (xh, xh, pv, pv, opv, opv), "v2i": (xh, yh, pv, pi, opv, opi),
            "i2i": (yh, yh, pi, pi, opi, opi), "i2v": (yh, xh, pi, pv, opi, opv)}
    for name, (xq, xkv, pq, pkv, oq, okv) in uses.items():
        got = L.nsa_cross_attention(xq, xkv, pq, pkv, None, ws[name], params, b_sel=4)
        want = O.nsa_use(xq, xkv, oq, okv, None, ows[name], O.AttentionParams(8, 1, 8),
                         b_sel=4)
        err = np.max(np.abs(got.astype(np.float64) - want))
        assert err < 1e-5, (name, err)


def _bf(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def test_tc_fused_attention_vs_oracle(c1):
    """bf16 tcgen05 fused cmp+sel+win+gates vs the f64 oracle on identical
    bf16-rounded inputs, paper heads 32/2/32 on the C1 token sets."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import _dev as D, _ops
    from paper_2604_05182_b200._native import call
    from paper_2604_05182_b200.engine import (block_major_rows, query_tiles, stream_meta)
    params = L.AttentionParams(32, 2, 32)
    wl = c1["wl"]
    plan = _plan(c1, wl)
    pv, pi = c1["pv"], c1["pi"]
    g = np.random.default_rng(5)
    for name, pq, pk, self_use in (("v2v", pv, pv, True), ("i2v", pi, pv, False),
                                   ("i2i", pi, pi, True), ("v2i", pv, pi, False)):
        nq, nk, B = pq.n_tokens, pk.n_tokens, pk.n_occupied
        ng = 3 if self_use else 2
        q = _bf(g.standard_normal((nq, 32, 32)))
        k = _bf(g.standard_normal((nk, 2, 32)))
        v = _bf(g.standard_normal((nk, 2, 32)))
        kc = _bf(g.standard_normal((B, 2, 32)) * 0.5)
        vc = _bf(g.standard_normal((B, 2, 32)))
        gl = _bf(g.standard_normal((nq, ng * 1024)))
        gb = (g.standard_normal(ng * 1024) * 0.1).astype(np.float32)
        # oracle (token order)
        lists = plan.tables[name].lists
        own = pk.block_of_token if self_use else None
        opk = O.partition_tokens(pk.modality, (c1["x_up"] if pk is pv else c1["y_up"]).coords,
                                 (c1["x_up"] if pk is pv else c1["y_up"]).grid_res)
        outs = [O.cmp_attention(q, kc, vc, O.AttentionParams(32, 2, 32)),
                O.sel_attention(q, k, v, opk, lists, O.AttentionParams(32, 2, 32), own)]
        if self_use:
            outs.append(O.win_attention(q, k, v, opk, O.AttentionParams(32, 2, 32)))
        z = gl.astype(np.float64) + gb.astype(np.float64)
        gate = 1.0 / (1.0 + np.exp(-z))
        ref = sum(gate[:, b * 1024:(b + 1) * 1024] * outs[b].reshape(nq, 1024).astype(np.float64)
                  for b in range(ng))
        # device call in block-major order
        mq, mk = stream_meta(pq), stream_meta(pk)
        tokq = pq.dev("block_token_ids")
        q_bm = _ops.gather_rows(D.dev(q.reshape(nq, 1024), torch.bfloat16), tokq)
        gl_bm = _ops.gather_rows(D.dev(gl, torch.bfloat16), tokq)
        kil = D.empty((2, mk.n_rows_pad, 32), torch.bfloat16)
        vil = D.empty((2, mk.n_rows_pad, 48), torch.bfloat16)
        st = D.stream()
        for src, dst, ones in ((k, kil, 0), (v, vil, 16)):
            s = D.dev(src.reshape(nk, 64), torch.bfloat16)
            call("lsrm_kv_interleave", 1, s.data_ptr(), 64, nk, 2, 32, ones,
                 pk.dev("block_token_ids").data_ptr(), mk.kv_off.data_ptr(), B,
                 mk.pad_off.data_ptr(), mk.n_rows_pad, dst.data_ptr(), st)
        bpad = (B + 15) // 16 * 16
        kcil = D.empty((2, bpad, 32), torch.bfloat16)
        vcil = D.empty((2, bpad, 48), torch.bfloat16)
        for src, dst, ones in ((kc, kcil, 0), (vc, vcil, 16)):
            s = D.dev(src.reshape(B, 64), torch.float32)
            call("lsrm_kv_interleave", 0, s.data_ptr(), 64, B, 2, 32, ones, None, None, 0, None,
                 bpad, dst.data_ptr(), st)
        rows, cnt = plan.device_rows[name]
        rb, cb = block_major_rows(rows, cnt, pq, pk, self_use)
        tiles = D.dev(query_tiles(pq, 16, self_use))
        merged = D.empty((nq, 1024), torch.bfloat16)
        gb_d = D.dev(gb)
        call("lsrm_nsa_attention_tc", q_bm.data_ptr(), 1024, nq, 32, 2, 32, kil.data_ptr(),
             vil.data_ptr(), mk.pad_off.data_ptr(), mk.kv_off.data_ptr(), mk.n_rows_pad,
             kcil.data_ptr(), vcil.data_ptr(), B, tiles.data_ptr(), int(tiles.shape[0]),
             rb.data_ptr(), cb.data_ptr(), int(rb.shape[1]), gl_bm.data_ptr(), ng * 1024, 0,
             gb_d.data_ptr(), ng, merged.data_ptr(), st)
        out = torch.empty_like(merged)
        _ops.scatter_rows(merged, tokq, out)
        got = out.float().cpu().numpy().astype(np.float64)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        mx = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
        print(f"{name}: rel-L2 {rel:.3e} max-abs/max {mx:.3e}")
        assert rel < 1e-2 and mx < 2e-2, (name, rel, mx)


@pytest.mark.parametrize("heads", [(32, 2, 32), (16, 2, 64), (16, 4, 32)])
def test_engine_layer_vs_fp32_path(c1, heads):
    """Whole bf16 layer (4 uses: GEMMs + compression + fused attention + W_o)
    vs the fp32 reference-API path on the same inputs: paper heads, head_dim
    64 (one pipeline per CTA) and group size 4 (32-token query tiles)."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import _dev as D, _ops
    from paper_2604_05182_b200.engine import SparseLayerEngine, USES
    from paper_2604_05182_b200.workloads import coarse_inputs, nsa_use_weights
    params = L.AttentionParams(*heads)
    wl = c1["wl"]
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, params.model_dim)
    x_up, y_up = L.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v, pe_i,
                                          wl.factor_vol, wl.factor_img)
    pv, pi = L.partition(x_up), L.partition(y_up)
    plan = L.build_routing_plan(L.volume_token_coords(x_up), wl.img_points, pv, pi,
                                wl.cameras, L.RoutingBudgets())
    ws = nsa_use_weights(params)
    g = np.random.default_rng(11)
    for wu in ws.values():   # nonzero gate biases: the engine folds them into its GEMM
        wu.gate_b = (g.standard_normal(wu.gate_b.shape) * 0.5).astype(np.float32)
    d = params.model_dim
    ones, zeros = np.ones(d, np.float32), np.zeros(d, np.float32)
    xh = O.layer_norm(x_up.features, ones, zeros)
    yh = O.layer_norm(y_up.features, ones, zeros)
    eng = SparseLayerEngine(pv, pi, plan.device_rows, ws, params)
    x_bm = _ops.gather_rows(D.dev(xh, torch.bfloat16), pv.dev("block_token_ids"))
    y_bm = _ops.gather_rows(D.dev(yh, torch.bfloat16), pi.dev("block_token_ids"))
    outs = eng.forward(x_bm, y_bm)
    parts = {"v2v": (xh, xh, pv, pv), "v2i": (xh, yh, pv, pi), "i2i": (yh, yh, pi, pi),
             "i2v": (yh, xh, pi, pv)}
    for use in USES:
        xq, xkv, pq, pk = parts[use]
        ref = L.nsa_cross_attention(xq, xkv, pq, pk, plan.tables[use], ws[use], params)
        o = torch.empty((pq.n_tokens, d), dtype=torch.bfloat16, device="cuda")
        _ops.scatter_rows(outs[use], pq.dev("block_token_ids"), o)
        got = o.float().cpu().numpy().astype(np.float64)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        print(f"engine {use}: rel-L2 {rel:.3e}")
        assert rel < 2e-2, (use, rel)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_engine_layer_vs_fp32_path_full_size(cuda, name):
    """The bf16 layer at BASELINE sizes (C3; C4 with twelve fully occupied
    512-token volume blocks, the maximum block size) against the fp32
    reference-API path on the same inputs and routing, every use."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.engine import USES
    from paper_2604_05182_b200.layer import SparseAttentionLayer, build_instance
    inst = build_instance(name)
    layer = SparseAttentionLayer(inst)
    outs = layer.forward_host(inst.x_hat, inst.y_hat)
    pv, pi = inst.part_vol, inst.part_img
    parts = {"v2v": (inst.x_hat, inst.x_hat, pv, pv), "v2i": (inst.x_hat, inst.y_hat, pv, pi),
             "i2i": (inst.y_hat, inst.y_hat, pi, pi), "i2v": (inst.y_hat, inst.x_hat, pi, pv)}
    from paper_2604_05182_b200.block_routing import _rows_to_selection
    for use in USES:
        xq, xkv, pq, pk = parts[use]
        sel = _rows_to_selection(*inst.plan_rows[use], pk)
        ref = L.nsa_cross_attention(xq, xkv, pq, pk, sel, inst.weights[use], inst.params)
        got = np.asarray(outs[use], np.float64)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        print(f"{name} engine {use}: rel-L2 {rel:.3e}")
        assert rel < 2e-2, (use, rel)


def test_routing_bit_exact_c5_sample(cuda):
    """Maximum size (C5: 333K volume + 99K image tokens, workload generated on
    the GPU): the four routing tables for a strided sample of queries equal
    the oracle's (bit-exact f64 distances, stable ties)."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import coarse_inputs, load_workload
    wl = load_workload("c5")
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 8)
    x_up, y_up = L.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v, pe_i,
                                          wl.factor_vol, wl.factor_img)
    c = dict(x_up=x_up, pv=L.partition(x_up), pi=L.partition(y_up))
    plan = _plan(c, wl)
    opv = O.partition_tokens("volume", x_up.coords, x_up.grid_res)
    opi = O.partition_tokens("image", y_up.coords, y_up.grid_res)
    assert np.array_equal(c["pv"].occupied_ids, opv.occupied_ids)
    assert np.array_equal(c["pi"].occupied_ids, opi.occupied_ids)
    vpts = (x_up.coords.astype(np.float64) + 0.5) / wl.s_vol
    ipts = np.asarray(wl.img_points, np.float64)
    sv = np.arange(0, vpts.shape[0], max(1, vpts.shape[0] // 192))
    si = np.arange(0, ipts.shape[0], max(1, ipts.shape[0] // 192))
    want = {"v2v": O.route_volume(vpts[sv], opv, 8), "i2v": O.route_volume(ipts[si], opv, 8),
            "v2i": O.route_image(vpts[sv], wl.cameras, opi, ipts, 16, 8),
            "i2i": O.route_image(ipts[si], wl.cameras, opi, ipts, 16, 8)}
    for name, idx in (("v2v", sv), ("i2v", si), ("v2i", sv), ("i2i", si)):
        got = [plan.tables[name].lists[i] for i in idx]
        bad = [k for k, (a, b) in enumerate(zip(got, want[name])) if not np.array_equal(a, b)]
        assert not bad, (name, len(bad), len(idx))


def _oracle_part(p):
    return O.Partition(p.modality, p.block_size, tuple(p.block_grid), p.n_blocks_total,
                       p.block_of_token, p.occupied_ids, p.block_offsets, p.block_token_ids,
                       p.occupancy, p.block_centers, p.block_views)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_engine_layer_vs_oracle_full_size_sample(cuda, name):
    """The headline layer at BASELINE size (C3; C4 with its 512-token blocks)
    checked directly against the f64 oracle: every use, a strided ~2K-query
    sample against the FULL key/value side (oracle/sample.py).  Inputs are
    the same LN'd f32 tokens, routing and weights (the reference's tagged
    init).  Bar: rel-L2 <= 1e-2, max-abs <= 2e-2 * max|ref|."""
    from oracle.sample import nsa_use_rows, strided_sample
    from paper_2604_05182_b200.block_routing import _rows_to_selection
    from paper_2604_05182_b200.engine import USES
    from paper_2604_05182_b200.layer import SparseAttentionLayer, build_instance
    inst = build_instance(name)
    layer = SparseAttentionLayer(inst)
    outs = layer.forward_host(inst.x_hat, inst.y_hat)
    pv, pi = inst.part_vol, inst.part_img
    opv, opi = _oracle_part(pv), _oracle_part(pi)
    ow = O.init_sparse_block(0, O.AttentionParams(32, 2, 32), 0).nsa
    parts = {"v2v": (inst.x_hat, inst.x_hat, opv, opv, pv),
             "v2i": (inst.x_hat, inst.y_hat, opv, opi, pi),
             "i2i": (inst.y_hat, inst.y_hat, opi, opi, pi),
             "i2v": (inst.y_hat, inst.x_hat, opi, opv, pv)}
    for use in USES:
        xq, xkv, oq, ok, pk = parts[use]
        lists = _rows_to_selection(*inst.plan_rows[use], pk).lists
        qids = strided_sample(xq.shape[0], 2048)
        ref = nsa_use_rows(xq, xkv, oq, ok, lists, ow[use], O.AttentionParams(32, 2, 32), qids)
        ref = np.asarray(ref, np.float64)
        got = np.asarray(outs[use], np.float64)[qids]
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        mx = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
        print(f"{name} {use} ({qids.size} queries vs f64 oracle): rel-L2 {rel:.3e} "
              f"max-abs/max|ref| {mx:.3e}")
        assert rel <= 1e-2 and mx <= 2e-2, (use, rel, mx)


@pytest.mark.parametrize("heads", [(32, 2, 32), (8, 1, 8), (4, 2, 3), (6, 3, 5)])
def test_score_topk_bit_exact_vs_einsum(cuda, heads):
    """score_topk_blocks ranks by the same f64 scores NumPy's einsum produces
    (its summation order restated in the kernel): lists bit-exact against the
    oracle (np.einsum + stable argsort) on random data, with exact ties
    (duplicated compressed rows) and near-ties (coarsely quantised inputs)."""
    import paper_2604_05182_b200 as L
    hq, hkv, dh = heads
    params = L.AttentionParams(hq, hkv, dh)
    g = np.random.default_rng(hq * 100 + dh)
    for quant in (None, 0.25):
        q = g.standard_normal((700, hq, dh)).astype(np.float32)
        kc = g.standard_normal((61, hkv, dh)).astype(np.float32)
        if quant:
            q = (np.round(q / quant) * quant).astype(np.float32)
            kc = (np.round(kc / quant) * quant).astype(np.float32)
        kc[7] = kc[3]
        kc[40] = kc[3]
        ids = np.sort(g.choice(5000, 61, replace=False)).astype(np.int64)
        got = L.score_topk_blocks(q, kc, 8, params, ids).lists
        want = O.score_topk_blocks(q, kc, 8, O.AttentionParams(hq, hkv, dh), ids)
        bad = [i for i, (a, b) in enumerate(zip(got, want)) if not np.array_equal(a, b)]
        assert not bad, (heads, quant, len(bad))
