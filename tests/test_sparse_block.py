"""Stage-2 sparse block (recon_pipeline.py:461-497) on the GPU.

* Reference-API path (`recon_pipeline.sparse_block_forward`, fp32/f64) against
  the block output the reference itself produced (`ref_c1.npz` block_x /
  block_y, desk heads 8/1/8, d = 64): max-abs <= 1e-5, the reference's own
  golden tolerance.
* bf16 engine (`SparseBlockEngine`, paper heads 32/2/32, d = 1024, C1
  geometry) against the f64 oracle (`oracle.block.sparse_block_forward`):
  rel-L2 <= 2e-2 (DESIGN.md tolerances).
"""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import unflat

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1_tokens(cuda):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import coarse_inputs
    from fixtures import load_workload
    wl = load_workload("c1")
    out = {"wl": wl}
    for d in (64, 1024):
        x_d, y_d, pe_v, pe_i = coarse_inputs(wl, d)
        x_up, y_up = L.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v, pe_i,
                                              wl.factor_vol, wl.factor_img)
        out[d] = (x_up, y_up)
    x_up, y_up = out[64]
    out["pv"], out["pi"] = L.partition(x_up), L.partition(y_up)
    return out


def test_sparse_block_reference_api_vs_golden(c1_tokens, ref_c1):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import recon_pipeline as R
    params = L.AttentionParams(8, 1, 8)
    x_up, y_up = c1_tokens[64]
    pv, pi = c1_tokens["pv"], c1_tokens["pi"]
    sels = {n: L.Selection(unflat(ref_c1[f"plan_{n}"], ref_c1[f"plan_{n}_len"]))
            for n in R.TABLE_NAMES}
    ctx = R.build_sparse_context(pv, pi, selections=sels)
    w = R.init_sparse_block(0, params, 0)
    xi = x_up.features @ w.inj_x.astype(np.float64)
    yi = y_up.features @ w.inj_y.astype(np.float64)
    xi, yi = xi.astype(np.float32), yi.astype(np.float32)
    x2, y2 = R.sparse_block_forward(np.zeros_like(xi), np.zeros_like(yi), xi, yi, w, ctx, params)
    ex = np.max(np.abs(x2.astype(np.float64) - ref_c1["block_x"]))
    ey = np.max(np.abs(y2.astype(np.float64) - ref_c1["block_y"]))
    print(f"sparse block vs reference: max-abs x {ex:.2e} y {ey:.2e}")
    assert ex < 1e-5 and ey < 1e-5


def test_sparse_block_engine_vs_oracle(c1_tokens):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import _dev as D, _ops
    from paper_2604_05182_b200 import recon_pipeline as R
    params = L.AttentionParams(32, 2, 32)
    wl = c1_tokens["wl"]
    x_up, y_up = c1_tokens[1024]
    pv, pi = L.partition(x_up), L.partition(y_up)
    plan = L.build_routing_plan(L.volume_token_coords(x_up), wl.img_points, pv, pi,
                                wl.cameras, L.RoutingBudgets())
    w = R.init_sparse_block(0, params, 0)
    eng = R.SparseBlockEngine(pv, pi, plan.device_rows, w, params)
    g = np.random.default_rng(3)
    x = (g.standard_normal(x_up.features.shape) * 0.5).astype(np.float32)
    y = (g.standard_normal(y_up.features.shape) * 0.5).astype(np.float32)
    xi = (x_up.features.astype(np.float64) @ w.inj_x).astype(np.float32)
    yi = (y_up.features.astype(np.float64) @ w.inj_y).astype(np.float32)
    tv, ti = pv.dev("block_token_ids"), pi.dev("block_token_ids")
    bm = [_ops.gather_rows(D.dev(a), t) for a, t in ((x, tv), (y, ti), (xi, tv), (yi, ti))]
    x2b, y2b = eng.forward(*bm)
    x2, y2 = (torch.empty_like(x2b), torch.empty_like(y2b))
    _ops.scatter_rows(x2b, tv, x2)
    _ops.scatter_rows(y2b, ti, y2)
    ow = O.init_sparse_block(0, O.AttentionParams(32, 2, 32), 0)
    opv = O.partition_tokens("volume", x_up.coords, x_up.grid_res)
    opi = O.partition_tokens("image", y_up.coords, y_up.grid_res)
    sels = {n: plan.tables[n].lists for n in R.TABLE_NAMES}
    own = {"v2v": opv.block_of_token, "i2i": opi.block_of_token}
    kvp = {"v2v": opv, "v2i": opi, "i2v": opv, "i2i": opi}
    tables = {n: O.build_gather_table(sels[n], kvp[n], own_block=own.get(n)) for n in sels}
    ctx = {"part_vol": opv, "part_img": opi, "selections": sels, "tables": tables}
    rx, ry = O.sparse_block_forward(x, y, xi, yi, ow, ctx, O.AttentionParams(32, 2, 32))
    for name, got, ref, base in (("x", x2, rx, x), ("y", y2, ry, y)):
        got = D.host(got).astype(np.float64)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        # the block is residual: also check the update (output - input) alone
        upd = np.linalg.norm((got - base) - (ref - base)) / np.linalg.norm(ref - base)
        print(f"block engine {name}: rel-L2 {rel:.3e}, update rel-L2 {upd:.3e}")
        assert rel < 2e-2 and upd < 2e-2, (name, rel, upd)


def test_parallel_sparse_stage_matches_reference(c1_tokens, ref_c1):
    """`seq_parallel.parallel_sparse_stage` (reference API, W = 3): states
    vs the reference's serial block + residual, and the message log equal to
    the reference's own parallel run (`ref_c1.npz` par3_log)."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import recon_pipeline as R
    params = L.AttentionParams(8, 1, 8)
    x_up, y_up = c1_tokens[64]
    pv, pi = c1_tokens["pv"], c1_tokens["pi"]
    sels = {n: L.Selection(unflat(ref_c1[f"plan_{n}"], ref_c1[f"plan_{n}_len"]))
            for n in R.TABLE_NAMES}
    ctx = R.build_sparse_context(pv, pi, selections=sels)
    w = R.init_sparse_block(0, params, 0)
    xs, ys, topo = L.parallel_sparse_stage(x_up, y_up, [w], ctx, params, 3)
    want_x = (ref_c1["block_x"].astype(np.float64) + x_up.features).astype(np.float32)
    want_y = (ref_c1["block_y"].astype(np.float64) + y_up.features).astype(np.float32)
    assert np.max(np.abs(xs.astype(np.float64) - want_x)) < 1e-5
    assert np.max(np.abs(ys.astype(np.float64) - want_y)) < 1e-5
    assert ["%s,%s,%d,%d,%d" % r for r in topo.message_log] == list(ref_c1["par3_log"])


def test_sparse_stage_engine_vs_fp32_stage(c1_tokens):
    """Two-layer bf16 SparseStageEngine (shared work buffers) against the
    fp32 reference-API `sparse_stage_forward` on the same routing, paper
    heads at C1 geometry."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import _dev as D, _ops
    from paper_2604_05182_b200 import recon_pipeline as R
    params = L.AttentionParams(32, 2, 32)
    wl = c1_tokens["wl"]
    x_up, y_up = c1_tokens[1024]
    pv, pi = L.partition(x_up), L.partition(y_up)
    plan = L.build_routing_plan(L.volume_token_coords(x_up), wl.img_points, pv, pi,
                                wl.cameras, L.RoutingBudgets())
    ws = [R.init_sparse_block(0, params, m) for m in range(2)]
    eng = R.SparseStageEngine(pv, pi, plan.device_rows, ws, params)
    tv, ti = pv.dev("block_token_ids"), pi.dev("block_token_ids")
    xs_b, ys_b = eng.forward(_ops.gather_rows(D.dev(x_up.features), tv),
                             _ops.gather_rows(D.dev(y_up.features), ti))
    xs, ys = torch.empty_like(xs_b), torch.empty_like(ys_b)
    _ops.scatter_rows(xs_b, tv, xs)
    _ops.scatter_rows(ys_b, ti, ys)
    ctx = R.build_sparse_context(pv, pi, selections=plan.tables)
    rx, ry = R.sparse_stage_forward(x_up, y_up, ws, ctx, params)
    for name, got, ref, base in (("x", xs, rx, x_up.features), ("y", ys, ry, y_up.features)):
        got = D.host(got).astype(np.float64)
        ref = np.asarray(ref, np.float64)
        upd = np.linalg.norm((got - base) - (ref - base)) / np.linalg.norm(ref - base)
        print(f"stage engine {name}: update rel-L2 {upd:.3e}")
        assert upd < 2e-2, (name, upd)
