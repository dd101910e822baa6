"""The reference API on the bf16 engines (`fastpath.py`, `dropin.install(...,
precision="bf16")`).

With precision "bf16", `nsa_cross_attention` (`lsrm/nsa_attention.py:287`),
`sparse_block_forward` (`lsrm/recon_pipeline.py:461`) and
`sparse_stage_forward` (`:500`) run on the tcgen05 engines. Checked against
the f64 oracle (the NSA uses) and against the package's fp32 reference-API
path (the block and the stage), at C1 geometry with paper heads (32/2/32,
d = 1024): rel-L2 <= 2e-2 (DESIGN.md tolerances). Also checked: the engine
cache re-uploads replaced or updated weights, score mode and unsupported
geometries stay on the fp32 path, and the native library is what ran.
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _rel(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / np.linalg.norm(want))


@pytest.fixture(scope="module")
def setup(cuda):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import recon_pipeline as R
    from paper_2604_05182_b200.workloads import coarse_inputs
    from fixtures import load_workload
    wl = load_workload("c1")
    params = L.AttentionParams(32, 2, 32)
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 1024)
    x_up, y_up = L.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v, pe_i,
                                          wl.factor_vol, wl.factor_img)
    pv, pi = L.partition(x_up), L.partition(y_up)
    plan = L.build_routing_plan(L.volume_token_coords(x_up), wl.img_points, pv, pi,
                                wl.cameras, L.RoutingBudgets())
    ctx = R.build_sparse_context(pv, pi, selections=plan.tables)
    ones, zeros = np.ones(1024, np.float32), np.zeros(1024, np.float32)
    xh = O.layer_norm(x_up.features, ones, zeros)
    yh = O.layer_norm(y_up.features, ones, zeros)
    return dict(L=L, R=R, params=params, x_up=x_up, y_up=y_up, pv=pv, pi=pi, plan=plan,
                ctx=ctx, xh=xh, yh=yh)


@pytest.fixture
def bf16():
    from paper_2604_05182_b200 import fastpath
    fastpath.set_precision("bf16")
    yield fastpath
    fastpath.set_precision("fp32")


@pytest.mark.parametrize("use", ["v2v", "v2i", "i2i", "i2v"])
def test_nsa_use_bf16_vs_oracle(setup, bf16, use):
    from paper_2604_05182_b200._native import launch_count, reset_launch_count
    s = setup
    L, R, params, ctx = s["L"], s["R"], s["params"], s["ctx"]
    xq, xkv, pq, pk = {"v2v": (s["xh"], s["xh"], s["pv"], s["pv"]),
                       "v2i": (s["xh"], s["yh"], s["pv"], s["pi"]),
                       "i2i": (s["yh"], s["yh"], s["pi"], s["pi"]),
                       "i2v": (s["yh"], s["xh"], s["pi"], s["pv"])}[use]
    ng = 3 if use in ("v2v", "i2i") else 2
    w = L.init_nsa_weights(0, params, ng, "dropin", use)
    reset_launch_count()
    got = L.nsa_cross_attention(xq, xkv, pq, pk, ctx.selections[use], w, params,
                                table=ctx.tables[use])
    assert launch_count() > 0
    assert any(k[0] == "use" for k in bf16._CACHE)   # the bf16 engine ran, not the fp32 path
    tok = {"v": s["x_up"], "i": s["y_up"]}
    oq = O.partition_tokens("volume" if use[0] == "v" else "image", tok[use[0]].coords,
                            tok[use[0]].grid_res)
    ok = O.partition_tokens("volume" if use[2] == "v" else "image", tok[use[2]].coords,
                            tok[use[2]].grid_res)
    ow = O.init_nsa_weights(0, O.AttentionParams(32, 2, 32), ng, "dropin", use)
    want = O.nsa_use(xq, xkv, oq, ok, s["plan"].tables[use].lists, ow, O.AttentionParams(32, 2, 32))
    rel = _rel(got, want)
    print(f"{use}: bf16 reference-API use vs f64 oracle rel-L2 {rel:.2e}")
    assert got.dtype == np.float32 and got.shape == want.shape
    assert rel < 2e-2


def test_engine_cache_sees_weight_updates(setup, bf16):
    s = setup
    L, params, ctx = s["L"], s["params"], s["ctx"]
    w = L.init_nsa_weights(0, params, 2, "dropin", "cache")
    a = L.nsa_cross_attention(s["xh"], s["yh"], s["pv"], s["pi"], ctx.selections["v2i"], w,
                              params, table=ctx.tables["v2i"])
    b = L.nsa_cross_attention(s["xh"], s["yh"], s["pv"], s["pi"], ctx.selections["v2i"], w,
                              params, table=ctx.tables["v2i"])
    assert np.array_equal(a, b)           # cached engine: deterministic, same bytes
    w.w_o *= 2.0                          # in-place update -> re-upload
    c = L.nsa_cross_attention(s["xh"], s["yh"], s["pv"], s["pi"], ctx.selections["v2i"], w,
                              params, table=ctx.tables["v2i"])
    assert _rel(c, 2.0 * a) < 1e-2


def test_unsupported_calls_stay_fp32(setup, bf16):
    """Score mode (no selection) and a self use whose key stream differs
    from its query stream are not engine calls: fp32 path, same result as
    with precision fp32."""
    s = setup
    L, params = s["L"], s["params"]
    w = L.init_nsa_weights(0, params, 2, "dropin", "score")
    got = L.nsa_cross_attention(s["xh"], s["yh"], s["pv"], s["pi"], None, w, params, b_sel=4)
    bf16.set_precision("fp32")
    want = L.nsa_cross_attention(s["xh"], s["yh"], s["pv"], s["pi"], None, w, params, b_sel=4)
    assert np.array_equal(got, want)


def test_sparse_block_and_stage_bf16(setup, bf16):
    s = setup
    R, params, ctx = s["R"], s["params"], s["ctx"]
    ws = [R.init_sparse_block(0, params, m) for m in range(2)]
    w = ws[0]
    x_up, y_up = s["x_up"], s["y_up"]
    g = np.random.default_rng(5)
    x = (g.standard_normal(x_up.features.shape) * 0.5).astype(np.float32)
    y = (g.standard_normal(y_up.features.shape) * 0.5).astype(np.float32)
    xi = (x_up.features.astype(np.float64) @ w.inj_x).astype(np.float32)
    yi = (y_up.features.astype(np.float64) @ w.inj_y).astype(np.float32)
    got = R.sparse_block_forward(x, y, xi, yi, w, ctx, params)
    assert any(k[0] == "block" for k in bf16._CACHE)
    got_stage = R.sparse_stage_forward(x_up, y_up, ws, ctx, params)
    assert any(k[0] == "stage" for k in bf16._CACHE)
    bf16.set_precision("fp32")
    want = R.sparse_block_forward(x, y, xi, yi, w, ctx, params)
    want_stage = R.sparse_stage_forward(x_up, y_up, ws, ctx, params)
    for name, gg, ww, base in (("x", got[0], want[0], x), ("y", got[1], want[1], y),
                               ("stage x", got_stage[0], want_stage[0], x_up.features),
                               ("stage y", got_stage[1], want_stage[1], y_up.features)):
        upd = _rel(np.asarray(gg, np.float64) - base, np.asarray(ww, np.float64) - base)
        print(f"bf16 {name}: update rel-L2 vs fp32 path {upd:.2e}")
        assert upd < 2e-2, (name, upd)


@pytest.mark.parametrize("W", [2, 3])
def test_parallel_sparse_stage_threads_bit_equal(setup, bf16, W):
    """precision bf16: `parallel_sparse_stage` (`lsrm/seq_parallel.py:321`)
    really runs W workers (threads, each a ShardedStage exchanging device
    buffers: dispatch all-to-all, per-use All-gather-KV, return all-to-all):
    bit-equal to the single-engine stage, dispatch / return bytes equal to
    the reference's all_to_all accounting."""
    s = setup
    L, R, params, ctx = s["L"], s["R"], s["params"], s["ctx"]
    from paper_2604_05182_b200 import seq_parallel as S
    ws = [R.init_sparse_block(0, params, m) for m in range(2)]
    x_up, y_up = s["x_up"], s["y_up"]
    xs, ys, topo = S.parallel_sparse_stage(x_up, y_up, ws, ctx, params, W)
    rx, ry = R.sparse_stage_forward(x_up, y_up, ws, ctx, params)
    assert np.array_equal(xs, rx) and np.array_equal(ys, ry)
    ref = S.WorkerTopology(W, [], [], [], [], np.zeros(W, np.int64))
    n = x_up.count + y_up.count
    aligned = [np.concatenate([topo.vol_tokens[w], topo.img_tokens[w] + x_up.count])
               for w in range(W)]
    naive = S.naive_contiguous_shards(n, W)
    S.all_to_all(naive, aligned, ref, "dispatch", 4 * 1024 + 12)
    got = sorted(e for e in topo.message_log if e[0] == "dispatch")
    assert got == sorted(ref.message_log)
    kv = [e for e in topo.message_log if e[1] == "all_gather_kv"]
    assert len(kv) == 2 * 4 * W * (W - 1)          # layers x uses x ordered pairs
