"""Block-aware sequence parallelism (`lsrm/seq_parallel.py`; reference tests
`pkg/tests/test_seq_parallel.py`).

CPU: sharding + message log against the reference's golden vectors, the
collectives' ProtocolError behaviour, the routed-workload LPT, the
canonical-placement segments, and a world_size-2 gloo all-gather-v of packed
KV shards.  GPU: W emulated ranks (in-process transport) reproduce the
unsharded engine's layer output row for row.
"""

import csv
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
from conftest import GOLDEN, golden, unflat
from paper_2604_05182_b200 import seq_parallel as S
from paper_2604_05182_b200.errors import ConfigurationError, ProtocolError


@pytest.fixture(scope="module")
def c1_parts():
    from paper_2604_05182_b200.workloads import coarse_inputs
    from fixtures import load_workload
    wl = load_workload("c1")
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 64)
    x_up, y_up = O.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v.tables,
                                          pe_i.tables, wl.factor_vol, wl.factor_img)
    return (O.partition_tokens("volume", x_up.coords, x_up.grid_res),
            O.partition_tokens("image", y_up.coords, y_up.grid_res))


def _bare(n):
    return S.WorkerTopology(n, [], [], [], [], np.zeros(n, np.int64))


# ---------------------------------------------------------------------------
# sharding


def test_shard_blocks_matches_reference(ref_c1, c1_parts):
    pv, pi = c1_parts
    for W in (2, 3, 8):
        topo = S.shard_blocks(pv, pi, W)
        assert np.array_equal(topo.loads, ref_c1[f"shard{W}_loads"])
        want_v = unflat(ref_c1[f"shard{W}_vol"], ref_c1[f"shard{W}_vol_len"])
        want_i = unflat(ref_c1[f"shard{W}_img"], ref_c1[f"shard{W}_img_len"])
        assert all(np.array_equal(a, b) for a, b in zip(topo.vol_rows, want_v))
        assert all(np.array_equal(a, b) for a, b in zip(topo.img_rows, want_i))
        # every occupied block exactly once; tokens tile both streams
        assert np.array_equal(np.sort(np.concatenate(topo.vol_rows)), np.arange(pv.n_occupied))
        assert np.array_equal(np.sort(np.concatenate(topo.vol_tokens)), np.arange(pv.n_tokens))
        assert np.array_equal(np.sort(np.concatenate(topo.img_tokens)), np.arange(pi.n_tokens))


def test_zero_workers_rejected(c1_parts):
    with pytest.raises(ConfigurationError):
        S.shard_blocks(*c1_parts, 0)


def test_assignment_map(c1_parts):
    pv, pi = c1_parts
    topo = S.shard_blocks(pv, pi, 3)
    amap = topo.assignment(pv, "volume")
    for w in range(3):
        assert (amap[pv.occupied_ids[topo.vol_rows[w]]] == w).all()
    occupied = np.zeros(pv.n_blocks_total, bool)
    occupied[pv.occupied_ids] = True
    assert (amap[~occupied] == -1).all()


def test_cost_lpt_balances_routed_workload(c1_parts):
    pv, pi = c1_parts
    rng = np.random.default_rng(0)
    lengths = {u: rng.integers(0, 400, n).astype(np.float64) for u, n in
               (("v2v", pv.n_tokens), ("v2i", pv.n_tokens), ("i2i", pi.n_tokens),
                ("i2v", pi.n_tokens))}
    cv, ci = S.block_costs(pv, pi, lengths)
    for W in (2, 4, 8):
        topo = S.shard_blocks_by_cost(pv, pi, W, cv, ci)
        loads = np.array([cv[topo.vol_rows[w]].sum() + ci[topo.img_rows[w]].sum()
                          for w in range(W)])
        assert np.allclose(loads, topo.loads)
        assert np.isclose(loads.sum(), cv.sum() + ci.sum())
        # greedy LPT guarantee: makespan <= mean + largest item
        assert loads.max() <= loads.mean() + max(cv.max(), ci.max()) + 1e-6
        assert np.array_equal(np.sort(np.concatenate(topo.img_rows)), np.arange(pi.n_occupied))


def test_naive_shards_and_makespan(c1_parts):
    sh = S.naive_contiguous_shards(10, 3)
    assert [s.tolist() for s in sh] == [[0, 1, 2], [3, 4, 5], [6, 7, 8, 9]]
    assert S.makespan_ratio(np.array([0, 0]), 2) == 1.0
    rep = S.imbalance_report([c1_parts], 4)[0]
    assert rep["ratio_block_aware"] <= rep["ratio_naive"] + 1e-12
    assert rep["ratio_block_aware"] >= 1.0


# ---------------------------------------------------------------------------
# collectives (reference API: accounting + invariant checks)


def test_identity_reshard_logs_nothing():
    topo = _bare(2)
    sh = S.naive_contiguous_shards(6, 2)
    S.all_to_all(sh, [s.copy() for s in sh], topo, "p", 4)
    assert topo.message_log == []


@pytest.mark.parametrize("shin,shout", [
    ([[0, 1], [1, 2]], [[0, 1], [1, 2]]),      # produced twice
    ([[0], [1]], [[0], [5]]),                  # never produced
    ([[0, 1], [2]], [[0], [2]]),               # dropped
])
def test_all_to_all_protocol_errors(shin, shout):
    with pytest.raises(ProtocolError):
        S.all_to_all([np.array(s) for s in shin], [np.array(s) for s in shout], _bare(2), "p", 4)


def test_all_to_all_shard_count_checked():
    with pytest.raises(ConfigurationError):
        S.all_to_all([np.array([0])], [np.array([0])], _bare(2), "p", 4)


def _kv_parts(n_blocks, n_tokens, width, seed):
    r = np.random.default_rng(seed)
    rows = np.array_split(r.permutation(n_blocks), 2)
    toks = np.array_split(r.permutation(n_tokens), 2)
    return [{"k": np.repeat(tt[:, None], width, 1).astype(np.float32),
             "v": 2.0 * np.repeat(tt[:, None], width, 1).astype(np.float32),
             "k_cmp": np.repeat(rr[:, None], width, 1).astype(np.float32),
             "v_cmp": 3.0 * np.repeat(rr[:, None], width, 1).astype(np.float32),
             "token_ids": tt, "block_rows": rr} for rr, tt in zip(rows, toks)]


def test_all_gather_kv_canonical_order_and_bytes():
    parts = _kv_parts(5, 9, 4, 0)
    topo = _bare(2)
    k, v, kc, vc = S.all_gather_kv(parts, topo, "p")
    assert np.array_equal(k[:, 0], np.arange(9)) and np.array_equal(v[:, 0], 2 * np.arange(9))
    assert np.array_equal(kc[:, 0], np.arange(5)) and np.array_equal(vc[:, 0], 3 * np.arange(5))
    for _, kind, src, dst, nb in topo.message_log:
        assert kind == "all_gather_kv" and src != dst
        assert nb == 4 * 2 * (parts[src]["k"].size + parts[src]["k_cmp"].size)


def test_all_gather_kv_ownership_errors():
    parts = _kv_parts(5, 9, 4, 2)
    parts[1]["block_rows"] = parts[0]["block_rows"].copy()
    with pytest.raises(ProtocolError):
        S.all_gather_kv(parts, _bare(2), "p")
    parts = _kv_parts(5, 9, 4, 3)
    parts[0]["token_ids"] = parts[0]["token_ids"] + 100
    with pytest.raises(ProtocolError):
        S.all_gather_kv(parts, _bare(2), "p")


def _stage_log(pv, pi, W, d, width, depth):
    """The reference parallel stage's message log through this package's API."""
    topo = S.shard_blocks(pv, pi, W)
    n_x = pv.n_tokens
    aligned = [np.concatenate([topo.vol_tokens[w], topo.img_tokens[w] + n_x]) for w in range(W)]
    naive = S.naive_contiguous_shards(n_x + pi.n_tokens, W)
    S.all_to_all(naive, aligned, topo, "dispatch", 4 * d + S.TOKEN_COORD_BYTES)
    for m in range(depth):
        for name, kv_vol, is_self in (("v2v", True, True), ("v2i", False, False),
                                      ("i2i", False, True), ("i2v", True, False)):
            toks = topo.vol_tokens if kv_vol else topo.img_tokens
            rows = topo.vol_rows if kv_vol else topo.img_rows
            parts = [{"k": np.zeros((t.size, width), np.float32),
                      "v": np.zeros((t.size, width), np.float32),
                      "k_cmp": np.zeros((r.size, width), np.float32),
                      "v_cmp": np.zeros((r.size, width), np.float32),
                      "token_ids": t, "block_rows": r} for t, r in zip(toks, rows)]
            S.all_gather_kv(parts, topo, f"layer{m}/{name}")
            if is_self:
                for w in range(W):
                    topo.log(f"layer{m}/{name}/win", "window", w, w, 0)
    S.all_to_all(aligned, naive, topo, "return", 4 * d + S.TOKEN_COORD_BYTES)
    return topo.message_log


def test_golden_run_messages_csv_byte_identical(tmp_path):
    z = golden("ref_goldenrun.npz")
    pv = O.partition_tokens("volume", z["x_coords"], tuple(z["x_grid"]))
    pi = O.partition_tokens("image", z["y_coords"], tuple(z["y_grid"]))
    log = _stage_log(pv, pi, int(z["workers"]), int(z["d"]), int(z["width"]), int(z["depth"]))
    out = tmp_path / "messages.csv"
    S.message_log_to_csv(log, out)
    with open(os.path.join(GOLDEN, "ref_goldenrun_messages.csv"), "rb") as fh:
        want = fh.read()
    assert out.read_bytes() == want


def test_c1_parallel_message_log(ref_c1, c1_parts):
    log = _stage_log(*c1_parts, 3, 64, 8, 1)
    assert ["%s,%s,%d,%d,%d" % r for r in log] == list(ref_c1["par3_log"])


# ---------------------------------------------------------------------------
# All-gather-KV data path: placement segments + gloo transport


def _canonical(occ, hkv, dh, w, seed):
    """Random global KV buffers in the engine's canonical byte layout, and
    each block's rows (padded rows zero)."""
    from paper_2604_05182_b200.engine import ONES_COLS, ROW_PAD
    rng = np.random.default_rng(seed)
    pad = (occ + ROW_PAD - 1) // ROW_PAD * ROW_PAD
    po = np.concatenate([[0], np.cumsum(pad)]).astype(np.int64)
    R = int(po[-1])
    k = np.zeros((hkv, R, dh), np.uint16)
    v = np.zeros((hkv, R, dh + ONES_COLS), np.uint16)
    for b in range(occ.size):
        k[:, po[b]:po[b] + occ[b]] = rng.integers(1, 65535, (hkv, occ[b], dh))
        v[:, po[b]:po[b] + occ[b]] = rng.integers(1, 65535, (hkv, occ[b], dh + ONES_COLS))
    kc = rng.standard_normal((occ.size, w)).astype(np.float32)
    vc = rng.standard_normal((occ.size, w)).astype(np.float32)
    return po, R, k, v, kc, vc


def _pack(rows, occ, po, k, v, kc, vc, hkv, dh, w):
    """What rank-local kv_prepare writes: the owned blocks, compact."""
    from paper_2604_05182_b200.engine import ONES_COLS, ROW_PAD, PackedShard
    rows = np.sort(rows)
    pad = (occ[rows] + ROW_PAD - 1) // ROW_PAD * ROW_PAD
    lpo = np.concatenate([[0], np.cumsum(pad)]).astype(np.int64)
    lay = PackedShard(hkv, dh, w, int(lpo[-1]), rows.size)
    kl = np.zeros((hkv, lay.rows_pad, dh), np.uint16)
    vl = np.zeros((hkv, lay.rows_pad, dh + ONES_COLS), np.uint16)
    kcl = np.zeros((lay.n_blocks, w), np.float32)
    vcl = np.zeros((lay.n_blocks, w), np.float32)
    for j, b in enumerate(rows):
        n = po[b + 1] - po[b]
        kl[:, lpo[j]:lpo[j] + n] = k[:, po[b]:po[b] + n]
        vl[:, lpo[j]:lpo[j] + n] = v[:, po[b]:po[b] + n]
        kcl[j], vcl[j] = kc[b], vc[b]
    buf = np.concatenate([a.view(np.uint8).ravel() for a in (kl, vl, kcl, vcl)])
    assert buf.size == lay.total
    return buf


def _place_all(stage, occ, po, R, shard_rows, hkv, dh, w):
    from paper_2604_05182_b200.engine import ONES_COLS
    offs, seg = S.placement_segments(occ, po, R, shard_rows, hkv, dh, w)
    out = {"k": np.zeros(hkv * R * dh * 2, np.uint8),
           "v": np.zeros(hkv * R * (dh + ONES_COLS) * 2, np.uint8),
           "kc": np.zeros(occ.size * w * 4, np.uint8), "vc": np.zeros(occ.size * w * 4, np.uint8)}
    for kind in out:
        S.apply_segments(stage, out[kind], seg[kind])
    return offs, out


@pytest.mark.parametrize("W", [1, 2, 3, 5])
def test_placement_segments_reassemble_canonical_layout(W):
    rng = np.random.default_rng(W)
    occ = rng.integers(1, 40, 23).astype(np.int64)
    hkv, dh, w = 2, 32, 64
    po, R, k, v, kc, vc = _canonical(occ, hkv, dh, w, W)
    owner = rng.integers(0, W, occ.size)
    owner[0] = W - 1                           # and leave rank 0 possibly empty
    shard_rows = [np.flatnonzero(owner == r) for r in range(W)]
    packs = [_pack(r, occ, po, k, v, kc, vc, hkv, dh, w) for r in shard_rows]
    offs, seg = S.placement_segments(occ, po, R, shard_rows, hkv, dh, w)
    assert [int(p.size) for p in packs] == list(np.diff(offs))
    stage = np.concatenate(packs)
    _, out = _place_all(stage, occ, po, R, shard_rows, hkv, dh, w)
    assert np.array_equal(out["k"], k.view(np.uint8).ravel())
    assert np.array_equal(out["v"], v.view(np.uint8).ravel())
    assert np.array_equal(out["kc"], kc.view(np.uint8).ravel())
    assert np.array_equal(out["vc"], vc.view(np.uint8).ravel())
    for s in seg.values():                     # the CUDA copy needs 16-byte segments
        assert (s % 16 == 0).all()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, result):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        rng = np.random.default_rng(7)
        occ = rng.integers(1, 40, 19).astype(np.int64)
        hkv, dh, w = 2, 64, 64
        po, R, k, v, kc, vc = _canonical(occ, hkv, dh, w, 7)
        owner = rng.integers(0, world, occ.size)
        shard_rows = [np.flatnonzero(owner == r) for r in range(world)]
        mine = torch.from_numpy(_pack(shard_rows[rank], occ, po, k, v, kc, vc, hkv, dh, w))
        offs, _ = S.placement_segments(occ, po, R, shard_rows, hkv, dh, w)
        stage = torch.zeros(offs[-1], dtype=torch.uint8)
        slots = [stage[offs[r]:offs[r + 1]] for r in range(world)]
        S.NcclTransport(rank, world)(mine, slots)()      # transport is backend-agnostic
        _, out = _place_all(stage.numpy(), occ, po, R, shard_rows, hkv, dh, w)
        ok = (np.array_equal(out["k"], k.view(np.uint8).ravel()) and
              np.array_equal(out["v"], v.view(np.uint8).ravel()) and
              np.array_equal(out["kc"], kc.view(np.uint8).ravel()) and
              np.array_equal(out["vc"], vc.view(np.uint8).ravel()))
        sizes = [3 + 2 * r for r in range(world)]
        got = S.allgather_v(torch.full((sizes[rank],), float(rank)), sizes)
        ok = ok and all(torch.equal(g, torch.full((sizes[r],), float(r))) for r, g in enumerate(got))
        result[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_all_gather_kv():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    with ctx.Manager() as mgr:
        result = mgr.dict()
        procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, result)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=180)
        assert all(p.exitcode == 0 for p in procs)
        assert dict(result) == {0: True, 1: True}


# ---------------------------------------------------------------------------
# dispatch / return all_to_all_v (TokenDispatch): plan + gloo world 2


def _cpu_gather(src, index, out=None):
    return src[index]


def _cpu_scatter(src, index, out):
    out[index] = src
    return out


@pytest.mark.parametrize("W", [2, 3, 8])
def test_token_dispatch_plan_matches_reference_accounting(c1_parts, W):
    """The device dispatch moves exactly the reference's all_to_all messages
    (`seq_parallel.py:146-178`, dispatch phase of `parallel_sparse_stage`)
    and its index arrays tile the naive and local orders."""
    pv, pi = c1_parts
    topo = S.shard_blocks(pv, pi, W)
    n = pv.n_tokens + pi.n_tokens
    aligned = [np.concatenate([topo.vol_tokens[w], topo.img_tokens[w] + pv.n_tokens])
               for w in range(W)]
    naive = S.naive_contiguous_shards(n, W)
    ref = S.WorkerTopology(W, [], [], [], [], np.zeros(W, np.int64))
    S.all_to_all(naive, aligned, ref, "dispatch", 4 * 64 + 12)
    dev = S.WorkerTopology(W, [], [], [], [], np.zeros(W, np.int64))
    plans = [S.TokenDispatch(pv, pi, topo, r, W) for r in range(W)]
    plans[0].log(dev, "dispatch", 4 * 64 + 12)
    assert dev.message_log == ref.message_log
    for r, p in enumerate(plans):
        assert sorted(p.send_index.tolist()) == list(range(naive[r].size))
        assert sorted(p.recv_index.tolist()) == list(range(p.n_local))
        assert np.array_equal(np.sort(p.local_tokens), np.sort(aligned[r]))
        assert sum(p.send_counts) == naive[r].size
        assert [q.recv_counts[r] for q in plans] == p.send_counts


def _dispatch_worker(rank, world, port, result):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        from paper_2604_05182_b200.workloads import coarse_inputs
        from fixtures import load_workload
        wl = load_workload("c1")
        x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 64)
        x_up, y_up = O.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v.tables,
                                              pe_i.tables, wl.factor_vol, wl.factor_img)
        pv = O.partition_tokens("volume", x_up.coords, x_up.grid_res)
        pi = O.partition_tokens("image", y_up.coords, y_up.grid_res)
        topo = S.shard_blocks(pv, pi, world)
        feats = torch.from_numpy(np.concatenate([x_up.features, y_up.features]))
        coords = torch.from_numpy(np.concatenate([x_up.coords, y_up.coords]).astype(np.int32))
        tk = S.TokenDispatch(pv, pi, topo, rank, world)
        lo = int(np.concatenate([[0], np.cumsum([a.size for a in tk.naive])])[rank])
        mine = slice(lo, lo + tk.n_naive)
        loc_f = torch.zeros((tk.n_local, 64))
        loc_c = torch.zeros((tk.n_local, 3), dtype=torch.int32)
        tr = S.HostStagedTransport(rank, world)
        tk.dispatch(tr, [feats[mine], coords[mine]], [loc_f, loc_c], _cpu_gather, _cpu_scatter)
        ok = torch.equal(loc_f, feats[tk.local_tokens]) and \
            torch.equal(loc_c, coords[tk.local_tokens])
        back = torch.zeros((tk.n_naive, 64))
        tk.gather_back(tr, [loc_f * 2.0], [back], _cpu_gather, _cpu_scatter)
        ok = ok and torch.equal(back, feats[mine] * 2.0)
        result[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_token_dispatch_round_trip():
    """dispatch -> (local op) -> return over a real gloo world of 2: every
    rank receives exactly its owned tokens in local order and gets its naive
    shard back."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    with ctx.Manager() as mgr:
        result = mgr.dict()
        procs = [ctx.Process(target=_dispatch_worker, args=(r, 2, port, result))
                 for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=180)
        assert all(p.exitcode == 0 for p in procs)
        assert dict(result) == {0: True, 1: True}


# ---------------------------------------------------------------------------
# GPU: emulated ranks reproduce the single-GPU engine


@pytest.mark.gpu
@pytest.mark.parametrize("W,by_cost", [(2, True), (3, False)])
@pytest.mark.parametrize("cross_global", [True, False])
def test_sharded_engine_matches_unsharded(cuda, W, by_cost, cross_global, monkeypatch):
    """Sharded engines vs the single-GPU engine.  With the default block
    tiles (cross_global=False) EVERY use is bit-identical for every W (the
    reference's serial == parallel contract, `tests/test_seq_parallel.py:
    285-325` of the reference).  The opt-in across-block cross tiles
    (LSRM_CROSS_GLOBAL_TILES=1) are not W-invariant: cross uses then differ
    by bf16 rounding only."""
    from paper_2604_05182_b200 import engine as E
    monkeypatch.setattr(E, "CROSS_GLOBAL_TILES", cross_global)
    from paper_2604_05182_b200 import _ops
    from paper_2604_05182_b200.engine import USE_GEOM, USES
    from paper_2604_05182_b200.layer import SparseAttentionLayer, build_instance
    from paper_2604_05182_b200.tensor_core import AttentionParams
    inst = build_instance("c1", params=AttentionParams(32, 2, 32))   # C1 geometry, paper heads
    layer = SparseAttentionLayer(inst)
    x_bm, y_bm = layer.device_inputs(inst.x_hat, inst.y_hat)
    ref = {u: t.clone() for u, t in layer.engine.forward(x_bm, y_bm).items()}
    engines, topo = S.build_sharded_engines(inst, W, by_cost=by_cost)
    for e in engines:
        e.forward_local(_ops.gather_rows(x_bm, e.meta["x"].loc2glob),
                        _ops.gather_rows(y_bm, e.meta["y"].loc2glob))
    outs = [e.forward_exchange() for e in engines]
    torch.cuda.synchronize()
    for use in USES:
        qs = USE_GEOM[use][0]
        full = torch.zeros_like(ref[use])
        for e, o in zip(engines, outs):
            if e.meta[qs].n_loc:
                full[e.meta[qs].loc2glob] = o[use]
        diff = (full.float() - ref[use].float()).abs().max().item()
        scale = ref[use].float().abs().max().item()
        print(f"W={W} {use}: max|diff| {diff:.3e} (scale {scale:.3e})")
        # same canonical KV bytes; same tiles unless the single-GPU engine
        # tiles the cross uses across blocks
        if USE_GEOM[use][2] == 3 or not cross_global:
            assert diff == 0.0, (use, diff)
        else:
            assert diff <= 1e-2 * scale
    # every rank logged its shard to every other rank for every use
    srcs = {src for _, kind, src, _, _ in topo.message_log if kind == "all_gather_kv"}
    assert srcs == set(range(W))


@pytest.mark.gpu
@pytest.mark.parametrize("W", [2, 3])
def test_torchrun_ranks_share_one_gpu(cuda, W):
    """Real multi-process path (torchrun, one process per rank, gloo +
    host-staged exchange on one GPU; the NCCL transport is the same call
    sequence with device buffers)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "tests", "sp_worker.py"), "c1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.gpu
@pytest.mark.parametrize("W", [2, 3])
def test_torchrun_sharded_stage(cuda, W):
    """Dispatch -> 2 sharded Stage-2 blocks (per-use All-gather-KV) -> return
    on W torchrun ranks sharing one GPU (gloo, host-staged): bit-equal to the
    single-GPU stage (tests/sp_stage_worker.py)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "tests", "sp_stage_worker.py"), "c1", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.gpu
@pytest.mark.parametrize("W,mode", [(2, "fp32"), (3, "fp32"), (2, "fast")])
def test_torchrun_sharded_training(cuda, W, mode):
    """One Stage-2 block training step under block-aware sequence parallelism
    (BASELINE config 5's step): W torchrun ranks sharing one GPU (gloo,
    host-staged), per-use All-gather-KV forward and its adjoint (partial
    dK / dV summed at the owners), parameter gradients summed over ranks.
    Outputs, input gradients and every parameter gradient match the one-GPU
    step (tests/sp_train_worker.py): fp32 kernels within 1e-4 (summation
    order only), the bf16 fast path within its oracle tolerance."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "tests", "sp_train_worker.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.gpu
def test_capi_nccl_transport_world1(cuda):
    """The C-ABI NCCL exchanges (`lsrm_allgather_kv`, `lsrm_all_to_all_v`)
    through CapiNcclTransport on a one-rank communicator (this box has one
    GPU; NCCL refuses two ranks on one device), and the sharded stage on it:
    bit-equal to the single-GPU stage."""
    from paper_2604_05182_b200 import _dev as D, _ops
    from paper_2604_05182_b200.layer import build_instance
    from paper_2604_05182_b200.recon_pipeline import SparseStageEngine, init_sparse_block
    from paper_2604_05182_b200.tensor_core import AttentionParams
    tr = S.CapiNcclTransport(0, 1)
    try:
        send = torch.arange(4096, dtype=torch.int32, device="cuda").view(torch.uint8)
        stage = torch.zeros_like(send)
        tr(send, [stage])()
        assert torch.equal(stage, send)
        recv = torch.zeros_like(send)
        tr.all_to_all_v([send], [recv])()
        assert torch.equal(recv, send)
        params = AttentionParams(32, 2, 32)
        inst = build_instance("c1", params=params)
        ws = [init_sparse_block(0, params, m) for m in range(2)]
        st = S.ShardedStage(inst.part_vol, inst.part_img, inst.plan_rows, ws, params, 0, 1,
                            transport=tr)
        feats = np.concatenate([inst.x_hat, inst.y_hat]).astype(np.float32)
        coords = np.zeros((feats.shape[0], 3), np.int32)
        out = D.host(st.forward(D.dev(feats), D.dev(coords)))
        ref_eng = SparseStageEngine(inst.part_vol, inst.part_img, inst.plan_rows, ws, params)
        tv, ti = inst.part_vol.dev("block_token_ids"), inst.part_img.dev("block_token_ids")
        xs, ys = ref_eng.forward(_ops.gather_rows(D.dev(inst.x_hat), tv),
                                 _ops.gather_rows(D.dev(inst.y_hat), ti))
        xo, yo = torch.empty_like(xs), torch.empty_like(ys)
        _ops.scatter_rows(xs, tv, xo)
        _ops.scatter_rows(ys, ti, yo)
        ref = np.concatenate([D.host(xo), D.host(yo)])
        assert np.array_equal(out, ref)
    finally:
        tr.close()


# ---------------------------------------------------------------------------
# sequence-parallel training: the host side of LocalQueries


@pytest.mark.parametrize("W", [2, 3, 8])
def test_local_queries_cover_owned_blocks(c1_parts, W):
    """Every rank's local rows are exactly its owned blocks' tokens (block-
    major, owned blocks ascending); over the ranks every token appears once;
    own rows name each local row's block; the window lists of a block hold
    the local rows of its tokens and are empty for blocks another rank owns."""
    from paper_2604_05182_b200.block_partition import BlockPartition
    from paper_2604_05182_b200.training import local_query_arrays
    for part, rows_of in zip(c1_parts, ("vol_rows", "img_rows")):
        bp = BlockPartition(**{f: getattr(part, f) for f in (
            "modality", "block_size", "block_grid", "n_blocks_total", "block_of_token",
            "occupied_ids", "block_offsets", "block_token_ids", "occupancy", "block_centers",
            "block_views")})
        topo = S.shard_blocks(*c1_parts, W)
        seen = []
        for r in range(W):
            owned, loc_tok, own_rows, win_offs, win_ids = local_query_arrays(
                bp, getattr(topo, rows_of)[r])
            want = [bp.tokens_in_row(int(b)) for b in owned]
            assert np.array_equal(loc_tok, np.concatenate(want) if want else np.zeros(0))
            assert np.array_equal(own_rows, np.repeat(owned, bp.occupancy[owned]))
            assert win_offs.size == bp.n_occupied + 1 and win_offs[-1] == loc_tok.size
            for b in range(bp.n_occupied):
                ids = win_ids[win_offs[b]:win_offs[b + 1]]
                if b in set(owned.tolist()):
                    assert np.array_equal(loc_tok[ids], bp.tokens_in_row(b))
                else:
                    assert ids.size == 0
            seen.append(loc_tok)
        allt = np.concatenate(seen)
        assert np.array_equal(np.sort(allt), np.arange(bp.n_tokens))
