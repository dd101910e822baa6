"""Block-aware sequence parallelism with All-gather-KV (drop-in for
`lsrm/seq_parallel.py`, plus the real multi-GPU runtime).

Reference semantics (in-process simulation, `lsrm/seq_parallel.py:1-15`):
blocks are assigned whole by greedy LPT over token counts; tokens reach their
workers through an all-to-all; every sparse attention use all-gathers KV
(original + compressed) while queries stay sharded; window attention is
worker-local; collectives append (phase, kind, src, dst, bytes) records.

B200 runtime (one process per GPU, NCCL over NVLink/NVSwitch):
  * `shard_blocks` (token LPT, the reference rule) or `shard_blocks_by_cost`
    (the north star's routed-block workload: sum of routed key counts over the
    block's queries for all uses + occupancy^2 for the window branch);
  * each rank runs `engine.SparseLayerEngine` on its owned blocks' tokens,
    computes K/V + compression for its owned KV blocks into ONE packed
    buffer per use, and `KVExchange` all-gathers the packed buffers with a
    grouped NCCL send/recv (all-gather-v; shards are uneven), then places
    every block into the canonical block-major layout with one segment-copy
    kernel per tensor — so each output row sees byte-identical KV whatever
    the number of ranks (W-invariance, `tests/test_seq_parallel.py:285-325`).
  * exchanges of all four uses are launched before the first attention, so
    later uses' transfers overlap earlier uses' attention.
"""

import csv
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _dev as D
from ._native import call
from .block_partition import BlockPartition
from .errors import ProtocolError, require

TOKEN_COORD_BYTES = 12     # three u32 spatial coords per moved token (seq_parallel.py:34)


# ---------------------------------------------------------------------------
# topology and message log


@dataclass
class WorkerTopology:
    """`lsrm/seq_parallel.py:37-58`."""
    n_workers: int
    vol_rows: list
    img_rows: list
    vol_tokens: list
    img_tokens: list
    loads: np.ndarray
    message_log: list = dc_field(default_factory=list)

    def assignment(self, part: BlockPartition, modality: str) -> np.ndarray:
        rows = self.vol_rows if modality == "volume" else self.img_rows
        out = np.full(part.n_blocks_total, -1, dtype=np.int64)
        for w, rr in enumerate(rows):
            out[part.occupied_ids[rr]] = w
        return out

    def log(self, phase: str, kind: str, src: int, dst: int, n_bytes: int) -> None:
        self.message_log.append((phase, kind, int(src), int(dst), int(n_bytes)))


def message_log_to_csv(log, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["phase", "kind", "src", "dst", "bytes"])
        w.writerows(log)


def _tokens_of(part, rows_per_worker):
    return [np.concatenate([part.tokens_in_row(r) for r in rr]) if rr.size
            else np.zeros(0, np.int64) for rr in rows_per_worker]


def _lpt(items, n_workers):
    """Greedy LPT: items = [(sort key, weight, modality 0/1, row)], heaviest
    first; each goes to the lightest worker (ties: lower worker id)."""
    loads = np.zeros(n_workers, dtype=np.float64)
    rows = [[[] for _ in range(n_workers)] for _ in range(2)]
    for _key, wgt, mod, row in sorted(items):
        w = int(np.argmin(loads))
        loads[w] += wgt
        rows[mod][w].append(row)
    return [[np.array(sorted(r), dtype=np.int64) for r in rm] for rm in rows], loads


def shard_blocks(part_vol: BlockPartition, part_img: BlockPartition,
                 n_workers: int) -> WorkerTopology:
    """Greedy LPT over pooled blocks by token count: occupancy descending,
    ties volume first then lower block id; lightest worker, ties lower id
    (`seq_parallel.py:93-131`)."""
    require(n_workers >= 1, "need at least one worker")
    items = [((-int(p.occupancy[r]), m, int(p.occupied_ids[r])), int(p.occupancy[r]), m, r)
             for m, p in enumerate((part_vol, part_img)) for r in range(p.n_occupied)]
    (vol_rows, img_rows), loads = _lpt(items, n_workers)
    return WorkerTopology(n_workers, vol_rows, img_rows, _tokens_of(part_vol, vol_rows),
                          _tokens_of(part_img, img_rows), loads.astype(np.int64))


def block_costs(part_vol, part_img, lengths: dict, window_uses=("v2v", "i2i")):
    """Routed-block workload per query block (SURVEY.md §7 hard part 7):
    sum over the block's tokens of the routed key count L_i of every use it
    queries, plus occupancy^2 per window use.  lengths: use -> [n_q] gathered
    key counts in the query partition's TOKEN order."""
    cost = {"v": np.zeros(part_vol.n_occupied), "i": np.zeros(part_img.n_occupied)}
    parts = {"v": part_vol, "i": part_img}
    for use, L in lengths.items():
        q = use[0]
        p = parts[q]
        Lb = np.asarray(L, np.float64)[p.block_token_ids]
        cost[q] += np.add.reduceat(Lb, p.block_offsets[:-1]) if p.n_occupied else 0.0
        if use in window_uses:
            cost[q] += p.occupancy.astype(np.float64) ** 2
    # compressed branch: every query attends all compressed rows of its KV side
    for use in lengths:
        q, k = use[0], use[2]
        cost[q] += parts[q].occupancy.astype(np.float64) * parts[k].n_occupied
    return cost["v"], cost["i"]


def shard_blocks_by_cost(part_vol, part_img, n_workers, cost_vol, cost_img) -> WorkerTopology:
    """LPT over routed-block workload (north star item 4); same tie rules."""
    require(n_workers >= 1, "need at least one worker")
    items = [((-float(c[r]), m, int(p.occupied_ids[r])), float(c[r]), m, r)
             for m, (p, c) in enumerate(((part_vol, cost_vol), (part_img, cost_img)))
             for r in range(p.n_occupied)]
    (vol_rows, img_rows), loads = _lpt(items, n_workers)
    return WorkerTopology(n_workers, vol_rows, img_rows, _tokens_of(part_vol, vol_rows),
                          _tokens_of(part_img, img_rows), loads)


def naive_contiguous_shards(n_tokens: int, n_workers: int):
    """`seq_parallel.py:134-139`."""
    edges = np.linspace(0, n_tokens, n_workers + 1).astype(np.int64)
    return [np.arange(lo, hi, dtype=np.int64) for lo, hi in zip(edges[:-1], edges[1:])]


# ---------------------------------------------------------------------------
# reference-API collectives (accounting + invariant checks)


def all_to_all(shards_in, shards_out, topology: WorkerTopology, phase: str,
               bytes_per_token: int):
    """Re-shard tokens; conservation checks raise ProtocolError; logs bytes
    per ordered pair (`seq_parallel.py:146-178`)."""
    n = topology.n_workers
    require(len(shards_in) == n and len(shards_out) == n,
            "shard lists must have one entry per worker")
    owner = np.concatenate([np.full(np.asarray(ids).size, w, np.int64)
                            for w, ids in enumerate(shards_in)])
    flat = np.concatenate([np.asarray(ids, np.int64).ravel() for ids in shards_in])
    uniq, first, counts = np.unique(flat, return_index=True, return_counts=True)
    if (counts > 1).any():
        # report the first repeated occurrence in production order
        seen = np.zeros(flat.size, bool)
        seen[first] = True
        raise ProtocolError(f"token {int(flat[np.flatnonzero(~seen)[0]])} produced by two workers")
    src = owner[first]
    moved = np.zeros((n, n), dtype=np.int64)
    for dst, ids in enumerate(shards_out):
        ids = np.asarray(ids, np.int64).ravel()
        pos = np.minimum(np.searchsorted(uniq, ids), max(uniq.size - 1, 0))
        ok = (uniq[pos] == ids) if uniq.size else np.zeros(ids.size, bool)
        if not ok.all():
            raise ProtocolError(f"token {int(ids[~ok][0])} requested by worker {dst} "
                                "was never produced")
        np.add.at(moved[:, dst], src[pos], 1)
    if int(moved.sum()) != flat.size:
        raise ProtocolError("all-to-all does not conserve the token set")
    for s in range(n):
        for d in range(n):
            if s != d and moved[s, d]:
                topology.log(phase, "all_to_all", s, d, int(moved[s, d]) * bytes_per_token)
    return shards_out


def all_gather_kv(local_parts, topology: WorkerTopology, phase: str):
    """Replicate per-worker KV into global tensors (k, v by token id; cmp rows
    by occupied row); ownership must tile both index spaces
    (`seq_parallel.py:181-218`).  NumPy in -> NumPy out."""
    n = topology.n_workers
    block_rows = np.concatenate([np.asarray(p["block_rows"]) for p in local_parts])
    if not np.array_equal(np.sort(block_rows), np.arange(block_rows.size)):
        raise ProtocolError("worker block ownership does not tile the occupied blocks")
    order = np.argsort(block_rows, kind="stable")
    k_cmp = np.concatenate([p["k_cmp"] for p in local_parts])[order]
    v_cmp = np.concatenate([p["v_cmp"] for p in local_parts])[order]
    token_ids = np.concatenate([np.asarray(p["token_ids"]) for p in local_parts])
    if not np.array_equal(np.sort(token_ids), np.arange(token_ids.size)):
        raise ProtocolError("worker token ownership does not tile the token sequence")
    tail = np.asarray(local_parts[0]["k"]).shape[1:]
    k_tok = np.zeros((token_ids.size,) + tail, np.float32)
    v_tok = np.zeros((token_ids.size,) + tail, np.float32)
    for p in local_parts:
        k_tok[p["token_ids"]] = p["k"]
        v_tok[p["token_ids"]] = p["v"]
    kv_bytes = [4 * 2 * (np.asarray(p["k"]).size + np.asarray(p["k_cmp"]).size)
                for p in local_parts]
    for s in range(n):
        for d in range(n):
            if s != d and kv_bytes[s]:
                topology.log(phase, "all_gather_kv", s, d, kv_bytes[s])
    return k_tok, v_tok, k_cmp, v_cmp


def parallel_sparse_stage(x_up, y_up, weights, ctx, params, n_workers: int):
    """Sharded sparse stage, reference API (`seq_parallel.py:321-434`):
    returns (x_s, y_s, topology) with the states in global token order.

    The topology and its message log follow the reference protocol exactly:
    the dispatch all-to-all, per layer and use one All-gather-KV of every
    worker's projected + compressed blocks (4*2*(|k| + |k_cmp|) bytes to each
    other worker), a zero-byte window entry per worker for self uses, and the
    return all-to-all.  The data path runs on this process's GPU: every
    output row depends only on its own query and the gathered (canonical)
    KV, so the W shards are computed in one pass of the fp32 stage
    (`recon_pipeline.sparse_stage_forward`) and the result is the serial one
    (the reference requires <= 1e-6; here it is identical).  The
    multi-process NCCL path with real per-rank shards is `ShardedLayer`.

    With the drop-in's precision "bf16" (`fastpath`) and a geometry the
    bf16 engine takes, the W workers really run: one thread per worker, each
    a `ShardedStage` (dispatch all-to-all, per-use All-gather-KV, return
    all-to-all) exchanging device buffers through `ThreadTransport`; the
    message log is then the bytes those exchanges moved."""
    from . import fastpath
    if fastpath.active():
        r = _parallel_stage_threads(x_up, y_up, weights, ctx, params, n_workers)
        if r is not None:
            return r
    from .recon_pipeline import sparse_stage_forward
    part_vol, part_img = ctx.part_vol, ctx.part_img
    require(x_up.count == part_vol.n_tokens and y_up.count == part_img.n_tokens,
            "token sets do not match the partitions in the context")
    require(x_up.count > 0 and y_up.count > 0, "parallel stage needs nonempty token streams")
    d = params.model_dim
    width = params.n_kv_heads * params.head_dim
    topology = shard_blocks(part_vol, part_img, n_workers)
    n_x = int(x_up.count)
    aligned = [np.concatenate([topology.vol_tokens[w], topology.img_tokens[w] + n_x])
               for w in range(n_workers)]
    naive = naive_contiguous_shards(n_x + int(y_up.count), n_workers)
    all_to_all(naive, aligned, topology, "dispatch", 4 * d + TOKEN_COORD_BYTES)
    x_s, y_s = sparse_stage_forward(x_up, y_up, weights, ctx, params)
    for m in range(len(weights)):
        for name, kv_vol, is_self in (("v2v", True, True), ("v2i", False, False),
                                      ("i2i", False, True), ("i2v", True, False)):
            toks = topology.vol_tokens if kv_vol else topology.img_tokens
            rows = topology.vol_rows if kv_vol else topology.img_rows
            kv_bytes = [4 * 2 * (t.size * width + r.size * width) for t, r in zip(toks, rows)]
            for s in range(n_workers):
                for dst in range(n_workers):
                    if s != dst and kv_bytes[s]:
                        topology.log(f"layer{m}/{name}", "all_gather_kv", s, dst, kv_bytes[s])
            if is_self:
                for w in range(n_workers):   # self use: queries are the kv tokens
                    if toks[w].size:
                        topology.log(f"layer{m}/{name}/win", "window", w, w, 0)
    all_to_all(aligned, naive, topology, "return", 4 * d + TOKEN_COORD_BYTES)
    return x_s, y_s, topology


def _parallel_stage_threads(x_up, y_up, weights, ctx, params, n_workers: int):
    """bf16 `parallel_sparse_stage`: W ShardedStage workers on threads."""
    import threading
    from . import fastpath
    from .nsa_attention import selection_rows
    if not fastpath._ctx_ok(ctx, params) or len(weights) == 0:
        return None
    require(n_workers >= 1, "need at least one worker")
    pv, pi = ctx.part_vol, ctx.part_img
    require(x_up.count == pv.n_tokens and y_up.count == pi.n_tokens,
            "token sets do not match the partitions in the context")
    plan_rows = fastpath._ctx_rows(ctx)
    topology = shard_blocks(pv, pi, n_workers)
    uses = [fastpath._block_uses(w) for w in weights]
    feats = np.concatenate([np.asarray(D.host(x_up.features) if D.is_device(x_up.features)
                                       else x_up.features, np.float32),
                            np.asarray(D.host(y_up.features) if D.is_device(y_up.features)
                                       else y_up.features, np.float32)])
    coords = np.concatenate([np.asarray(D.host(c) if D.is_device(c) else c)
                             for c in (x_up.coords, y_up.coords)]).astype(np.int32)
    shared, outs, errs = ThreadTransport.make_shared(n_workers), [None] * n_workers, []
    dev = torch.cuda.current_device()

    def worker(r):
        try:
            torch.cuda.set_device(dev)
            tr = ThreadTransport(r, n_workers, shared)
            st = ShardedStage(pv, pi, plan_rows, weights, params, r, n_workers,
                              topology=topology if r == 0 else _topology_copy(topology),
                              transport=tr, uses=uses)
            tk = st.tokens
            lo = int(np.concatenate([[0], np.cumsum([a.size for a in tk.naive])])[r])
            out = st.forward(D.dev(feats[lo:lo + tk.n_naive]), D.dev(coords[lo:lo + tk.n_naive]))
            outs[r] = (lo, D.host(out), st.topology.message_log)
        except BaseException as exc:   # noqa: BLE001 (re-raised on the caller's thread)
            errs.append(exc)
            shared["barrier"].abort()
    threads = [threading.Thread(target=worker, args=(r,)) for r in range(n_workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    res = np.empty_like(feats)
    log = []
    for lo, o, lg in outs:
        res[lo:lo + o.shape[0]] = o
    for r in range(n_workers):     # worker logs, in rank order
        log += outs[r][2] if r else []
    topology.message_log.extend(log)
    n_x = int(x_up.count)
    return res[:n_x], res[n_x:], topology


def _topology_copy(t: WorkerTopology) -> WorkerTopology:
    return WorkerTopology(t.n_workers, t.vol_rows, t.img_rows, t.vol_tokens, t.img_tokens,
                          t.loads)


# ---------------------------------------------------------------------------
# load-balance reporting (`seq_parallel.py:441-470`)


def makespan_ratio(loads, n_workers: int) -> float:
    total = float(np.sum(loads))
    return 1.0 if total == 0.0 else float(np.max(loads)) / (total / n_workers)


def naive_split_loads(part_vol, part_img, n_workers: int) -> np.ndarray:
    occ = np.concatenate([part_vol.occupancy, part_img.occupancy])
    return np.array([int(r.sum()) for r in np.array_split(occ, n_workers)], dtype=np.int64)


def imbalance_report(instances, n_workers: int):
    out = []
    for pv, pi in instances:
        topo = shard_blocks(pv, pi, n_workers)
        naive = naive_split_loads(pv, pi, n_workers)
        out.append({"loads": topo.loads.tolist(), "naive_loads": naive.tolist(),
                    "ratio_block_aware": makespan_ratio(topo.loads, n_workers),
                    "ratio_naive": makespan_ratio(naive, n_workers)})
    return out


# ---------------------------------------------------------------------------
# distributed All-gather-KV for the bf16 engine


def placement_segments(occupancy, pad_off, n_rows_pad: int, shard_rows, hkv: int, dh: int,
                       w: int):
    """Staging layout of an all-gathered stream and the byte segments that
    place every rank's blocks into the canonical global buffers.

    Returns (stage_off [W+1] byte offsets of each rank's packed shard,
    {"k","v","kc","vc": int64 [n_seg, 3] (src byte offset in staging, dst
    byte offset in the global buffer, bytes)}).  Global buffers: interleaved
    K [hkv, n_rows_pad, dh] / V [hkv, n_rows_pad, dh+16] bf16 with block b at
    padded row pad_off[b]; compressed K/V [n_blocks, w] f32 (engine.py).
    """
    from .engine import ONES_COLS, ROW_PAD, PackedShard
    occ = np.asarray(occupancy, np.int64)
    gpo = np.asarray(pad_off, np.int64)
    vw = dh + ONES_COLS
    offs = [0]
    seg = {"k": [], "v": [], "kc": [], "vc": []}
    for rows in shard_rows:
        rows = np.sort(np.asarray(rows, np.int64))
        lpo = np.concatenate([[0], np.cumsum((occ[rows] + ROW_PAD - 1) // ROW_PAD * ROW_PAD)])
        lay = PackedShard(hkv, dh, w, int(lpo[-1]), rows.size)
        base = offs[-1]
        j = np.arange(rows.size)
        plen = gpo[rows + 1] - gpo[rows]
        for h in range(hkv):
            seg["k"].append(np.stack([base + (h * lay.rows_pad + lpo[:-1]) * dh * 2,
                                      (h * n_rows_pad + gpo[rows]) * dh * 2, plen * dh * 2], 1))
            seg["v"].append(np.stack([base + lay.off_v + (h * lay.rows_pad + lpo[:-1]) * vw * 2,
                                      (h * n_rows_pad + gpo[rows]) * vw * 2, plen * vw * 2], 1))
        seg["kc"].append(np.stack([base + lay.off_kc + j * w * 4, rows * w * 4,
                                   np.full(rows.size, w * 4)], 1))
        seg["vc"].append(np.stack([base + lay.off_vc + j * w * 4, rows * w * 4,
                                   np.full(rows.size, w * 4)], 1))
        offs.append(base + lay.total)
    seg = {k: np.concatenate(v).astype(np.int64).reshape(-1, 3) if v else
           np.zeros((0, 3), np.int64) for k, v in seg.items()}
    return offs, seg


def apply_segments(src: np.ndarray, dst: np.ndarray, segs: np.ndarray) -> None:
    """Host restatement of lsrm_copy_segments (tests): byte arrays."""
    for so, do, nb in segs.tolist():
        dst[do:do + nb] = src[so:so + nb]


class KVExchange:
    """All-gather-KV for a sharded SparseLayerEngine.

    shards: per stream, the owned occupied rows of every rank (same on all
    ranks).  transport(send, recv_slots) moves the packed per-use shards; the
    default is a grouped NCCL send/recv through torch.distributed
    (all-gather-v: shards are uneven); `InProcessTransport` is used by the
    single-GPU tests that emulate several ranks.
    """

    def __init__(self, engine, rank: int, world: int, shards: dict, transport=None,
                 topology: WorkerTopology = None):
        from .engine import USE_GEOM, USES
        self.rank, self.world = rank, world
        self.transport = transport or NcclTransport(rank, world)
        self.topology = topology
        self.layer_index = 0
        p = engine.params
        hkv, dh, w = p.n_kv_heads, p.head_dim, engine.w
        self.stage_off, self.segs, self.stage = {}, {}, {}
        for s in ("x", "y"):
            m = engine.meta[s]
            offs, seg = placement_segments(m.part.occupancy, m.pad_off_host, m.n_rows_pad,
                                           shards[s], hkv, dh, w)
            self.stage_off[s] = offs
            self.segs[s] = {k: D.dev(v) for k, v in seg.items()}
        for use in USES:
            _, ks, _ = USE_GEOM[use]
            require(int(engine.buf[("packed", use)].numel()) ==
                    self.stage_off[ks][rank + 1] - self.stage_off[ks][rank],
                    "seq_parallel: shard layout disagrees with the engine's")
            self.stage[use] = D.zeros((self.stage_off[ks][-1],), torch.uint8)
        self.packed = {use: engine.buf[("packed", use)] for use in USES}

    def start(self, use: str):
        """Launch the all-gather of `use`'s packed shard into its staging
        buffer; returns the transport's wait callable (stream-ordered)."""
        from .engine import USE_GEOM
        _, ks, _ = USE_GEOM[use]
        offs = self.stage_off[ks]
        slots = [self.stage[use][offs[r]:offs[r + 1]] for r in range(self.world)]
        if self.topology is not None:
            nbytes = self.packed[use].numel()
            for d in range(self.world):
                if d != self.rank:
                    self.topology.log(f"layer{self.layer_index}/{use}", "all_gather_kv",
                                      self.rank, d, nbytes)
        return self.transport(self.packed[use], slots)

    def place(self, engine, use: str):
        """Staging -> canonical global K/V and compressed rows (4 segment-copy
        launches; capturable in a CUDA graph)."""
        from .engine import USE_GEOM
        _, ks, _ = USE_GEOM[use]
        st = D.stream()
        stage = self.stage[use]
        for kind, dst in (("k", engine.buf[("k_il", use)]), ("v", engine.buf[("v_il", use)]),
                          ("kc", engine.buf[("kc", use)]), ("vc", engine.buf[("vc", use)])):
            segs = self.segs[ks][kind]
            call("lsrm_copy_segments", stage.data_ptr(), dst.data_ptr(), segs.data_ptr(),
                 int(segs.shape[0]), st)

    def __call__(self, engine, use: str):
        """engine hook: start the exchange; the returned callable waits and
        places."""
        wait = self.start(use)

        def finish():
            wait()
            self.place(engine, use)
        return finish


class NcclTransport:
    """All-gather-v of one packed buffer per rank: grouped NCCL send/recv
    (`torch.distributed.batch_isend_irecv`), own slot copied locally."""

    def __init__(self, rank, world, group=None):
        self.rank, self.world, self.group = rank, world, group

    def __call__(self, send: torch.Tensor, slots):
        import torch.distributed as dist
        slots[self.rank].copy_(send)
        ops = []
        for peer in range(self.world):
            if peer == self.rank:
                continue
            ops.append(dist.P2POp(dist.isend, send, peer, group=self.group))
            ops.append(dist.P2POp(dist.irecv, slots[peer], peer, group=self.group))
        reqs = dist.batch_isend_irecv(ops) if ops else []

        def wait():
            for r in reqs:
                r.wait()
        return wait

    def all_to_all_v(self, sends, recvs):
        """sends[p] -> peer p, recvs[p] <- peer p (own chunk copied); grouped
        NCCL send/recv, stream-ordered. Returns the wait callable."""
        import torch.distributed as dist
        if sends[self.rank].numel():
            recvs[self.rank].copy_(sends[self.rank])
        ops = []
        for peer in range(self.world):
            if peer == self.rank:
                continue
            if sends[peer].numel():
                ops.append(dist.P2POp(dist.isend, sends[peer], peer, group=self.group))
            if recvs[peer].numel():
                ops.append(dist.P2POp(dist.irecv, recvs[peer], peer, group=self.group))
        reqs = dist.batch_isend_irecv(ops) if ops else []

        def wait():
            for r in reqs:
                r.wait()
        return wait


class CapiNcclTransport:
    """The same exchanges through this library's own C ABI
    (`lsrm_allgather_kv` / `lsrm_all_to_all_v`, csrc/comm.cu): a
    non-Python host's path. The communicator is created by the library
    (the NCCL unique id is shared over the existing process group); the
    transfers run on a side stream that waits for the producer, and the
    returned wait makes the caller's stream wait for them, so they overlap
    whatever the caller enqueues in between."""

    def __init__(self, rank, world, group=None):
        import ctypes
        import torch.distributed as dist
        from ._native import call
        self.rank, self.world = rank, world
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            call("lsrm_comm_unique_id", ctypes.addressof(uid))
        obj = [bytes(uid)]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        comm = ctypes.c_void_p()
        call("lsrm_comm_init", ctypes.addressof(uid), world, rank, ctypes.byref(comm))
        self.comm = comm
        self.side = torch.cuda.Stream()

    def close(self):
        from ._native import call
        if self.comm:
            call("lsrm_comm_destroy", self.comm)
            self.comm = None

    def _launch(self, tensors, fn):
        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        for t in tensors:
            t.record_stream(self.side)
        with torch.cuda.stream(self.side):
            fn(self.side.cuda_stream)
        side = self.side
        return lambda: torch.cuda.current_stream().wait_stream(side)

    def __call__(self, send: torch.Tensor, slots):
        import ctypes
        from ._native import call
        base = slots[0].data_ptr()
        offs = [s_.data_ptr() - base for s_ in slots] + \
            [slots[-1].data_ptr() - base + slots[-1].numel() * slots[-1].element_size()]
        off_arr = (ctypes.c_int64 * len(offs))(*offs)
        nbytes = send.numel() * send.element_size()
        return self._launch([send] + list(slots), lambda st: call(
            "lsrm_allgather_kv", self.comm, self.rank, self.world, send.data_ptr(), nbytes,
            base, off_arr, None, None, None, 0, st))

    def all_to_all_v(self, sends, recvs):
        import ctypes
        from ._native import call
        sb = (ctypes.c_int64 * self.world)(*[t.numel() * t.element_size() for t in sends])
        rb = (ctypes.c_int64 * self.world)(*[t.numel() * t.element_size() for t in recvs])
        s0 = next((t.data_ptr() for t in sends if t.numel()), 0)
        r0 = next((t.data_ptr() for t in recvs if t.numel()), 0)
        return self._launch([t for t in sends + recvs if t.numel()], lambda st: call(
            "lsrm_all_to_all_v", self.comm, self.rank, self.world, s0, sb, r0, rb, st))


class InProcessTransport:
    """Emulates W ranks inside one process (single-GPU tests): every
    engine's packed buffer is visible to every other."""

    def __init__(self, rank, registry: dict, use_of: dict):
        self.rank, self.registry, self.use_of = rank, registry, use_of

    def __call__(self, send: torch.Tensor, slots):
        use = self.use_of[send.data_ptr()]

        def wait():
            for r, slot in enumerate(slots):
                slot.copy_(self.registry[r][use])
        return wait


class ThreadTransport:
    """W workers as threads of ONE process on one GPU (the reference's own
    execution model: `_run_phase` runs the workers on a thread pool,
    `lsrm/seq_parallel.py:68-86`). Every exchange is a rendezvous: each
    worker publishes its send buffers, all wait at a barrier, each copies
    what it receives (device copies on the shared stream, so stream order
    puts them after every producer), and a second barrier keeps a sender
    from reusing its buffer before every receiver has enqueued its copy."""

    def __init__(self, rank: int, world: int, shared: dict):
        self.rank, self.world = rank, world
        self.shared = shared      # {"barrier": threading.Barrier(world), "slots": [None] * world}

    @staticmethod
    def make_shared(world: int) -> dict:
        import threading
        return {"barrier": threading.Barrier(world), "slots": [None] * world}

    def _rendezvous(self, mine, take):
        sh = self.shared
        sh["slots"][self.rank] = mine
        sh["barrier"].wait()
        take(sh["slots"])
        sh["barrier"].wait()

    def __call__(self, send: torch.Tensor, slots):
        def take(pub):
            for r, sl in enumerate(slots):
                if sl.numel():
                    sl.copy_(pub[r])
        self._rendezvous(send, take)
        return lambda: None

    def all_to_all_v(self, sends, recvs):
        def take(pub):
            for r, rv in enumerate(recvs):
                if rv.numel():
                    rv.copy_(pub[r][self.rank])
        self._rendezvous(list(sends), take)
        return lambda: None


class HostStagedTransport:
    """All-gather-v of device buffers over a CPU backend (gloo): stage through
    host memory.  Used to run several ranks on ONE GPU in tests (NCCL refuses
    two ranks on the same device); blocking."""

    def __init__(self, rank, world, group=None):
        self.rank, self.world, self.group = rank, world, group

    def __call__(self, send: torch.Tensor, slots):
        import torch.distributed as dist
        host = send.cpu()
        recv = [torch.empty(int(sl.numel()), dtype=sl.dtype) for sl in slots]
        recv[self.rank] = host
        ops = []
        for peer in range(self.world):
            if peer != self.rank:
                ops.append(dist.P2POp(dist.isend, host, peer, group=self.group))
                ops.append(dist.P2POp(dist.irecv, recv[peer], peer, group=self.group))
        for r in (dist.batch_isend_irecv(ops) if ops else []):
            r.wait()
        for sl, h in zip(slots, recv):
            sl.copy_(h)
        return lambda: None

    def all_to_all_v(self, sends, recvs):
        """Blocking all_to_all_v through host memory (gloo)."""
        import torch.distributed as dist
        hs = [t.cpu() for t in sends]
        hr = [torch.empty(tuple(t.shape), dtype=t.dtype) for t in recvs]
        hr[self.rank] = hs[self.rank]
        ops = []
        for peer in range(self.world):
            if peer == self.rank:
                continue
            if hs[peer].numel():
                ops.append(dist.P2POp(dist.isend, hs[peer], peer, group=self.group))
            if hr[peer].numel():
                ops.append(dist.P2POp(dist.irecv, hr[peer], peer, group=self.group))
        for r in (dist.batch_isend_irecv(ops) if ops else []):
            r.wait()
        for t, h in zip(recvs, hr):
            if t.numel():
                t.copy_(h)
        return lambda: None


def allgather_v(send: torch.Tensor, sizes, group=None) -> list:
    """Generic all-gather of unevenly sized 1-D tensors via grouped P2P
    (works on NCCL/CUDA and gloo/CPU); returns one tensor per rank."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    out = [torch.empty(int(n), dtype=send.dtype, device=send.device) for n in sizes]
    out[rank].copy_(send)
    ops = []
    for peer in range(world):
        if peer != rank:
            ops.append(dist.P2POp(dist.isend, send, peer, group=group))
            ops.append(dist.P2POp(dist.irecv, out[peer], peer, group=group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return out


def build_sharded_engines(inst, world: int, by_cost: bool = True):
    """Single-process construction of W sharded engines wired through
    `InProcessTransport` (tests / simulation); returns (engines, topology)."""
    from .engine import USES, SparseLayerEngine
    topo = sharding_for(inst, world, by_cost)
    shards = {"x": topo.vol_rows, "y": topo.img_rows}
    registry, engines = {}, []
    for r in range(world):
        eng = SparseLayerEngine(inst.part_vol, inst.part_img, inst.plan_rows, inst.weights,
                                inst.params, shard={"x": shards["x"][r], "y": shards["y"][r]})
        use_of = {}
        tr = InProcessTransport(r, registry, use_of)
        ex = KVExchange(eng, r, world, shards, transport=tr, topology=topo)
        registry[r] = ex.packed
        for use in USES:
            use_of[ex.packed[use].data_ptr()] = use
        eng.exchange = ex
        engines.append(eng)
    return engines, topo


def sharding_for(inst, world: int, by_cost: bool = True) -> WorkerTopology:
    """Token-LPT (reference rule) or routed-workload LPT for an instance."""
    if not by_cost:
        return shard_blocks(inst.part_vol, inst.part_img, world)
    from .engine import USES
    lengths = {}
    for use in USES:
        rows, cnt = inst.plan_rows[use]
        pk = inst.part_vol if use[2] == "v" else inst.part_img
        r, c = D.host(rows), D.host(cnt)
        occ = pk.occupancy.astype(np.float64)
        mask = np.arange(r.shape[1])[None, :] < c[:, None]
        lengths[use] = np.where(mask, occ[np.clip(r, 0, None)], 0.0).sum(axis=1)
    cv, ci = block_costs(inst.part_vol, inst.part_img, lengths)
    return shard_blocks_by_cost(inst.part_vol, inst.part_img, world, cv, ci)


class ShardedLayer:
    """One rank's share of the LSRM sparse-attention layer under block-aware
    sequence parallelism (the device counterpart of `_run_use` /
    `parallel_sparse_stage`, `lsrm/seq_parallel.py:260-434`).

    The rank owns whole query blocks (`topology`), computes K/V for the
    blocks it owns, all-gathers them per use and attends its own queries.
    `step()` replays two CUDA graphs around the exchange: A = projections +
    the four KV shards, B = placement + attention + W_o of the four uses.
    """

    def __init__(self, inst, rank: int, world: int, topology: WorkerTopology = None,
                 transport=None, by_cost: bool = True):
        from .engine import SparseLayerEngine
        self.inst, self.rank, self.world = inst, rank, world
        self.topology = topology or sharding_for(inst, world, by_cost)
        shards = {"x": self.topology.vol_rows, "y": self.topology.img_rows}
        self.engine = SparseLayerEngine(inst.part_vol, inst.part_img, inst.plan_rows,
                                        inst.weights, inst.params,
                                        shard={"x": shards["x"][rank], "y": shards["y"][rank]})
        self.exchange = KVExchange(self.engine, rank, world, shards, transport=transport)
        self.engine.exchange = self.exchange
        m = self.engine.meta
        # reference token ids of this rank's local rows, per stream
        self.tok_host = {s: m[s].part.block_token_ids[D.host(m[s].loc2glob)]
                         for s in ("x", "y")}
        self.graphs = None

    @property
    def n_local(self) -> int:
        return self.engine.meta["x"].n_loc + self.engine.meta["y"].n_loc

    def local_inputs(self, x_hat: np.ndarray, y_hat: np.ndarray):
        """Token-order f32 host features -> this rank's rows, local order, bf16."""
        from . import _ops
        return [_ops.cast(D.dev(np.ascontiguousarray(a[self.tok_host[s]], np.float32)),
                          torch.bfloat16) for s, a in (("x", x_hat), ("y", y_hat))]

    def forward(self, x_loc, y_loc) -> dict:
        """Eager: use -> [Nq_loc, d] bf16 in local order."""
        return self.engine.forward(x_loc, y_loc)

    def _phase_b(self):
        from .engine import USES
        for use in USES:
            self.exchange.place(self.engine, use)
            self.engine.finish_kv(use)
        self.engine.attend_all()
        self.engine.output_all()

    def capture(self, x_loc, y_loc):
        """Record graphs A_x, A_y (one stream's projections + KV shards
        each) and B (placement + attention + W_o) over fixed input buffers."""
        self._gin = (x_loc, y_loc)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):              # warm-up outside capture
            self.forward(x_loc, y_loc)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        ga = {s: torch.cuda.CUDAGraph() for s in ("x", "y")}
        gb = torch.cuda.CUDAGraph()
        for s in ("x", "y"):
            with torch.cuda.graph(ga[s]):
                self.engine.project(x_loc, y_loc, streams=(s,))
                self.engine.prepare_kv(s)
        with torch.cuda.graph(gb):
            self._phase_b()
        self.graphs = (ga, gb)

    def step(self) -> dict:
        """A_x -> start the exchanges of the uses that read x as KV (v2v,
        i2v) -> A_y (overlaps them) -> start v2i, i2i -> wait -> B."""
        from .engine import USES
        ga, gb = self.graphs
        waits = []
        for s in ("x", "y"):
            ga[s].replay()
            waits += [self.exchange.start(u) for u in self.engine.uses_with_kv(s)]
        for w in waits:
            w()
        gb.replay()
        return {u: self.engine.buf[("out", u)] for u in USES}

    def outputs_token_order(self, outs: dict) -> dict:
        """(host) use -> (token ids, [Nq_loc, d] f32) for gathering on rank 0."""
        from .engine import USE_GEOM
        return {u: (self.tok_host[USE_GEOM[u][0]], D.host(o.float())) for u, o in outs.items()}

    def attention_ms(self, reps: int = 5) -> float:
        """Device time of this rank's attention launch (all four uses; events
        on the launching stream; KV already placed by the last step)."""
        st = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(reps):
            self.engine.attend_all()
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def time_host_path(self, x_hat, y_hat, steps: int = 5):
        """End to end on this rank: pinned host rows -> H2D -> cast -> layer
        (graphs + exchange) -> cast -> D2H.  Returns (mean ms, h2d, d2h bytes)."""
        from . import _ops
        from .engine import USES
        xs = torch.from_numpy(np.ascontiguousarray(x_hat[self.tok_host["x"]], np.float32)).pin_memory()
        ys = torch.from_numpy(np.ascontiguousarray(y_hat[self.tok_host["y"]], np.float32)).pin_memory()
        x32, y32 = D.empty(tuple(xs.shape), torch.float32), D.empty(tuple(ys.shape), torch.float32)
        xb, yb = self._gin
        outs = self.engine.buf
        pinned = {u: torch.empty(tuple(outs[("out", u)].shape), dtype=torch.float32,
                                 pin_memory=True) for u in USES}

        def once():
            x32.copy_(xs, non_blocking=True)
            y32.copy_(ys, non_blocking=True)
            if x32.numel():
                xb.copy_(_ops.cast(x32, torch.bfloat16))
            if y32.numel():
                yb.copy_(_ops.cast(y32, torch.bfloat16))
            res = self.step()
            for u in USES:
                if res[u].numel():
                    pinned[u].copy_(_ops.cast(res[u], torch.float32), non_blocking=True)

        once()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(steps):
            once()
        b.record(st)
        torch.cuda.synchronize()
        h2d = (xs.numel() + ys.numel()) * 4
        d2h = sum(p.numel() * 4 for p in pinned.values())
        return a.elapsed_time(b) / steps, h2d, d2h


# ---------------------------------------------------------------------------
# dispatch / return (token all_to_all_v) and the sharded Stage-2 stage


def plan_rows_lengths(part_vol, part_img, plan_rows) -> dict:
    """Routed key count L_i per query (token order) of every use."""
    lengths = {}
    for use, (rows, cnt) in plan_rows.items():
        pk = part_vol if use[2] == "v" else part_img
        r, c = D.host(rows), D.host(cnt)
        occ = pk.occupancy.astype(np.float64)
        mask = np.arange(r.shape[1])[None, :] < c[:, None]
        lengths[use] = np.where(mask, occ[np.clip(r, 0, None)], 0.0).sum(axis=1)
    return lengths


class TokenDispatch:
    """The stage's two all-to-alls on the device (`lsrm/seq_parallel.py:
    341-349` dispatch, `:431-433` return): token rows move between the naive
    contiguous shards of the concatenated [volume; image] sequence
    (`naive_contiguous_shards`, the layout the stage starts and ends in) and
    the block-aligned owners of the topology.

    Rank-local order on an owner = its owned volume tokens then its owned
    image tokens, each in block-major order of the owned blocks (the order of
    `engine.stream_meta(part, owned)`). Every message s -> d carries the
    tokens of s's naive shard that d owns, in d's local order, so one gather
    (sender) and one scatter (receiver) per tensor place every row.
    `messages()` gives the (src, dst, tokens) list the reference logs."""

    def __init__(self, part_vol, part_img, topology: WorkerTopology, rank: int, world: int):
        n_x, n_y = part_vol.n_tokens, part_img.n_tokens
        self.rank, self.world, self.n_x = rank, world, n_x
        naive = naive_contiguous_shards(n_x + n_y, world)
        edges = np.concatenate([[0], np.cumsum([a.size for a in naive])]).astype(np.int64)
        self.naive = naive
        local = []
        for r in range(world):
            tx = np.concatenate([part_vol.tokens_in_row(b) for b in topology.vol_rows[r]]) \
                if len(topology.vol_rows[r]) else np.zeros(0, np.int64)
            ty = np.concatenate([part_img.tokens_in_row(b) for b in topology.img_rows[r]]) \
                if len(topology.img_rows[r]) else np.zeros(0, np.int64)
            local.append((tx.astype(np.int64), ty.astype(np.int64) + n_x))
        self.n_loc_x, self.n_loc_y = local[rank][0].size, local[rank][1].size
        # message (src -> dst) token lists in dst's local order
        self.msg = {}
        for d in range(world):
            seq = np.concatenate(local[d])
            src = np.searchsorted(edges, seq, side="right") - 1
            pos = np.arange(seq.size)
            for s_ in range(world):
                m = src == s_
                self.msg[(s_, d)] = (seq[m], pos[m])      # tokens, dst-local positions
        r = rank
        self.send_counts = [self.msg[(r, d)][0].size for d in range(world)]
        self.recv_counts = [self.msg[(s_, r)][0].size for s_ in range(world)]
        lo = int(edges[r])
        self.send_index = np.concatenate([self.msg[(r, d)][0] - lo for d in range(world)]
                                         ).astype(np.int64)
        self.recv_index = np.concatenate([self.msg[(s_, r)][1] for s_ in range(world)]
                                         ).astype(np.int64)
        self.n_naive = int(naive[r].size)
        self.n_local = self.n_loc_x + self.n_loc_y
        self.local_tokens = np.concatenate(local[r])
        self._dev = None

    def messages(self):
        """[(src, dst, n_tokens)] for src != dst with tokens to move."""
        return [(s_, d, int(self.msg[(s_, d)][0].size)) for s_ in range(self.world)
                for d in range(self.world) if s_ != d and self.msg[(s_, d)][0].size]

    def log(self, topology: WorkerTopology, phase: str, bytes_per_token: int, reverse=False,
            only_src: int = None):
        """Log the messages (all pairs, or only those `only_src` sends)."""
        for s_, d, n in self.messages():
            a, b = (d, s_) if reverse else (s_, d)
            if only_src is None or a == only_src:
                topology.log(phase, "all_to_all", a, b, n * bytes_per_token)

    @staticmethod
    def _chunks(t, counts):
        out, o = [], 0
        for c in counts:
            out.append(t[o:o + c])
            o += c
        return out

    def _indices(self):
        if self._dev is None:
            self._dev = (D.dev(self.send_index), D.dev(self.recv_index))
        return self._dev

    def dispatch(self, transport, tensors, outs, gather=None, scatter=None):
        """tensors: this rank's naive-shard rows ([n_naive, ...] each);
        outs: [n_local, ...] buffers in the rank-local order. One gather, one
        all_to_all_v and one scatter per tensor."""
        from . import _ops
        gather = gather or _ops.gather_rows
        scatter = scatter or _ops.scatter_rows
        si, ri = self._indices() if tensors[0].is_cuda else (torch.from_numpy(self.send_index),
                                                            torch.from_numpy(self.recv_index))
        waits, recvs = [], []
        for t, o in zip(tensors, outs):
            send = gather(t, si)
            recv = torch.empty((int(sum(self.recv_counts)),) + tuple(t.shape[1:]), dtype=t.dtype,
                               device=t.device)
            waits.append(transport.all_to_all_v(self._chunks(send, self.send_counts),
                                                self._chunks(recv, self.recv_counts)))
            recvs.append((recv, o))
        for w in waits:
            w()
        for recv, o in recvs:
            if recv.shape[0]:
                scatter(recv, ri, o)
        return outs

    def gather_back(self, transport, tensors, outs, gather=None, scatter=None):
        """The return all-to-all: rank-local rows -> naive-shard rows."""
        from . import _ops
        gather = gather or _ops.gather_rows
        scatter = scatter or _ops.scatter_rows
        si, ri = self._indices() if tensors[0].is_cuda else (torch.from_numpy(self.send_index),
                                                            torch.from_numpy(self.recv_index))
        waits, recvs = [], []
        for t, o in zip(tensors, outs):
            send = gather(t, ri)          # local rows, grouped by naive owner
            recv = torch.empty((int(sum(self.send_counts)),) + tuple(t.shape[1:]), dtype=t.dtype,
                               device=t.device)
            waits.append(transport.all_to_all_v(self._chunks(send, self.recv_counts),
                                                self._chunks(recv, self.send_counts)))
            recvs.append((recv, o))
        for w in waits:
            w()
        for recv, o in recvs:
            if recv.shape[0]:
                scatter(recv, si, o)
        return outs


# ---------------------------------------------------------------------------
# Training under block-aware sequence parallelism (BASELINE config 5): each
# rank runs the Stage-2 block's forward and backward for the query blocks it
# owns (training.SparseBlockModule(..., shard=...)); per NSA use the K/V rows
# are all-gathered from their owners (All-gather-KV) and, in the backward,
# every rank's partial dK / dV rows are summed at the owner (the adjoint);
# parameter gradients are summed over ranks (allreduce_grads).


class RowExchange:
    """All-gather of one stream's rows (this rank's `loc_tok[rank]` rows, any
    width) into token order, and its adjoint: the ranks' partial gradients
    of every row summed, in rank order, at the rank that owns the row."""

    def __init__(self, loc_tok: list, n_total: int, rank: int, transport):
        self.loc_tok = [np.asarray(t, np.int64) for t in loc_tok]
        self.rank, self.world, self.n_total = rank, len(loc_tok), int(n_total)
        self.transport = transport
        self.idx = [D.dev(t) for t in self.loc_tok]
        self.bytes_moved = 0

    @property
    def n_local(self) -> int:
        return int(self.loc_tok[self.rank].size)

    def gather(self, t_loc: torch.Tensor) -> torch.Tensor:
        from . import _ops
        w = int(t_loc.shape[1])
        recvs = [D.empty((int(t.size), w), t_loc.dtype) for t in self.loc_tok]
        self.transport.all_to_all_v([t_loc.contiguous()] * self.world, recvs)()
        full = D.empty((self.n_total, w), t_loc.dtype)
        for r, buf in enumerate(recvs):
            if buf.shape[0]:
                _ops.scatter_rows(buf, self.idx[r], full)
        self.bytes_moved += (self.world - 1) * t_loc.numel() * t_loc.element_size()
        return full

    def reduce_scatter(self, t_full: torch.Tensor) -> torch.Tensor:
        from . import _ops
        from ._native import call
        require(t_full.dtype == torch.float32, "reduce_scatter: f32 gradients")
        w, n = int(t_full.shape[1]), self.n_local
        sends = [_ops.gather_rows(t_full, i) for i in self.idx]
        stack = D.empty((self.world, n, w), torch.float32)
        self.transport.all_to_all_v(sends, [stack[r] for r in range(self.world)])()
        out = D.empty((n, w), torch.float32)
        if n * w:
            call("lsrm_sum_slices_f32", stack.data_ptr(), self.world, n * w, out.data_ptr(), 0,
                 D.stream())
        self.bytes_moved += sum(int(sn.numel()) * 4 for r, sn in enumerate(sends) if r != self.rank)
        return out


@dataclass
class StreamShard:
    queries: object          # training.LocalQueries of this rank
    exchange: RowExchange


def training_shard(part_vol, part_img, topology: WorkerTopology, rank: int, transport) -> dict:
    """Per stream ("x" volume, "y" image): this rank's LocalQueries and the
    RowExchange over every rank's owned rows, for
    training.SparseBlockModule(..., shard=...)."""
    from .training import local_queries
    out = {}
    for s, part, rows in (("x", part_vol, topology.vol_rows), ("y", part_img, topology.img_rows)):
        lq = [local_queries(part, r) for r in rows]
        out[s] = StreamShard(lq[rank], RowExchange([q.loc_tok for q in lq], part.n_tokens,
                                                   rank, transport))
    return out


def allreduce_grads(params, host_staged: bool = False, group=None) -> None:
    """Sum every parameter's gradient over the ranks (one flat buffer; through
    host memory for a CPU backend)."""
    import torch.distributed as dist
    grads = [p.grad for p in params if p.grad is not None]
    if not grads:
        return
    flat = torch.cat([g.reshape(-1) for g in grads])
    buf = flat.cpu() if host_staged else flat
    dist.all_reduce(buf, group=group)
    if host_staged:
        flat.copy_(buf)
    o = 0
    for g in grads:
        g.copy_(flat[o:o + g.numel()].view_as(g))
        o += g.numel()


class ShardedStage:
    """One rank of the block-aware sequence-parallel Stage-2 stage
    (`lsrm/seq_parallel.py:321-434`) on the bf16 engines:

      dispatch (all_to_all_v of features + coords, naive shard -> owners)
      -> depth x sharded `SparseBlockEngine` (row-local injection / LN /
         gates / FFN on the owned tokens; per NSA use one All-gather-KV,
         started per KV stream while the other stream is still projected)
      -> return (all_to_all_v, owners -> naive shard).

    Every output row is computed by the same tiles from byte-identical
    canonical KV whatever W is, so the result is bit-equal to the
    single-GPU `SparseStageEngine` (tests/sp_stage_worker.py). The message
    log follows the reference protocol (dispatch / layer m use / return)."""

    def __init__(self, part_vol, part_img, plan_rows, weights, params, rank: int, world: int,
                 topology: WorkerTopology = None, transport=None, by_cost: bool = True,
                 uses: list = None):
        from .recon_pipeline import SparseStageEngine
        self.rank, self.world, self.params = rank, world, params
        if topology is None:
            if by_cost:
                cv, ci = block_costs(part_vol, part_img,
                                     plan_rows_lengths(part_vol, part_img, plan_rows))
                topology = shard_blocks_by_cost(part_vol, part_img, world, cv, ci)
            else:
                topology = shard_blocks(part_vol, part_img, world)
        self.topology = topology
        self.transport = transport or NcclTransport(rank, world)
        shards = {"x": topology.vol_rows, "y": topology.img_rows}
        self.stage = SparseStageEngine(part_vol, part_img, plan_rows, weights, params,
                                       uses=uses,
                                       shard={"x": shards["x"][rank], "y": shards["y"][rank]})
        for m, blk in enumerate(self.stage.blocks):
            ex = KVExchange(blk.layer, rank, world, shards, transport=self.transport,
                            topology=topology)
            ex.layer_index = m
            blk.layer.exchange = ex
        self.tokens = TokenDispatch(part_vol, part_img, topology, rank, world)
        d = params.model_dim
        self.bytes_per_token = 4 * d + TOKEN_COORD_BYTES
        tk = self.tokens
        self.x_loc = D.empty((tk.n_loc_x, d), torch.float32)
        self.y_loc = D.empty((tk.n_loc_y, d), torch.float32)
        self._loc = D.empty((tk.n_local, d), torch.float32)
        self._coords = D.empty((tk.n_local, 3), torch.int32)
        self._out = D.empty((tk.n_local, d), torch.float32)

    def forward(self, feats_naive: torch.Tensor, coords_naive: torch.Tensor) -> torch.Tensor:
        """feats_naive [n_naive, d] f32 and coords_naive [n_naive, 3] int32:
        this rank's naive contiguous shard of the concatenated [volume;
        image] tokens. Returns the stage output rows of the same shard."""
        tk, d = self.tokens, self.params.model_dim
        tk.dispatch(self.transport, [feats_naive, coords_naive], [self._loc, self._coords])
        tk.log(self.topology, "dispatch", self.bytes_per_token, only_src=self.rank)
        nx = tk.n_loc_x
        self.stage.forward(self._loc[:nx], self._loc[nx:],
                           out=(self._out[:nx], self._out[nx:]))
        for m, blk in enumerate(self.stage.blocks):
            self._log_window(m)
        out = D.empty((tk.n_naive, d), torch.float32)
        tk.gather_back(self.transport, [self._out], [out])
        tk.log(self.topology, "return", self.bytes_per_token, reverse=True, only_src=self.rank)
        return out

    def _log_window(self, m):
        """Zero-byte window entries of the self uses (`seq_parallel.py:311`)."""
        for name, toks in (("v2v", self.topology.vol_tokens), ("i2i", self.topology.img_tokens)):
            if toks[self.rank].size:
                self.topology.log(f"layer{m}/{name}/win", "window", self.rank, self.rank, 0)
