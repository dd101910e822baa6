"""Benchmark: LSRM sparse-attention layer tokens/s (BASELINE.json metric).

One step = one sparse-attention LAYER = the four gated NSA uses (v2v, v2i,
i2i, i2v) of a Stage-2 block over all N_vol + N_img query tokens of the C3
fine-stage workload (16 views, S_vol = S_img = 96, heads 32/2/32, d = 1024,
bf16 storage / fp32 accumulation, 3D routing with default budgets).
Synthetic inputs follow SURVEY.md §8d (reference fixture geometry, tagged
Philox features and weights).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N>1 is launched by torchrun (one rank per GPU, NCCL): block-aware sequence
parallelism over the C4 skewed workload, All-gather-KV per use (see
paper_2604_05182_b200/seq_parallel.py).  `--impl reference` times the CPU
oracle port (oracle/, the reference algorithm restated in NumPy) on a
bounded query sample on the host cores.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), ws


# ---------------------------------------------------------------------------
# CPU oracle timing (reference arm and cpu_baseline)


class OracleLayer:
    """The reference algorithm's layer (four gated NSA uses, paper heads) on
    the host cores: the oracle port (oracle/, NumPy f64 restatement of
    lsrm.nsa_attention).  Instance setup (compaction, partitions, routing
    plan, LayerNorm'd inputs) is done once and not timed, like the GPU arm's
    `build_instance`.  `run(i, n)` times the i-th of n contiguous query-block
    chunks of every use against the full K/V side; the use's K/V projections
    and compression are computed (and timed) on its first call.  The n chunks
    together are exactly one full layer."""

    USES = ("v2v", "v2i", "i2i", "i2v")

    def __init__(self, wl_name="c3", seed=0):
        import oracle as O
        from paper_2604_05182_b200.workloads import coarse_inputs, load_workload
        self.O = O
        wl = load_workload(wl_name)
        self.params = params = O.AttentionParams(32, 2, 32)
        d = params.model_dim
        x_d, y_d, pe_v, pe_i = coarse_inputs(wl, d)
        x_up, y_up = O.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v.tables,
                                              pe_i.tables, wl.factor_vol, wl.factor_img)
        pv = O.partition_tokens("volume", x_up.coords, x_up.grid_res)
        pi = O.partition_tokens("image", y_up.coords, y_up.grid_res)
        vpts = (x_up.coords.astype(np.float64) + 0.5) / wl.s_vol
        self.plan = O.build_routing_plan(vpts, wl.img_points, pv, pi, wl.cameras,
                                         dict(b_i=16, b_v2v=8, b_v2i=8, b_i2v=8, b_i2i=8))
        self.blk = O.init_sparse_block(seed, params, 0)
        ones, zeros = np.ones(d, np.float32), np.zeros(d, np.float32)
        xh = O.layer_norm(x_up.features, ones, zeros)
        yh = O.layer_norm(y_up.features, ones, zeros)
        self.uses = {"v2v": (xh, xh, pv, pv), "v2i": (xh, yh, pv, pi), "i2i": (yh, yh, pi, pi),
                     "i2v": (yh, xh, pi, pv)}
        self.n_tokens = x_up.count + y_up.count
        self.kv = {}
        self.wl_name = wl_name

    def run(self, i, n_chunks):
        """Time chunk i of n; returns (queries done, seconds)."""
        O, params = self.O, self.params
        d = params.model_dim
        done, t_total = 0, 0.0
        for name in self.USES:
            xq, xkv, pq, pk = self.uses[name]
            # contiguous query-block chunk holding ~1/n_chunks of the queries
            cut = np.searchsorted(pq.block_offsets, np.linspace(0, pq.n_tokens, n_chunks + 1))
            b0, b1 = int(cut[i]), int(cut[i + 1])
            qids = pq.block_token_ids[pq.block_offsets[min(b0, pq.n_occupied)]:
                                      pq.block_offsets[min(b1, pq.n_occupied)]]
            if qids.size == 0:
                continue
            lists = [self.plan.tables[name][j] for j in qids]
            own = pk.block_of_token[qids] if name in ("v2v", "i2i") else None
            w = self.blk.nsa[name]
            t0 = time.perf_counter()
            if name not in self.kv:
                k = O.affine(xkv, w.w_k).reshape(-1, params.n_kv_heads, params.head_dim)
                v = O.affine(xkv, w.w_v).reshape(-1, params.n_kv_heads, params.head_dim)
                self.kv[name] = (k, v) + tuple(O.compress_block_kv(k, v, pk, w.compress))
            k, v, kc, vc = self.kv[name]
            n = qids.size
            q = O.affine(xq[qids], w.w_q).reshape(n, params.n_q_heads, params.head_dim)
            outs = [O.cmp_attention(q, kc, vc, params).reshape(n, d),
                    O.sel_attention(q, k, v, pk, lists, params, own).reshape(n, d)]
            if name in ("v2v", "i2i"):
                outs.append(_win_sample(O, q, qids, k, v, pk, params).reshape(n, d))
            O.combine_branches(xq[qids], outs, w)
            t_total += time.perf_counter() - t0
            done += n
        return done, t_total


def cpu_oracle_sample(wl_name="c3", frac=1.0 / 8, seed=0):
    """Bounded sample for the GPU arm's cpu_baseline: the first 1/round(1/frac)
    query-block chunk of every use.  Returns (tokens_done, seconds, desc)."""
    lay = OracleLayer(wl_name, seed)
    n_chunks = max(1, int(round(1.0 / frac)))
    done, secs = lay.run(0, n_chunks)
    done //= 2          # queries over the four uses = 2 x layer tokens
    desc = (f"oracle 4 NSA uses, {wl_name.upper()} paper heads 32/2/32 d=1024: first of "
            f"{n_chunks} contiguous query-block chunks of every use ({2 * done} queries = {done} "
            f"layer tokens) against the full KV side, incl. the uses' K/V projections and "
            f"compression")
    return done, secs, desc


def _win_sample(O, q, qids, k, v, pk, params):
    out = np.zeros((qids.size, params.n_q_heads, params.head_dim), np.float32)
    pos = {int(t): i for i, t in enumerate(qids)}
    rows = np.unique(pk.block_of_token[qids])
    row_of = pk.row_of_block()
    for b in rows:
        t = pk.tokens_in_row(row_of[int(b)])
        o = O.dense_attention(q[[pos[int(x)] for x in t]], k[t], v[t], params)
        for j, x in enumerate(t):
            out[pos[int(x)]] = o[j]
    return out


def host_info():
    info = {"cpu_count": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    info["cpu_model"] = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas_threads"] = [p.get("num_threads") for p in threadpool_info()]
    except Exception:
        pass
    return info


def run_reference(args):
    """The reference algorithm on the host cores (oracle port), on the SAME
    workload as our arm: the K timed steps are K contiguous query-block
    chunks that together cover the full layer exactly once (same_config);
    value = the layer's tokens / the summed step times."""
    rank, _, ws = dist_env()
    if rank != 0:
        return
    # the same workload our arm runs at this N (C3 on one GPU, C4 under torchrun)
    wl_name = args.workload or ("c4" if ws > 1 else "c3")
    # every host thread (torchrun sets OMP_NUM_THREADS=1 for its workers)
    from threadpoolctl import threadpool_limits
    lay = OracleLayer(wl_name)
    times, tokens = [], 0
    with threadpool_limits(limits=os.cpu_count()):
        for _ in range(args.warmup):            # untimed: a thin slice of the layer
            OracleLayer.run(lay, 0, 512)
        lay.kv.clear()
        for i in range(args.steps):
            done, secs = lay.run(i, args.steps)
            tokens += done
            times.append(secs)
        hi = host_info()
    # every token is the query of two uses (v2v + v2i, or i2i + i2v)
    assert tokens == 2 * lay.n_tokens, (tokens, lay.n_tokens)
    tokens = lay.n_tokens
    total = float(np.sum(times))
    v = tokens / total
    desc = (f"oracle port of the reference's 4 gated NSA uses (NumPy f64), full {wl_name.upper()} "
            f"layer ({tokens} queries, paper heads 32/2/32, d=1024) split into {args.steps} "
            f"contiguous query-block chunks, one per timed step; {total:.1f} s total")
    line = {"impl": "reference", "metric": "LSRM sparse-attn layer tokens/s",
            "value": v, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference fixture geometry, tagged Philox features/weights)",
            "config": {"workload": WORKLOAD_DESC.get(wl_name, wl_name),
                       "parallelism": "cpu (host cores)", "sample": desc, "same_config": True,
                       "layer_seconds": total},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": hi["cpu_count"],
                             "kind": "port", "sample": desc, "host": hi},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


def run_gpu(args):
    import torch
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import _dev as D
    from paper_2604_05182_b200._native import launch_count, reset_launch_count
    from paper_2604_05182_b200.layer import SparseAttentionLayer, build_instance

    rank, local_rank, ws = dist_env()
    torch.cuda.set_device(local_rank % torch.cuda.device_count())   # gloo tests share a GPU
    if ws > 1:
        return run_sp(args)
    wl_name = args.workload or "c3"
    inst = build_instance(wl_name)
    layer = SparseAttentionLayer(inst)
    x_bm, y_bm = layer.device_inputs(inst.x_hat, inst.y_hat)
    n_tok = inst.n_vol + inst.n_img
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        layer.engine.forward(x_bm, y_bm)
    torch.cuda.synchronize()
    reset_launch_count()
    layer.engine.forward(x_bm, y_bm)      # own-kernel launches per step (cuBLAS excluded)
    per_step_launches = launch_count()
    use_graph = not args.no_graph
    if use_graph:
        try:
            layer.engine.capture(x_bm, y_bm)
        except Exception as exc:  # report, fall back to eager launches
            print(f"# CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            use_graph = False
    step = layer.engine.replay if use_graph else (lambda: layer.engine.forward(x_bm, y_bm))
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    # -- timed region: K steps, device events per step, L2 flushed in between
    sampler = ClockSampler(local_rank)
    sampler.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(st)
        step()
        evs[i][1].record(st)
    torch.cuda.synchronize()
    launches = per_step_launches * args.steps
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(step_ms))
    # -- per-kernel breakdown (separate pass, events on the launching stream)
    brk = layer.profile_breakdown(x_bm, y_bm, reps=max(3, args.steps))
    clocks = sampler.stop()
    # -- end to end through the reference-facing call (NumPy host buffers)
    api_ms, api_h2d, api_d2h = time_reference_api(inst, args.steps)
    # -- and through the package's pipelined host API (pinned host buffers)
    e2e_ms, h2d, d2h = layer.time_host_path(inst.x_hat, inst.y_hat, steps=args.steps)
    pcie = pcie_bandwidth()
    # e2e roofline: the duplex copy of one step's inputs and outputs
    # a true lower bound on the step: each direction's bytes at that
    # direction's best standalone rate (the pipeline overlaps the two)
    e2e_bound_ms = max(h2d / (pcie["h2d_gbps"] * 1e9), d2h / (pcie["d2h_gbps"] * 1e9)) * 1e3
    e2e_duplex_ms = max(h2d / (pcie["duplex_h2d_gbps"] * 1e9),
                        d2h / (pcie["duplex_d2h_gbps"] * 1e9)) * 1e3
    peaks, src = load_peaks()
    attn_flops = sum(sum(v.values()) for v in layer.engine.attention_flops().values())
    attn_ms = brk["attention_ms"]
    achieved = attn_flops / (attn_ms * 1e-3) / 1e12
    peak = float(peaks["bf16_tflops"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "attention_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get("bytes_per_launch")
    cpu = None
    if not args.no_cpu_baseline:
        tok, secs, desc = cpu_oracle_sample(frac=args.ref_frac)
        hi = host_info()
        cpu = {"value": tok / secs, "unit": "tokens/s", "cores": hi["cpu_count"],
               "kind": "port", "sample": desc,
               "note": "bounded sample; `bench.py --impl reference` times the full layer"}
    proj_flops = layer.engine.projection_flops()
    block = time_sparse_block(inst, n_tok, args.steps)
    # (C5: ≈ 370 ms per step, 67 GB peak; a few seconds with the warm-ups)
    train = time_train_step(inst)
    setup = time_setup(wl_name) if wl_name in ("c3", "c4") else None
    c1 = time_c1_fp32(max(5, args.steps)) if wl_name == "c3" else None
    line = {
        "metric": "LSRM sparse-attn layer tokens/s", "value": n_tok / (ms * 1e-3),
        "unit": "tokens/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (reference fixture geometry, tagged Philox features/weights)",
        "config": {"workload": WORKLOAD_DESC.get(wl_name, wl_name),
                   "n_vol": inst.n_vol, "n_img": inst.n_img, "global_batch": n_tok,
                   "parallelism": "single GPU", "l2": "flushed (256 MiB write) between steps",
                   "cuda_graph": use_graph},
        "roofline": {"bound": "tensor", "kernel": "nsa_fused_kernel (one launch per step: four uses, LPT queue)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"{src} bf16_tflops (burst)",
                     "algorithmic_flops_per_step": attn_flops,
                     # d_h = 32: 4*d_h flops per (row, key) pair against one exp2 on
                     # the MUFU (16/clk/SM), so the special-function unit binds first
                     "mufu": mufu_roofline(attn_flops, attn_ms, layer.inst.params, peaks)},
        "breakdown_ms": brk,
        "layer_tflops": (attn_flops + proj_flops) / (ms * 1e-3) / 1e12,
        "sparse_block": block,
        "train_step": train,
        "setup_kernels": setup,
        "c1_fp32": c1,
        "cpu_baseline": cpu,
        "e2e": {"value": n_tok / (api_ms * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": api_h2d, "d2h_bytes_per_step": api_d2h,
                "ms_per_step": api_ms,
                "what": "reference-API nsa_cross_attention x 4 uses (drop-in precision='bf16'), "
                        "NumPy f32 host buffers in and out, wall clock per layer",
                "pcie_bound_ms": max(api_h2d / (pcie["h2d_gbps"] * 1e9),
                                     api_d2h / (pcie["d2h_gbps"] * 1e9)) * 1e3},
        "e2e_pipelined": {"value": n_tok / (e2e_ms * 1e-3), "unit": "tokens/s",
                "what": "package host API layer.HostPipeline: pinned f32 in/out, H2D / compute / "
                        "D2H on separate streams, two steps in flight",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "roofline": {"bound": "pcie", "pcie_measured": pcie,
                             "bound_ms": e2e_bound_ms, "frac": e2e_bound_ms / e2e_ms,
                             "duplex_copy_ms": e2e_duplex_ms,
                             "bound_note": "slower direction's bytes at its best standalone "
                                           "pinned-copy rate"}},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def time_c1_fp32(steps):
    """BASELINE config 1 (C1: 4 views, desk heads 8/1/8, d = 64, fp32 fwd,
    1 GPU): the reference-API layer on the fp32 path the C1 oracle pins
    (≤1e-5): four `nsa_cross_attention` calls on device-resident f32 inputs
    (fp32 projections, f64-sum compression, CUDA-core fp32 attention). Device
    events around each layer. The bf16 engine does not take d_h = 8."""
    import torch
    from paper_2604_05182_b200 import _dev as D
    from paper_2604_05182_b200.layer import build_instance
    from paper_2604_05182_b200.nsa_attention import (GatherTable, Selection, nsa_cross_attention,
                                                     resolve_rows)
    from paper_2604_05182_b200.engine import SparseLayerEngine  # noqa: F401 (native lib loaded)
    inst = build_instance("c1")
    p = inst.params
    parts = {"x": inst.part_vol, "y": inst.part_img}
    feats = {"x": D.dev(inst.x_hat), "y": D.dev(inst.y_hat)}
    geom = {"v2v": ("x", "x"), "v2i": ("x", "y"), "i2i": ("y", "y"), "i2v": ("y", "x")}
    tables = {}
    for use, (qs, ks) in geom.items():
        r, c = inst.plan_rows[use]
        own = parts[ks].block_of_token if qs == ks else None
        rr, cc, lens, _, _ = resolve_rows(r, c, parts[ks], own, True)
        rh, ch = D.host(r), D.host(c)
        sel = Selection([parts[ks].occupied_ids[rh[i, :ch[i]]] for i in range(rh.shape[0])])
        tables[use] = (GatherTable(None, None, D.host(lens), rr, cc), lens, sel)

    def layer():
        return {use: nsa_cross_attention(feats[qs], feats[ks], parts[qs], parts[ks],
                                         tables[use][2], inst.weights[use], p,
                                         table=tables[use][0])
                for use, (qs, ks) in geom.items()}
    for _ in range(3):
        layer()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ms = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        layer()
        b.record(st)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = float(np.median(ms))
    n_tok = inst.n_vol + inst.n_img
    # algorithmic attention-core FLOPs, useful work only
    flops = 0.0
    for use, (qs, ks) in geom.items():
        pk, pq = parts[ks], parts[qs]
        nq = pq.n_tokens
        L_ = float(D.host(tables[use][1]).sum())
        flops += 4.0 * p.n_q_heads * p.head_dim * (nq * pk.n_occupied + L_)
        if qs == ks:
            flops += 4.0 * p.n_q_heads * p.head_dim * float((pq.occupancy.astype(np.float64) ** 2).sum())
    # fp32 FFMA peak: 148 SMs x 128 lanes x 2 flops x 1.965 GHz
    peak = 148 * 128 * 2 * 1.965e9 / 1e12
    return {"workload": WORKLOAD_DESC["c1"], "n_vol": inst.n_vol, "n_img": inst.n_img,
            "ms_per_layer": t, "tokens_per_s": n_tok / (t * 1e-3), "dtype": "fp32",
            "attention_flops": flops, "attention_tflops_incl_projections_time": flops / (t * 1e-3) / 1e12,
            "fp32_peak_tflops": peak,
            "what": "reference-API nsa_cross_attention x 4 uses, fp32 path (<=1e-5 of the "
                    "reference at C1), device-resident inputs, CUDA events, median of steps"}


def time_reference_api(inst, steps):
    """e2e through the reference-facing call: the drop-in's precision="bf16"
    `nsa_cross_attention` (the reference's signature, `lsrm/nsa_attention.py:287`)
    called for the four uses of the layer with NumPy f32 host buffers in and
    out, as `lsrm.recon_pipeline._nsa_use` calls it (`recon_pipeline.py:451-458`).
    Each call copies its host inputs to the device, runs the one-use bf16
    engine (cached across calls, like a reference user's repeated calls) and
    returns a fresh NumPy array. Returns (ms per layer, h2d B, d2h B)."""
    import torch
    from paper_2604_05182_b200 import _dev as D, fastpath
    from paper_2604_05182_b200.nsa_attention import Selection, nsa_cross_attention
    pv, pi = inst.part_vol, inst.part_img
    parts = {"x": pv, "y": pi}
    feats = {"x": np.ascontiguousarray(inst.x_hat, np.float32),
             "y": np.ascontiguousarray(inst.y_hat, np.float32)}
    geom = {"v2v": ("x", "x"), "v2i": ("x", "y"), "i2i": ("y", "y"), "i2v": ("y", "x")}
    sels = {}
    for use, (qs, ks) in geom.items():
        r, c = (D.host(t) for t in inst.plan_rows[use])
        occ = parts[ks].occupied_ids
        sels[use] = Selection([occ[r[i, :c[i]]] for i in range(r.shape[0])])
    fastpath.set_precision("bf16")
    try:
        def layer():
            outs = {}
            for use, (qs, ks) in geom.items():
                outs[use] = nsa_cross_attention(feats[qs], feats[ks], parts[qs], parts[ks],
                                                sels[use], inst.weights[use], inst.params)
            return outs
        outs = layer()                     # engine build + warm-up (not timed), in the
        outs = layer()                     # timed loop's pattern: the previous layer's
        outs = layer()                     # outputs are alive while the next is computed
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            outs = layer()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / steps
    finally:
        fastpath.set_precision("fp32")
    # bytes each step moves: every call uploads its query rows and (cross
    # uses) its key rows; self uses pass one buffer, uploaded once
    h2d = sum(feats[qs].nbytes + (feats[ks].nbytes if qs != ks else 0)
              for qs, ks in geom.values())
    d2h = sum(o.nbytes for o in outs.values())
    return ms, h2d, d2h


def time_setup(wl_name, reps=5):
    """The instance-setup kernels of the path: voxel
    mask, foreground patch mask, compaction, partition, the four routing
    tables. Each public call is timed with CUDA events (median of reps, after
    a warm-up call) on device-resident inputs; achieved GB/s uses the
    algorithmic bytes of §8d against the measured HBM peak (these are
    HBM/latency-bound integer kernels, run once per instance)."""
    import torch
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import _dev as D
    from paper_2604_05182_b200.block_routing import (ImageSide, RoutingBudgets,
                                                     route_image_rows, route_volume_rows,
                                                     volume_token_coords)
    from paper_2604_05182_b200.camera_geometry import silhouettes
    from paper_2604_05182_b200.workloads import (SCENE, coarse_inputs, load_workload,
                                                 orbit_cameras, params_of)
    peaks, _ = load_peaks()
    hbm = float(peaks.get("hbm_gbs", 7700.0))
    wl = load_workload(wl_name)
    d = params_of(wl_name).model_dim
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, d)
    xd, yd = D.dev(x_d), D.dev(y_d)
    cams = orbit_cameras(wl.views, 1.7, 20.0, (8 * wl.s_img, 8 * wl.s_img))
    alpha = silhouettes(SCENE, cams, as_device=True)
    vm, im = D.dev(wl.vol_mask), D.dev(wl.img_mask)
    st = torch.cuda.current_stream()

    def timed(fn):
        out = fn()
        torch.cuda.synchronize()
        ms = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            out = fn()
            b.record(st)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        return float(np.median(ms)), out

    def entry(ms, nbytes, what):
        gbps = nbytes / (ms * 1e-3) / 1e9
        return {"ms": ms, "bytes": int(nbytes), "gbps": gbps, "frac_hbm": gbps / hbm, "what": what}

    res = {}
    t, _ = timed(lambda: L.informative_voxel_mask(SCENE, wl.s_vol, as_device=True))
    res["voxel_mask"] = entry(t, wl.s_vol ** 3, f"S={wl.s_vol}: 64 analytic-SDF samples per voxel, "
                                                "S^3 bytes written (compute-bound)")
    v, h, w = (int(s) for s in alpha.shape)
    t, _ = timed(lambda: L.foreground_patch_mask(alpha))
    res["foreground_mask"] = entry(t, 4 * v * h * w + v * (h // 8) * (w // 8),
                                   f"{v} views x {h}x{w} f32 alpha read, patch mask written")
    t, (x_up, y_up) = timed(lambda: L.upsample_select_tokens(xd, yd, vm, im, pe_v, pe_i,
                                                             wl.factor_vol, wl.factor_img))
    n = x_up.count + y_up.count
    res["compaction"] = entry(t, n * (4 * d + 12) + n * 4 * d,
                              f"{n} tokens x d={d}: features + coords written, parents read; "
                              "public call incl. mask scans and the token-count readback")
    # the compaction's row kernels alone (no mask scan, no host readback):
    # N x (4d + 24) written, N x 4d parent rows read
    from paper_2604_05182_b200.tokenizer import _compact_rows, _compact_scan
    tv = [D.weight(t) for t in pe_v.tables]
    ti = [D.weight(t) for t in pe_i.tables]
    vm8, im8 = vm.to(torch.uint8), im.to(torch.uint8)
    ws_v, nc_v, n_v = _compact_scan("volume", vm8, 1, wl.vol_mask.shape[0], wl.factor_vol)
    ws_i, nc_i, n_i = _compact_scan("image", im8, wl.img_mask.shape[0], wl.img_mask.shape[1],
                                    wl.factor_img)
    cv, fv = D.empty((n_v, 3), torch.int64), D.empty((n_v, d), torch.float32)
    ci, fi = D.empty((n_i, 3), torch.int64), D.empty((n_i, d), torch.float32)

    def rows():
        _compact_rows("volume", ws_v, nc_v, n_v, xd, d, tv, 1, wl.vol_mask.shape[0],
                      wl.factor_vol, cv, fv)
        _compact_rows("image", ws_i, nc_i, n_i, yd, d, ti, wl.img_mask.shape[0],
                      wl.img_mask.shape[1], wl.factor_img, ci, fi)
    t, _ = timed(rows)
    res["compaction_rows"] = entry(t, (n_v + n_i) * (8 * d + 24),
                                   "compaction row kernels alone (cell lists from the scan): "
                                   "features + coords written, parent rows read")
    # BASELINE config 2 on DECODED geometry (the paper's coarse-to-fine
    # scoring, `lsrm/runner.py:301-311`): coarse tokens -> dense feature grid
    # -> Eq. 11 on the decoded SDF (4^3 samples per fine voxel, each a
    # trilinear feature lookup + the SDF head, in-kernel)
    from paper_2604_05182_b200.recon_pipeline import (decode_feature_volume, init_decode,
                                                      init_decoder_heads)
    from paper_2604_05182_b200.sdf import decoded_sdf_field
    dw = init_decode(0, d, "dec_coarse")
    t_dec, grid = timed(lambda: decode_feature_volume(xd, dw))
    res["decode_grid"] = entry(t_dec, int(xd.numel()) * 4 + grid.numel() * 4,
                               f"coarse tokens {tuple(xd.shape)} -> dense grid "
                               f"{tuple(grid.shape)} f32 (f64 affine, einsum order)")
    field = decoded_sdf_field(grid, init_decoder_heads(0))
    t_vmd, vmd = timed(lambda: L.informative_voxel_mask(field, wl.s_vol, as_device=True))
    res["voxel_mask_decoded"] = entry(t_vmd, grid.numel() * 4 + wl.s_vol ** 3,
                                      f"S={wl.s_vol}: 64 decoded-SDF samples per voxel "
                                      f"(grid read, S^3 bytes written; f64, compute-bound)")
    res["voxel_mask_decoded"]["informative_voxels"] = int(D.host(vmd).sum())
    coarse_ms = (t_dec + t_vmd + res["foreground_mask"]["ms"] + res["compaction"]["ms"])
    res["coarse_stage"] = {
        "ms": coarse_ms, "tokens": int(n), "tokens_per_s": n / (coarse_ms * 1e-3),
        "what": "BASELINE config 2: decode grid + decoded-SDF voxel informativeness + "
                f"foreground pruning ({v} views) + compaction (d={d}); sum of the public calls"}
    t, pv = timed(lambda: L.partition(x_up))
    _, pi = timed(lambda: L.partition(y_up))
    res["partition_volume"] = entry(t, x_up.count * 16, "N x 16 B (incl. host metadata copy)")
    vp = D.dev(volume_token_coords(x_up).points)
    ip = D.dev(wl.img_points)
    bud = RoutingBudgets()
    t, _ = timed(lambda: route_volume_rows(vp, pv, bud.b_v2v))
    res["route_v2v"] = entry(t, x_up.count * 24 + pv.n_occupied * 24 + x_up.count * bud.b_v2v * 4,
                             "points + centers read, rows written (bit-exact f64)")
    t, side = timed(lambda: ImageSide(pi, ip, wl.cameras))
    res["route_image_side"] = entry(t, y_up.count * 24 * 2 + pi.n_occupied * 48,
                                    "image-router prep, once per plan: block-major SoA token "
                                    "points + per-block bounding boxes")
    for name, qp, nq_, b in (("route_v2i", vp, x_up.count, bud.b_v2i),
                             ("route_i2i", ip, y_up.count, bud.b_i2i)):
        t, _ = timed(lambda: route_image_rows(qp, wl.cameras, pi, ip, bud.b_i, b, side))
        res[name] = entry(t, nq_ * 24 + pi.n_occupied * 24 + y_up.count * 24 + nq_ * b * 4,
                          "two-stage image rule: projection top-b_i + 3D min-distance "
                          "ranking with exact box pruning (bit-exact f64; latency/compute-bound)")
    return res


def time_train_step(inst, steps=3):
    """Training step of one full Stage-2 block (SURVEY §8f ranks 1-2,
    BASELINE config 5's fwd+bwd at one layer): training.SparseBlockModule,
    fast path (bf16 tensor-core branches and tcgen05 GEMMs, fp32 master weights):
    add + LayerNorm, use gates, the four NSA uses, gated mixture +
    LayerNorm, FFN, residuals; loss = sum of squares of both outputs; then
    one Adam step. Device events around forward, backward and the step."""
    import torch
    from paper_2604_05182_b200.recon_pipeline import init_sparse_block
    from paper_2604_05182_b200.training import SparseBlockModule, resolve_plan_rows
    res = resolve_plan_rows(inst.plan_rows, inst.part_vol, inst.part_img)
    mod = SparseBlockModule(inst.params, weights=init_sparse_block(0, inst.params, 0),
                            fast_backward=True)
    opt = torch.optim.Adam(mod.parameters(), lr=1e-4)
    x = torch.tensor(inst.x_hat, device="cuda", requires_grad=True)
    y = torch.tensor(inst.y_hat, device="cuda", requires_grad=True)
    xi, yi = (0.1 * x).detach(), (0.1 * y).detach()

    def fwd():
        x2, y2 = mod(x, y, xi, yi, inst.part_vol, inst.part_img, res)
        return (x2 * x2).sum() + (y2 * y2).sum()
    for _ in range(3):   # warm-up (lazy module loading of the sort kernels, allocator)
        opt.zero_grad()
        fwd().backward()
        opt.step()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    fw, bw, op = [], [], []
    for _ in range(steps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        opt.zero_grad()
        e[0].record(st)
        loss = fwd()
        e[1].record(st)
        loss.backward()
        e[2].record(st)
        opt.step()
        e[3].record(st)
        torch.cuda.synchronize()
        fw.append(e[0].elapsed_time(e[1]))
        bw.append(e[1].elapsed_time(e[2]))
        op.append(e[2].elapsed_time(e[3]))
    f, b, o = float(np.mean(fw)), float(np.mean(bw)), float(np.mean(op))
    n_tok = inst.n_vol + inst.n_img
    return {"ms_per_step": f + b + o, "forward_ms": f, "backward_ms": b, "optimizer_ms": o,
            "tokens_per_s": n_tok / ((f + b + o) * 1e-3),
            "what": "one full Stage-2 block (4 gated NSA uses + add/LN, use gates, gated "
                    "mixture/LN, FFN 4d, residuals): fwd + bwd + Adam step; attention forward "
                    "on the fused tcgen05 kernel (branches, lse and gated merge in one launch "
                    "per use), backward on bf16 mma.sync, bf16 tcgen05 GEMMs (fp32 "
                    "accumulation, MN-major weight-gradient operands), fp32 master weights"}


def pcie_bandwidth(sizes=(64 << 20, 128 << 20, 256 << 20), reps=5):
    """Pinned host <-> device copy bandwidth on this box (GB/s): H2D alone,
    D2H alone, and both directions at once (the e2e pipeline overlaps them),
    each the BEST over several sizes and repetitions, so the bound the e2e
    number is compared with is not under-measured by a slow sample."""
    import torch
    nmax = max(sizes)
    h_in = torch.empty(nmax, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nmax, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nmax, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nmax, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def gbps(n, fn_list):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            evs = []
            for s, fn in fn_list:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    a.record(s)
                    fn(n)
                    b.record(s)
                evs.append((a, b))
            torch.cuda.synchronize()
            bw = [n / 1e9 / (a.elapsed_time(b) * 1e-3) for a, b in evs]
            best = bw if best is None else [max(x, y) for x, y in zip(best, bw)]
        return best
    h2d = lambda n: d_a[:n].copy_(h_in[:n], non_blocking=True)    # noqa: E731
    d2h = lambda n: h_out[:n].copy_(d_b[:n], non_blocking=True)   # noqa: E731
    out = {"h2d_gbps": 0.0, "d2h_gbps": 0.0, "duplex_h2d_gbps": 0.0, "duplex_d2h_gbps": 0.0}
    for n in sizes:
        out["h2d_gbps"] = max(out["h2d_gbps"], gbps(n, [(s1, h2d)])[0])
        out["d2h_gbps"] = max(out["d2h_gbps"], gbps(n, [(s1, d2h)])[0])
        both = gbps(n, [(s1, h2d), (s2, d2h)])
        out["duplex_h2d_gbps"] = max(out["duplex_h2d_gbps"], both[0])
        out["duplex_d2h_gbps"] = max(out["duplex_d2h_gbps"], both[1])
    out["how"] = f"best of {reps} reps x sizes {[n >> 20 for n in sizes]} MiB, pinned host memory"
    return out


def time_sparse_block(inst, n_tok, steps):
    """The full Stage-2 block around the four uses (injection + LayerNorm,
    use-gate mixture, FFN 4d, residuals; recon_pipeline.py:461-497) on the
    bf16 engine, CUDA graph, device events, L2 flushed between steps.
    Reported next to the layer metric."""
    import torch
    from paper_2604_05182_b200 import _dev as D, _ops
    from paper_2604_05182_b200.recon_pipeline import SparseBlockEngine, init_sparse_block
    w = init_sparse_block(0, inst.params, 0)
    eng = SparseBlockEngine(inst.part_vol, inst.part_img, inst.plan_rows, w, inst.params)
    d = inst.params.model_dim
    g = torch.Generator(device="cuda").manual_seed(0)
    ins = [torch.randn((n, d), generator=g, device="cuda", dtype=torch.float32)
           for n in (inst.n_vol, inst.n_img, inst.n_vol, inst.n_img)]
    st = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(st)
    with torch.cuda.stream(side):
        eng.forward(*ins)
    st.wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        eng.forward(*ins)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for a, b in evs:
        flush.zero_()
        a.record(st)
        graph.replay()
        b.record(st)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    ffn_flops = 2.0 * n_tok * d * 4 * d * 2
    gate_flops = 2.0 * n_tok * d * 2 * d
    return {"ms_per_step": ms, "tokens_per_s": n_tok / (ms * 1e-3),
            "what": "one Stage-2 sparse block: 4 gated NSA uses + injection/LayerNorm, "
                    "use-gate mixture, FFN 4d (erf gelu), residuals; bf16 engine",
            "ffn_and_gate_gflop": (ffn_flops + gate_flops) / 1e9}


def mufu_roofline(attn_flops, attn_ms, params, peaks):
    """Exponentials of the useful (row, key) pairs (4*d_h flops each) per second
    against the MUFU ex2 peak (16 per clock per SM, measured in
    tools/microbench.cu) x SMs x max SM clock."""
    import torch
    exps = attn_flops / (4.0 * params.head_dim)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    peak = 16.0 * n_sm * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    ach = exps / (attn_ms * 1e-3)
    return {"achieved": ach / 1e9, "peak": peak / 1e9, "unit": "Gexp/s", "frac": ach / peak}


WORKLOAD_DESC = {
    "c3": "C3 fine stage: 16 views, S_vol=S_img=96, heads 32/2/32, d=1024, 3D routing b_i=16 "
          "budgets 8, one layer = 4 gated NSA uses",
    "c4": "C4 SP stress: C3 + 12 fully occupied 8^3 volume blocks (skewed per-block sparsity), "
          "heads 32/2/32, d=1024, one layer = 4 gated NSA uses",
    "c1": "C1 tiny: 4 views, S_vol=32, S_img=96, heads 8/1/8, d=64",
    "c5": "C5 scaled context: 18 views, S_vol=408, S_img=288 (fixture scene, masks and points "
          "generated on the GPU), heads 32/2/32, d=1024, one layer = 4 gated NSA uses",
}


def run_sp(args):
    """N>1 (torchrun, one rank per GPU): block-aware sequence parallelism.
    Strong scaling on the C4 skewed workload: every rank builds the same
    instance, owns the query blocks LPT assigns it (routed-block workload),
    all-gathers K/V per use over NCCL (grouped send/recv) and attends its own
    queries.  Timed on the device, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2604_05182_b200._native import launch_count, reset_launch_count
    from paper_2604_05182_b200.layer import build_instance
    from paper_2604_05182_b200 import seq_parallel as S

    rank, local_rank, ws = dist_env()
    backend = args.sp_backend
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        transport = S.NcclTransport(rank, ws)
        red_dev = torch.device("cuda", local_rank)
    else:   # gloo: several ranks may share one GPU (tests)
        dist.init_process_group("gloo")
        transport = S.HostStagedTransport(rank, ws)
        red_dev = torch.device("cpu")

    def max_all(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_all(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    wl_name = args.workload or "c4"
    inst = build_instance(wl_name)
    n_tok = inst.n_vol + inst.n_img
    sl = S.ShardedLayer(inst, rank, ws, transport=transport, by_cost=not args.token_lpt)
    x_loc, y_loc = sl.local_inputs(inst.x_hat, inst.y_hat)
    for _ in range(args.warmup):
        sl.forward(x_loc, y_loc)
    torch.cuda.synchronize()
    reset_launch_count()
    sl.forward(x_loc, y_loc)
    per_step_launches = launch_count()
    use_graph = not args.no_graph
    if use_graph:
        try:
            sl.capture(x_loc, y_loc)
        except Exception as exc:
            print(f"# rank {rank}: CUDA graph capture failed ({exc}); eager", file=sys.stderr)
            use_graph = False
    if not max_all(0.0 if use_graph else 1.0) == 0.0:
        use_graph = False            # all ranks must take the same path
    step = sl.step if use_graph else (lambda: sl.forward(x_loc, y_loc))
    for _ in range(2):
        step()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st)
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(st)
        step()
        evs[i][1].record(st)
    t1.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms_local = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    ms = max_all(ms_local)
    attn_ms = max_all(sl.attention_ms(reps=max(3, args.steps)))
    flops = sum(sum(v.values()) for v in sl.engine.attention_flops().values())
    total_flops = sum_all(flops)
    e2e_local, h2d, d2h = sl.time_host_path(inst.x_hat, inst.y_hat, steps=args.steps)
    e2e_ms = max_all(e2e_local)
    h2d_all, d2h_all = sum_all(h2d), sum_all(d2h)
    launches = int(sum_all(per_step_launches * args.steps))
    loads = np.asarray(sl.topology.loads, np.float64)
    # NVLink bytes of the All-gather-KV: every rank sends its packed shard
    # [k_il | v_il | k_cmp | v_cmp] of every use to every other rank
    sent = sum(int(sl.exchange.packed[u].numel()) for u in sl.exchange.packed) * (ws - 1)
    sent_all = sum_all(sent)
    # the whole sequence-parallel stage (dispatch -> depth blocks -> return)
    sp_stage = None
    if args.sp_stage_depth > 0:
        from paper_2604_05182_b200.recon_pipeline import init_sparse_block
        wts = [init_sparse_block(0, inst.params, m) for m in range(args.sp_stage_depth)]
        stg = S.ShardedStage(inst.part_vol, inst.part_img, inst.plan_rows, wts, inst.params,
                             rank, ws, topology=sl.topology, transport=transport)
        tk = stg.tokens
        lo = int(np.concatenate([[0], np.cumsum([a.size for a in tk.naive])])[rank])
        feats = np.concatenate([inst.x_hat, inst.y_hat])[lo:lo + tk.n_naive]
        from paper_2604_05182_b200 import _dev as D
        fn, cn = D.dev(np.ascontiguousarray(feats, np.float32)), D.zeros((tk.n_naive, 3), torch.int32)
        for _ in range(2):
            stg.forward(fn, cn)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(max(2, args.steps // 4)):
            stg.forward(fn, cn)
        b.record(st)
        torch.cuda.synchronize()
        stage_ms = max_all(a.elapsed_time(b) / max(2, args.steps // 4))
        sp_stage = {"depth": args.sp_stage_depth, "ms_per_stage": stage_ms,
                    "tokens_per_s": n_tok / (stage_ms * 1e-3),
                    "what": "ShardedStage: dispatch all_to_all_v (features + coords) -> "
                            f"{args.sp_stage_depth} sharded Stage-2 blocks (per-use "
                            "All-gather-KV) -> return all_to_all_v; eager, max over ranks"}
    # one Stage-2 block TRAINING step under the same sharding (BASELINE
    # config 5's step): fwd + bwd with per-use All-gather-KV and its adjoint,
    # parameter gradients summed over ranks, Adam; max over ranks
    sp_train = None
    if args.sp_train_steps > 0:
        from paper_2604_05182_b200 import _dev as D
        from paper_2604_05182_b200.recon_pipeline import init_sparse_block
        from paper_2604_05182_b200.training import SparseBlockModule, resolve_plan_rows
        res = resolve_plan_rows(inst.plan_rows, inst.part_vol, inst.part_img)
        shard = S.training_shard(inst.part_vol, inst.part_img, sl.topology, rank, transport)
        mod = SparseBlockModule(inst.params, weights=init_sparse_block(0, inst.params, 0),
                                fast_backward=True)
        opt = torch.optim.Adam(mod.parameters(), lr=1e-4)
        lx = torch.as_tensor(shard["x"].queries.loc_tok, device="cuda")
        ly = torch.as_tensor(shard["y"].queries.loc_tok, device="cuda")
        xl = D.dev(inst.x_hat)[lx].requires_grad_(True)
        yl = D.dev(inst.y_hat)[ly].requires_grad_(True)
        xi, yi = (0.1 * xl).detach(), (0.1 * yl).detach()

        def train_step():
            opt.zero_grad()
            x2, y2 = mod(xl, yl, xi, yi, inst.part_vol, inst.part_img, res, shard=shard)
            ((x2 * x2).sum() + (y2 * y2).sum()).backward()
            S.allreduce_grads(list(mod.parameters()), host_staged=backend != "nccl")
            opt.step()
        for _ in range(2):
            train_step()
        torch.cuda.synchronize()
        dist.barrier()
        n_tr = args.sp_train_steps
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(n_tr):
            train_step()
        b.record(st)
        torch.cuda.synchronize()
        tr_ms = max_all(a.elapsed_time(b) / n_tr)
        moved = sum_all(shard["x"].exchange.bytes_moved + shard["y"].exchange.bytes_moved)
        sp_train = {"ms_per_step": tr_ms, "tokens_per_s": n_tok / (tr_ms * 1e-3),
                    "exchange_bytes_per_step": moved / (n_tr + 2),
                    "what": "one Stage-2 block training step under block-aware SP: each rank "
                            "its own query blocks, per-use All-gather-KV of K/V rows and its "
                            "adjoint (partial dK/dV summed at owners), gradients all-reduced, "
                            "Adam; fused tcgen05 forward, bf16 backward; max over ranks"}
    single = None
    if not args.no_single_compare:
        # the same workload on ONE GPU (rank 0), same timing rules: the
        # denominator for strong-scaling efficiency on THIS workload
        if rank == 0:
            from paper_2604_05182_b200.layer import SparseAttentionLayer
            layer = SparseAttentionLayer(inst)
            xb, yb = layer.device_inputs(inst.x_hat, inst.y_hat)
            for _ in range(args.warmup):
                layer.engine.forward(xb, yb)
            layer.engine.capture(xb, yb)
            e = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)]
            for i in range(args.steps):
                flush.zero_()
                e[i][0].record(st)
                layer.engine.replay()
                e[i][1].record(st)
            torch.cuda.synchronize()
            ms1 = float(np.mean([a.elapsed_time(b) for a, b in e]))
            single = {"value": n_tok / (ms1 * 1e-3), "ms_per_step": ms1}
        dist.barrier()
    peaks, src = load_peaks()
    peak = float(peaks["bf16_tflops"]) * ws
    achieved = total_flops / (attn_ms * 1e-3) / 1e12
    if rank == 0:
        line = {
            "metric": "LSRM sparse-attn layer tokens/s", "value": n_tok / (ms * 1e-3),
            "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference fixture geometry, tagged Philox features/weights)",
            "config": {"workload": WORKLOAD_DESC.get(wl_name, wl_name),
                       "n_vol": inst.n_vol, "n_img": inst.n_img, "global_batch": n_tok,
                       "parallelism": f"sp{ws}: block-aware sequence parallelism, "
                                      f"{'token' if args.token_lpt else 'routed-workload'} LPT, "
                                      f"All-gather-KV per use ({backend} grouped send/recv)",
                       "makespan_ratio": float(loads.max() / loads.mean()) if loads.sum() else 1.0,
                       "l2": "flushed (256 MiB write) between steps", "cuda_graph": use_graph},
            "roofline": {"bound": "tensor", "kernel": "nsa_fused_kernel (one launch per step per rank: four uses, LPT queue)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "peak_source": f"{src} bf16_tflops x {ws} GPUs",
                         "algorithmic_flops_per_step": total_flops,
                         "attention_ms_max_over_ranks": attn_ms},
            "single_gpu_same_workload": single,
            "exchange": {"all_gather_kv_bytes_per_step": int(sent_all),
                         "per_rank_sent_bytes_per_step": int(sent),
                         "what": "packed bf16 K/V + f32 compressed rows of the 4 uses, "
                                 "(W-1) peers per rank"},
            "sp_stage": sp_stage,
            "sp_train": sp_train,
            "cpu_baseline": None,
            "e2e": {"value": n_tok / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(h2d_all), "d2h_bytes_per_step": int(d2h_all),
                    "ms_per_step": e2e_ms},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-frac", type=float, default=1.0 / 8,
                    help="cpu_baseline sample of our arm (the reference arm runs the full layer)")
    ap.add_argument("--warmup-ref", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches")
    ap.add_argument("--workload", default=None, choices=["c1", "c3", "c4", "c5"],
                    help="default: c3 at N=1, c4 (skewed) under torchrun N>1")
    ap.add_argument("--sp-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo = host-staged exchange, lets ranks share one GPU (tests)")
    ap.add_argument("--sp-stage-depth", type=int, default=2,
                    help="N>1: also time the sharded stage (dispatch, depth blocks, return)")
    ap.add_argument("--token-lpt", action="store_true",
                    help="shard by token counts (reference rule) instead of routed workload")
    ap.add_argument("--sp-train-steps", type=int, default=3,
                    help="N>1: timed SP training steps of one Stage-2 block (0 = skip)")
    ap.add_argument("--no-single-compare", action="store_true",
                    help="N>1: skip timing the same workload on one GPU")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and ws == 0:
        # not under torchrun: launch one rank per GPU ourselves
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
               "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if ws and ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    main()
