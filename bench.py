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


def cpu_oracle_sample(wl_name="c3", frac=1.0 / 32, seed=0):
    """Time the oracle's four NSA uses on a bounded query sample of the
    workload: the first query blocks holding ~frac of each use's queries,
    against the FULL key/value side.  Returns (tokens_done, seconds, desc)."""
    import oracle as O
    from paper_2604_05182_b200.workloads import coarse_inputs, load_workload
    wl = load_workload(wl_name)
    params = O.AttentionParams(32, 2, 32)
    d = params.model_dim
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, d)
    x_up, y_up = O.upsample_select_tokens(x_d, y_d, wl.vol_mask, wl.img_mask, pe_v.tables,
                                          pe_i.tables, wl.factor_vol, wl.factor_img)
    pv = O.partition_tokens("volume", x_up.coords, x_up.grid_res)
    pi = O.partition_tokens("image", y_up.coords, y_up.grid_res)
    vpts = (x_up.coords.astype(np.float64) + 0.5) / wl.s_vol
    plan = O.build_routing_plan(vpts, wl.img_points, pv, pi, wl.cameras,
                                dict(b_i=16, b_v2v=8, b_v2i=8, b_i2v=8, b_i2i=8))
    blk = O.init_sparse_block(seed, params, 0)
    ones, zeros = np.ones(d, np.float32), np.zeros(d, np.float32)
    xh = O.layer_norm(x_up.features, ones, zeros)
    yh = O.layer_norm(y_up.features, ones, zeros)
    uses = {"v2v": (xh, xh, pv, pv), "v2i": (xh, yh, pv, pi), "i2i": (yh, yh, pi, pi),
            "i2v": (yh, xh, pi, pv)}
    done, t_total = 0, 0.0
    for name, (xq, xkv, pq, pk) in uses.items():
        n_take = max(1, int(pq.n_tokens * frac))
        r = int(np.searchsorted(pq.block_offsets, n_take))
        qids = pq.block_token_ids[:pq.block_offsets[min(r, pq.n_occupied)]]
        lists = [plan.tables[name][i] for i in qids]
        own = pk.block_of_token[qids] if name in ("v2v", "i2i") else None
        w = blk.nsa[name]
        t0 = time.perf_counter()
        # the oracle's nsa_use with the query side restricted to the sample
        n = qids.size
        q = O.affine(xq[qids], w.w_q).reshape(n, params.n_q_heads, params.head_dim)
        k = O.affine(xkv, w.w_k).reshape(-1, params.n_kv_heads, params.head_dim)
        v = O.affine(xkv, w.w_v).reshape(-1, params.n_kv_heads, params.head_dim)
        kc, vc = O.compress_block_kv(k, v, pk, w.compress)
        outs = [O.cmp_attention(q, kc, vc, params).reshape(n, d),
                O.sel_attention(q, k, v, pk, lists, params, own).reshape(n, d)]
        if name in ("v2v", "i2i"):
            outs.append(_win_sample(O, q, qids, k, v, pk, params).reshape(n, d))
        O.combine_branches(xq[qids], outs, w)
        t_total += time.perf_counter() - t0
        done += n
    desc = (f"oracle 4 NSA uses, C3 paper heads 32/2/32 d=1024, first query blocks holding "
            f"~{frac:.4f} of each use's queries ({done} queries) against the full KV side")
    return done, t_total, desc


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
    rank, _, ws = dist_env()
    if rank != 0:
        return
    for _ in range(args.warmup_ref):
        pass
    times, tokens, desc = [], 0, ""
    for _ in range(args.steps):
        tokens, secs, desc = cpu_oracle_sample(frac=args.ref_frac)
        times.append(secs)
    v = tokens / float(np.mean(times))
    hi = host_info()
    line = {"impl": "reference", "metric": "LSRM sparse-attn layer tokens/s",
            "value": v, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference fixture geometry, tagged Philox features/weights)",
            "config": {"workload": "C3 fine stage (16 views, S_vol=S_img=96, heads 32/2/32, "
                                   "d=1024), bounded query sample", "parallelism": "cpu"},
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
    torch.cuda.set_device(local_rank)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        from paper_2604_05182_b200.seq_parallel import run_sp_bench
        return run_sp_bench(args)
    wl_name = "c3"
    inst = build_instance(wl_name)
    layer = SparseAttentionLayer(inst)
    x_bm, y_bm = layer.device_inputs(inst.x_hat, inst.y_hat)
    n_tok = inst.n_vol + inst.n_img
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        layer.engine.forward(x_bm, y_bm)
    torch.cuda.synchronize()
    # -- timed region: K steps, device events per step, L2 flushed in between
    sampler = ClockSampler(local_rank)
    sampler.start()
    reset_launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(st)
        layer.engine.forward(x_bm, y_bm)
        evs[i][1].record(st)
    torch.cuda.synchronize()
    launches = launch_count()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(step_ms))
    # -- per-kernel breakdown (separate pass, events on the launching stream)
    brk = layer.profile_breakdown(x_bm, y_bm, reps=max(3, args.steps))
    clocks = sampler.stop()
    # -- end to end through the public host API (pinned host buffers)
    e2e_ms, h2d, d2h = layer.time_host_path(inst.x_hat, inst.y_hat, steps=args.steps)
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
               "kind": "port", "sample": desc}
    proj_flops = layer.engine.projection_flops()
    line = {
        "metric": "LSRM sparse-attn layer tokens/s", "value": n_tok / (ms * 1e-3),
        "unit": "tokens/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (reference fixture geometry, tagged Philox features/weights)",
        "config": {"workload": "C3 fine stage: 16 views, S_vol=S_img=96, heads 32/2/32, d=1024, "
                               "3D routing b_i=16 budgets 8, one layer = 4 gated NSA uses",
                   "n_vol": inst.n_vol, "n_img": inst.n_img, "global_batch": n_tok,
                   "parallelism": "single GPU", "l2": "flushed (256 MiB write) between steps"},
        "roofline": {"bound": "tensor", "kernel": "nsa_fused_kernel (4 launches/step)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"{src} bf16_tflops (burst)",
                     "algorithmic_flops_per_step": attn_flops},
        "breakdown_ms": brk,
        "layer_tflops": (attn_flops + proj_flops) / (ms * 1e-3) / 1e12,
        "cpu_baseline": cpu,
        "e2e": {"value": n_tok / (e2e_ms * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-frac", type=float, default=1.0 / 32)
    ap.add_argument("--warmup-ref", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        args.steps = min(args.steps, 3)
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    main()
