"""Time the bf16 Stage-2 sparse stage (SparseStageEngine, `depth` blocks over
one routing) on the GPU: build time and forward ms (CUDA events, after
warm-up).

    python tools/stage_time.py [--workload c3] [--depth 24]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--depth", type=int, default=24)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2604_05182_b200 import _dev as D, _ops
    from paper_2604_05182_b200.layer import build_instance
    from paper_2604_05182_b200.recon_pipeline import SparseStageEngine, init_sparse_block
    inst = build_instance(a.workload)
    t0 = time.time()
    ws = [init_sparse_block(0, inst.params, m) for m in range(a.depth)]
    eng = SparseStageEngine(inst.part_vol, inst.part_img, inst.plan_rows, ws, inst.params)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    d = inst.params.model_dim
    g = torch.Generator(device="cuda").manual_seed(0)
    xu = torch.randn((inst.n_vol, d), generator=g, device="cuda")
    yu = torch.randn((inst.n_img, d), generator=g, device="cuda")
    eng.forward(xu, yu)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ms = []
    for _ in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        eng.forward(xu, yu)
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    n = inst.n_vol + inst.n_img
    m = sum(ms) / len(ms)
    print(json.dumps({"workload": a.workload, "depth": a.depth, "n_tokens": n,
                      "build_s": build_s, "forward_ms": m, "ms_per_layer": m / a.depth,
                      "tokens_per_s": n / (m * 1e-3),
                      "mem_gb": torch.cuda.max_memory_allocated() / 1e9}))


if __name__ == "__main__":
    main()
