"""Time one training step of the four NSA uses of a Stage-2 layer (fp32
forward + backward through training.NsaLayerModule) on the GPU.

    python tools/train_step.py [--workload c3] [--steps 3]

Prints one JSON line: forward / backward ms (CUDA events on the current
stream, after warm-up) and the per-kernel split of one backward."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--fast", action="store_true", help="tensor-core (bf16) attention backward")
    a = ap.parse_args()
    import torch
    from paper_2604_05182_b200.layer import build_instance
    from paper_2604_05182_b200.training import NsaLayerModule, resolve_plan_rows
    inst = build_instance(a.workload)
    res = resolve_plan_rows(inst.plan_rows, inst.part_vol, inst.part_img)
    mod = NsaLayerModule(inst.params, weights=inst.weights, fast_backward=a.fast)
    x = torch.tensor(inst.x_hat, device="cuda", requires_grad=True)
    y = torch.tensor(inst.y_hat, device="cuda", requires_grad=True)

    def step():
        outs = mod(x, y, inst.part_vol, inst.part_img, res)
        loss = sum((o * o).sum() for o in outs.values())
        return loss

    for _ in range(a.warmup):
        step().backward()
    torch.cuda.synchronize()
    fw, bw = [], []
    st = torch.cuda.current_stream()
    for _ in range(a.steps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(st)
        loss = step()
        e[1].record(st)
        loss.backward()
        e[2].record(st)
        torch.cuda.synchronize()
        fw.append(e[0].elapsed_time(e[1]))
        bw.append(e[1].elapsed_time(e[2]))
    n_tok = inst.n_vol + inst.n_img
    ms = sum(fw) / len(fw) + sum(bw) / len(bw)
    print(json.dumps({"workload": a.workload, "n_tokens": n_tok, "dtype": "f32",
                      "backward": "mma.sync bf16" if a.fast else "fp32 CUDA cores",
                      "forward_ms": sum(fw) / len(fw), "backward_ms": sum(bw) / len(bw),
                      "step_ms": ms, "tokens_per_s": n_tok / (ms * 1e-3),
                      "per_step_ms": [round(a + b, 3) for a, b in zip(fw, bw)]}))
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        step().backward()
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))


if __name__ == "__main__":
    main()
