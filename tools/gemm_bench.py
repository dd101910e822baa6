"""Time the tcgen05 GEMM (csrc/gemm_tc.cu) against cuBLAS (torch.matmul) on
the layer's C3 shapes: the two per-stream fused projections (one grouped
launch) and the four W_o GEMMs (one grouped launch).

    python tools/gemm_bench.py [--iters 50]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_05182_b200 import _ops  # noqa: E402


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    torch.manual_seed(0)
    dev = "cuda"
    d, ncol = 1024, 7424
    nv, ni = 16815, 10318
    out = {}
    # fused projections: both streams in one launch
    X = {s: torch.randn(n, d, device=dev).to(torch.bfloat16) for s, n in (("x", nv), ("y", ni))}
    W = {s: (torch.randn(d, ncol, device=dev) * 0.02).to(torch.bfloat16) for s in X}
    Wt = {s: W[s].t().contiguous() for s in X}
    bias = {s: torch.zeros(ncol, device=dev, dtype=torch.bfloat16) for s in X}
    Y = {s: torch.empty(X[s].shape[0], ncol, device=dev, dtype=torch.bfloat16) for s in X}
    probs = [_ops.gemm_problem(X[s], Wt[s], Y[s], bias=bias[s]) for s in X]
    flops = sum(2.0 * X[s].shape[0] * d * ncol for s in X)
    t_tc = timeit(lambda: _ops.gemm_tc(probs), args.iters)
    t_cb = timeit(lambda: [torch.matmul(X[s], W[s], out=Y[s]) for s in X], args.iters)
    out["projection"] = {"flops": flops, "tc_ms": t_tc, "cublas_ms": t_cb,
                         "tc_tflops": flops / t_tc / 1e9, "cublas_tflops": flops / t_cb / 1e9}
    # W_o: four uses (v2v, v2i on the volume stream; i2i, i2v on the image stream)
    M = [torch.randn(n, d, device=dev).to(torch.bfloat16) for n in (nv, nv, ni, ni)]
    Wo = [(torch.randn(d, d, device=dev) * 0.02).to(torch.bfloat16) for _ in M]
    Wot = [w.t().contiguous() for w in Wo]
    O = [torch.empty(m.shape[0], d, device=dev, dtype=torch.bfloat16) for m in M]
    probs = [_ops.gemm_problem(m, w, o) for m, w, o in zip(M, Wot, O)]
    flops = sum(2.0 * m.shape[0] * d * d for m in M)
    t_tc = timeit(lambda: _ops.gemm_tc(probs), args.iters)
    t_cb = timeit(lambda: [torch.matmul(m, w, out=o) for m, w, o in zip(M, Wo, O)], args.iters)
    out["w_o"] = {"flops": flops, "tc_ms": t_tc, "cublas_ms": t_cb,
                  "tc_tflops": flops / t_tc / 1e9, "cublas_tflops": flops / t_cb / 1e9}
    # square reference point
    a = torch.randn(8192, 8192, device=dev).to(torch.bfloat16)
    bt = torch.randn(8192, 8192, device=dev).to(torch.bfloat16)
    c = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
    p = [_ops.gemm_problem(a, bt, c)]
    flops = 2.0 * 8192 ** 3
    t_tc = timeit(lambda: _ops.gemm_tc(p), 20)
    t_cb = timeit(lambda: torch.matmul(a, bt.t(), out=c), 20)
    out["square_8192"] = {"tc_ms": t_tc, "cublas_ms": t_cb, "tc_tflops": flops / t_tc / 1e9,
                          "cublas_tflops": flops / t_cb / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
