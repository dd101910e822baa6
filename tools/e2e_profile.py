"""Where the reference-API e2e time goes (C3, one B200): per-phase timings of
the drop-in `nsa_cross_attention` call path (host staging copy, H2D, engine,
D2H) and the raw host/PCIe rates they are bounded by.

    python tools/e2e_profile.py            # prints one JSON object
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))) + "/..")


def wall(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts))


def main():
    import bench
    from paper_2604_05182_b200 import fastpath
    inst_mod = __import__("paper_2604_05182_b200.layer", fromlist=["build_instance"])
    inst = inst_mod.build_instance("c3")
    x = np.ascontiguousarray(inst.x_hat, np.float32)
    out = {"x_mb": x.nbytes / 1e6, "cpu_count": os.cpu_count()}
    dev = torch.device("cuda")
    pin = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
    pin16 = torch.empty(x.shape, dtype=torch.bfloat16, pin_memory=True)
    d = torch.empty(x.shape, dtype=torch.float32, device=dev)
    out["host_copy_threads_ms"] = wall(lambda: fastpath._host_copy(pin.numpy(), x))
    out["host_copy_1t_ms"] = wall(lambda: np.copyto(pin.numpy(), x))
    out["h2d_pinned_ms"] = wall(lambda: d.copy_(pin, non_blocking=True))
    out["h2d_pageable_ms"] = wall(lambda: d.copy_(torch.from_numpy(x), non_blocking=False))
    out["d2h_pinned_ms"] = wall(lambda: pin.copy_(d, non_blocking=True))
    xn = np.empty_like(x)
    out["d2h_pageable_ms"] = wall(lambda: torch.from_numpy(xn).copy_(d))
    out["pinned_alloc_ms"] = wall(lambda: torch.empty(x.shape, dtype=torch.float32,
                                                      pin_memory=True))
    out["np_empty_touch_ms"] = wall(lambda: np.empty_like(x).fill(0))

    def reg():
        cudart = torch.cuda.cudart()
        p = x.__array_interface__["data"][0]
        r = cudart.cudaHostRegister(p, x.nbytes, 0)
        cudart.cudaHostUnregister(p)
        return r
    try:
        out["host_register_unregister_ms"] = wall(reg)
    except Exception as e:   # noqa: BLE001
        out["host_register_unregister_ms"] = repr(e)
    # the whole reference-API layer and its per-use calls
    ms, h2d, d2h = bench.time_reference_api(inst, 5)
    out["api_layer_ms"] = ms
    # phase split of the same calls (after two warm-up layers): the drop-in's
    # helpers wrapped with synchronising wall-clock timers (slower overall)
    from paper_2604_05182_b200 import _dev as D
    from paper_2604_05182_b200 import engine as E
    from paper_2604_05182_b200.nsa_attention import Selection, nsa_cross_attention
    acc = {}

    def timed(name, fn):
        def w(*a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn(*a, **k)
            torch.cuda.synchronize()
            acc[name] = acc.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
            return r
        return w
    for nm in ("_to_block_major", "_to_token_order", "_download", "_cached", "nsa_use"):
        setattr(fastpath, nm, timed(nm, getattr(fastpath, nm)))
    E.SparseLayerEngine.forward = timed("engine_forward", E.SparseLayerEngine.forward)
    parts = {"x": inst.part_vol, "y": inst.part_img}
    feats = {"x": np.ascontiguousarray(inst.x_hat, np.float32),
             "y": np.ascontiguousarray(inst.y_hat, np.float32)}
    geom = {"v2v": ("x", "x"), "v2i": ("x", "y"), "i2i": ("y", "y"), "i2v": ("y", "x")}
    sels = {}
    for use, (qs, ks) in geom.items():
        r, c = (D.host(t) for t in inst.plan_rows[use])
        occ = parts[ks].occupied_ids
        sels[use] = Selection([occ[r[i, :c[i]]] for i in range(r.shape[0])])
    fastpath.set_precision("bf16")

    def layer():
        return {u: nsa_cross_attention(feats[qs], feats[ks], parts[qs], parts[ks], sels[u],
                                       inst.weights[u], inst.params)
                for u, (qs, ks) in geom.items()}
    layer()
    layer()
    acc.clear()
    t0 = time.perf_counter()
    for _ in range(3):
        layer()
    out["api_layer_ms_instrumented"] = (time.perf_counter() - t0) * 1e3 / 3
    out["phases_ms_per_layer"] = {k: v / 3 for k, v in acc.items()}
    out["h2d_bytes"], out["d2h_bytes"] = h2d, d2h
    print(json.dumps(out))


if __name__ == "__main__":
    main()
