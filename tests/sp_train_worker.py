"""torchrun worker for tests/test_seq_parallel.py::test_torchrun_sharded_training:
W ranks (gloo, host-staged exchanges; they may share one GPU) run one
training step of the Stage-2 block (training.SparseBlockModule) under
block-aware sequence parallelism -- each rank its own query blocks, K/V
all-gathered per use, partial dK / dV summed at their owners, parameter
gradients summed over ranks -- and rank 0 compares outputs, input gradients
and every parameter gradient with the single-GPU step.  Exit 0 = match.

    torchrun --nproc-per-node W tests/sp_train_worker.py [fp32|fast]"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_05182_b200 import _dev as D                                # noqa: E402
from paper_2604_05182_b200 import seq_parallel as S                        # noqa: E402
from paper_2604_05182_b200.layer import build_instance                     # noqa: E402
from paper_2604_05182_b200.recon_pipeline import init_sparse_block         # noqa: E402
from paper_2604_05182_b200.tensor_core import AttentionParams              # noqa: E402
from paper_2604_05182_b200.training import SparseBlockModule, resolve_plan_rows  # noqa: E402

# vs the one-GPU step: fp32 kernels differ by summation order only; the fast
# path's bf16 operands turn those 1e-7 differences into bf16 rounding flips
# (the tolerance of the fast path against the f64 oracle, test_training.py)
TOL = {"fp32": 1e-4, "fast": 3e-2}


def step(mod, x, y, xi, yi, inst, res, shard=None):
    x = x.clone().requires_grad_(True)
    y = y.clone().requires_grad_(True)
    x2, y2 = mod(x, y, xi, yi, inst.part_vol, inst.part_img, res, shard=shard)
    loss = (x2 * x2).sum() + (y2 * y2).sum()
    loss.backward()
    return x2.detach(), y2.detach(), x.grad, y.grad


def main():
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    dist.init_process_group("gloo")
    mode = sys.argv[1] if len(sys.argv) > 1 else "fp32"
    params = AttentionParams(32, 2, 32)
    inst = build_instance("c1", params=params)
    res = resolve_plan_rows(inst.plan_rows, inst.part_vol, inst.part_img)
    topo = S.sharding_for(inst, ws)
    shard = S.training_shard(inst.part_vol, inst.part_img, topo, rank,
                             S.HostStagedTransport(rank, ws))
    weights = init_sparse_block(0, params, 0, scale=0.05)
    x_full = D.dev(inst.x_hat)
    y_full = D.dev(inst.y_hat)
    lx = torch.as_tensor(shard["x"].queries.loc_tok, device="cuda")
    ly = torch.as_tensor(shard["y"].queries.loc_tok, device="cuda")
    mod = SparseBlockModule(params, weights=weights, fast_backward=mode == "fast")
    outs = step(mod, x_full[lx], y_full[ly], 0.1 * x_full[lx], 0.1 * y_full[ly], inst, res, shard)
    S.allreduce_grads(list(mod.parameters()), host_staged=True)
    mine = {"lx": D.host(lx), "ly": D.host(ly), "out": [D.host(t) for t in outs],
            "grads": {n: D.host(p.grad) for n, p in mod.named_parameters()},
            "bytes": shard["x"].exchange.bytes_moved + shard["y"].exchange.bytes_moved}
    got = [None] * ws if rank == 0 else None
    dist.gather_object(mine, got, dst=0)
    status = 0
    if rank == 0:
        ref_mod = SparseBlockModule(params, weights=weights, fast_backward=mode == "fast")
        ref = [D.host(t) for t in step(ref_mod, x_full, y_full, 0.1 * x_full, 0.1 * y_full,
                                       inst, res)]
        asm = [np.full_like(r, np.nan) for r in ref]
        for g in got:
            for i, (idx, o) in enumerate(zip((g["lx"], g["ly"], g["lx"], g["ly"]), g["out"])):
                asm[i][idx] = o

        ref_g = {n: D.host(p.grad) for n, p in ref_mod.named_parameters()}
        # floor: 1% of the largest gradient, for gradients that vanish exactly
        # (the K compression's b2 shifts every compressed key of a head
        # equally: the cmp softmax is invariant to it, fp32 leaves noise)
        floor = 1e-2 * max(float(np.abs(g).max()) for g in ref_g.values())

        def rel(a, b, fl=1e-30):
            return float(np.abs(a - b).max() / max(np.abs(b).max(), fl))
        errs = {nm: rel(a, b) for nm, a, b in zip(("x2", "y2", "dx", "dy"), asm, ref)}
        for n, g in ref_g.items():
            errs[n] = rel(got[0]["grads"][n], g, floor)
        worst = max(errs, key=errs.get)
        ok = all(np.isfinite(a).all() for a in asm) and errs[worst] <= TOL[mode]
        print(f"W={ws} {mode}: worst rel err {errs[worst]:.2e} ({worst}); outputs "
              f"{max(errs[k] for k in ('x2', 'y2')):.2e}; exchanged "
              f"{sum(g['bytes'] for g in got) / 1e6:.1f} MB", flush=True)
        status = 0 if ok else 1
    t = torch.tensor([status])
    dist.broadcast(t, 0)
    dist.destroy_process_group()
    sys.exit(int(t.item()))


if __name__ == "__main__":
    main()
