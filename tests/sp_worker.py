"""torchrun worker for tests/test_seq_parallel.py::test_torchrun_two_ranks_*:
W ranks (gloo, host-staged exchange, may share one GPU) run the sharded
layer with CUDA graphs; rank 0 reassembles token order and compares with the
single-GPU engine.  Exit 0 = match."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_05182_b200 import seq_parallel as S          # noqa: E402
from paper_2604_05182_b200.engine import USES, USE_GEOM       # noqa: E402
from paper_2604_05182_b200.layer import SparseAttentionLayer, build_instance  # noqa: E402


def main():
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    dist.init_process_group("gloo")
    wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
    from paper_2604_05182_b200.tensor_core import AttentionParams
    inst = build_instance(wl, params=AttentionParams(32, 2, 32))   # paper heads
    sl = S.ShardedLayer(inst, rank, ws, transport=S.HostStagedTransport(rank, ws))
    x_loc, y_loc = sl.local_inputs(inst.x_hat, inst.y_hat)
    eager = sl.outputs_token_order(sl.forward(x_loc, y_loc))
    sl.capture(x_loc, y_loc)
    for _ in range(2):
        outs = sl.step()
    torch.cuda.synchronize()
    graphed = sl.outputs_token_order(outs)
    got = [None] * ws if rank == 0 else None
    dist.gather_object((eager, graphed), got, dst=0)
    status = 0
    if rank == 0:
        layer = SparseAttentionLayer(inst)
        ref = layer.forward_host(inst.x_hat, inst.y_hat)
        for use in USES:
            n = ref[use].shape[0]
            for k, tag in ((0, "eager"), (1, "graph")):
                full = np.full_like(ref[use], np.nan)
                for parts in got:
                    ids, val = parts[k][use]
                    full[ids] = val
                diff = float(np.nanmax(np.abs(full - ref[use]))) if n else 0.0
                scale = float(np.abs(ref[use]).max()) if n else 1.0
                ok = not np.isnan(full).any() and diff <= 1e-2 * scale
                print(f"W={ws} {use} {tag}: max|diff| {diff:.3e} scale {scale:.3e} "
                      f"{'ok' if ok else 'MISMATCH'}", flush=True)
                status |= 0 if ok else 1
    t = torch.tensor([status])
    dist.broadcast(t, 0)
    dist.destroy_process_group()
    sys.exit(int(t.item()))


if __name__ == "__main__":
    main()
