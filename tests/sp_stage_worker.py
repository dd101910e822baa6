"""torchrun worker for tests/test_seq_parallel.py::test_torchrun_sharded_stage:
W ranks (gloo, host-staged transport; they may share one GPU) run the
block-aware sequence-parallel Stage-2 stage end to end -- dispatch
all_to_all_v from the naive contiguous shards, `depth` sharded blocks with
per-use All-gather-KV, return all_to_all_v -- and rank 0 compares the
reassembled output with the single-GPU `SparseStageEngine`: BIT-EQUAL
(the reference's serial == parallel contract). Exit 0 = match."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_05182_b200 import _dev as D, _ops                        # noqa: E402
from paper_2604_05182_b200 import seq_parallel as S                       # noqa: E402
from paper_2604_05182_b200.layer import build_instance                    # noqa: E402
from paper_2604_05182_b200.recon_pipeline import SparseStageEngine, init_sparse_block  # noqa
from paper_2604_05182_b200.tensor_core import AttentionParams             # noqa: E402


def main():
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    dist.init_process_group("gloo")
    wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
    depth = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    params = AttentionParams(32, 2, 32)
    inst = build_instance(wl, params=params)
    weights = [init_sparse_block(0, params, m) for m in range(depth)]
    pv, pi = inst.part_vol, inst.part_img
    # stage input: the fine tokens' features (x_hat / y_hat stand in for
    # x_up / y_up), token order, concatenated [volume; image]
    feats = np.concatenate([inst.x_hat, inst.y_hat]).astype(np.float32)
    rng = np.random.default_rng(1)
    coords = rng.integers(0, 96, (feats.shape[0], 3)).astype(np.int32)
    st = S.ShardedStage(pv, pi, inst.plan_rows, weights, params, rank, ws,
                        transport=S.HostStagedTransport(rank, ws))
    tk = st.tokens
    lo = int(np.concatenate([[0], np.cumsum([a.size for a in tk.naive])])[rank])
    f_naive = D.dev(feats[lo:lo + tk.n_naive])
    c_naive = D.dev(coords[lo:lo + tk.n_naive])
    out = D.host(st.forward(f_naive, c_naive))
    out2 = D.host(st.forward(f_naive, c_naive))       # rerun: same bytes
    got = [None] * ws if rank == 0 else None
    dist.gather_object((lo, out, out2, st.topology.message_log), got, dst=0)
    status = 0
    if rank == 0:
        ref_eng = SparseStageEngine(pv, pi, inst.plan_rows, weights, params)
        tv, ti = pv.dev("block_token_ids"), pi.dev("block_token_ids")
        xb = _ops.gather_rows(D.dev(inst.x_hat), tv)
        yb = _ops.gather_rows(D.dev(inst.y_hat), ti)
        xs, ys = ref_eng.forward(xb, yb)
        xo, yo = torch.empty_like(xs), torch.empty_like(ys)
        _ops.scatter_rows(xs, tv, xo)
        _ops.scatter_rows(ys, ti, yo)
        ref = np.concatenate([D.host(xo), D.host(yo)])
        full = np.full_like(ref, np.nan)
        full2 = np.full_like(ref, np.nan)
        for lo_r, o, o2, _ in got:
            full[lo_r:lo_r + o.shape[0]] = o
            full2[lo_r:lo_r + o2.shape[0]] = o2
        same = np.array_equal(full, ref)
        rerun = np.array_equal(full2, full)
        diff = float(np.nanmax(np.abs(full - ref)))
        kinds = {}
        for log in (g[3] for g in got):
            for ph, kind, s_, d_, nb in log:
                kinds.setdefault(kind, 0)
                kinds[kind] += nb
        print(f"W={ws} depth={depth}: stage bit-equal {same} (max|diff| {diff:.3e}), "
              f"rerun identical {rerun}; bytes moved {kinds}", flush=True)
        status = 0 if (same and rerun) else 1
    t = torch.tensor([status])
    dist.broadcast(t, 0)
    dist.destroy_process_group()
    sys.exit(int(t.item()))


if __name__ == "__main__":
    main()
