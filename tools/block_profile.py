"""Per-kernel split of one Stage-2 sparse block on the bf16 engine (C3):
torch.profiler over 3 eager forwards after warm-up.

    python tools/block_profile.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2604_05182_b200.layer import build_instance
    from paper_2604_05182_b200.recon_pipeline import SparseBlockEngine, init_sparse_block
    inst = build_instance("c3")
    w = init_sparse_block(0, inst.params, 0)
    eng = SparseBlockEngine(inst.part_vol, inst.part_img, inst.plan_rows, w, inst.params)
    d = inst.params.model_dim
    ins = [torch.randn((n, d), device="cuda") for n in (inst.n_vol, inst.n_img, inst.n_vol,
                                                         inst.n_img)]
    for _ in range(3):
        eng.forward(*ins)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            eng.forward(*ins)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=90))


if __name__ == "__main__":
    main()
