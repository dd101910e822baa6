#!/bin/bash
# ncu --set full of the kernels added after the attention profile: the Stage-2
# block's row kernels and the full-block training step (fused tcgen05
# forward, mma.sync dQ / dK,dV, res-block and LayerNorm backward, casts,
# split-K sums, tcgen05 GEMMs).
#   bash tools/profile_extra.sh <tag>              (GPU box; writes gpurun_out/)
#   bash tools/profile_extra.sh <tag> --summarise  (here; writes profiles/<tag>/)
TAG=${1:-r1}
if [ "$2" != "--summarise" ]; then
  mkdir -p gpurun_out
  ncu --set full --import-source on --clock-control none \
      -k "regex:gate_mix_ln_fast|add_ln_fast|bias_act_fast" --launch-count 6 \
      -o gpurun_out/block_full_$TAG -f python tools/block_profile.py > /dev/null 2>&1
  ncu --set full --import-source on --clock-control none \
      -k "regex:nsa_fused|dq_mma|dkdv_mma|res_block_bwd|layer_norm_bwd|cast8|sum_slices|gemm_tc" \
      --launch-skip 400 --launch-count 24 -o gpurun_out/train_full_$TAG -f \
      python tools/train_launches.py > /dev/null 2>&1
  exit 0
fi
mkdir -p profiles/$TAG
for what in block train; do
  ncu -i gpurun_out/${what}_full_$TAG.ncu-rep --page raw --csv > gpurun_out/${what}_full_$TAG.csv
  python - "gpurun_out/${what}_full_$TAG.csv" "profiles/$TAG/${what}_full_summary.csv" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
idx = [h.index(k) for k in keep if k in h]
out = [[h[j] + (f" [{units[j]}]" if units[j] else "") for j in idx]]
out += [[r[j] for j in idx] for r in rows[2:]]
csv.writer(open(sys.argv[2], "w", newline="")).writerows(out)
print(sys.argv[2], len(out) - 1, "kernels")
PY
done
