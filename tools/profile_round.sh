#!/bin/bash
# Round profile on one GPU: ncu launch list of a short bench run, `--set full`
# of one layer's K/V-prep launch and its (merged, four-use) attention launch,
# and the attention DRAM traffic per launch that bench.py reports.
#   bash tools/profile_round.sh <tag>      (outputs under gpurun_out/; on the
#   workstation, `bash tools/profile_round.sh <tag> --summarise` turns them into
#   profiles/<tag>/ and profiles/attention_traffic.json)
TAG=${1:-r1}
OUT=profiles/$TAG
mkdir -p gpurun_out
if [ "$2" != "--summarise" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k "regex:nsa_fused|kv_prep" \
    --launch-count 2 -o gpurun_out/layer_full_$TAG -f \
    python tools/attn_trace.py --use v2v > /dev/null 2>&1
exit 0
fi
mkdir -p "$OUT"
cp gpurun_out/launches_$TAG.csv "$OUT/launches_c3_bench.csv"
ncu -i gpurun_out/layer_full_$TAG.ncu-rep --page raw --csv > gpurun_out/layer_full_$TAG.csv
python - "$TAG" <<'PY'
import csv, json, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/layer_full_{tag}.csv")))
h = rows[0]
keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
idx = [h.index(k) for k in keep]
units = rows[1]
out = [[keep[i] + (f" [{units[j]}]" if units[j] else "") for i, j in enumerate(idx)]]
attn = []
for r in rows[2:]:
    out.append([r[j] for j in idx])
    if "nsa_fused" in r[idx[0]]:
        rb = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
        wb = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        ur = units[h.index("dram__bytes_read.sum")]
        uw = units[h.index("dram__bytes_write.sum")]
        attn.append(rb * scale.get(ur, 1.0) + wb * scale.get(uw, 1.0))
with open(f"profiles/{tag}/layer_full_summary.csv", "w", newline="") as fh:
    csv.writer(fh).writerows(out)
if attn:
    json.dump({"bytes_per_launch": sum(attn) / len(attn), "launches": len(attn),
               "source": f"ncu --set full dram__bytes_read.sum + dram__bytes_write.sum, "
                         f"profiles/{tag}/layer_full_summary.csv"},
              open("profiles/attention_traffic.json", "w"), indent=1)
print("\n".join(",".join(r) for r in out))
PY
