#!/bin/bash
# Build each fused-attention variant (LSRM_NVCC_FLAGS) and time the four C3
# attention launches: bash tools/attn_sweep.sh "flags A" "flags B" ...
for v in "$@"; do
  LSRM_NVCC_FLAGS="$v" python -m paper_2604_05182_b200.build > /dev/null || { echo "build failed: $v"; continue; }
  echo "== variant: ${v:-default}"
  timeout 120 python tools/attn_trace.py --use v2v --time 2>&1 | grep "attention total\|attention v2v\|merged"
done
