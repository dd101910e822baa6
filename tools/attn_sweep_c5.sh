for v in "" "-DLSRM_POLY_PER16=2" "-DLSRM_POLY_PER16=4"; do
  LSRM_NVCC_FLAGS="$v" python -m paper_2604_05182_b200.build > /dev/null || { echo "build failed: $v"; continue; }
  echo "== variant: ${v:-default}"
  timeout 300 python tools/attn_trace.py --use v2v --time --workload c5 2>&1 | grep "attention total\|merged"
done
