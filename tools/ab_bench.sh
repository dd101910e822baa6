#!/bin/bash
# Same-box A/B of the layer bench: the current tree against an older tree
# exported under scratch/old (git archive <rev> ... | tar -x -C scratch/old,
# built there).  Alternates the two, twice each.
#   bash tools/ab_bench.sh
for i in 1 2 3; do
  for side in new old; do
    dir=$([ $side = new ] && echo . || echo scratch/old)
    (cd $dir && timeout 600 python bench.py --steps 20 --no-cpu-baseline 2>/dev/null) | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
b = d['breakdown_ms']
print('$side', round(d['ms_per_step'], 4), 'attn', round(b['attention_ms'], 4), 'proj',
      round(b['project_gemm_ms'], 4), 'wo', round(b['wo_gemm_ms'], 4))"
  done
done
