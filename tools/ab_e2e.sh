#!/bin/bash
# Same-box A/B of the reference-API e2e (bench.time_reference_api, C3): the
# current tree against scratch/old, alternating, three times each.
for i in 1 2 3; do
  for side in new old; do
    dir=$([ $side = new ] && echo . || echo scratch/old)
    (cd $dir && timeout 600 python -c "
import sys; sys.path.insert(0, '.')
import bench
from paper_2604_05182_b200.layer import build_instance
ms, _, _ = bench.time_reference_api(build_instance('c3'), 10)
print('$side', round(ms, 3))" 2>/dev/null)
  done
done
