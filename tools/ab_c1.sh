#!/bin/bash
# Same-box A/B of the C1 fp32 reference-API layer (bench.time_c1_fp32): the
# current tree against scratch/old, alternating, three times each.
for i in 1 2 3; do
  for side in new old; do
    dir=$([ $side = new ] && echo . || echo scratch/old)
    (cd $dir && timeout 600 python -c "
import sys; sys.path.insert(0, '.')
import bench
r = bench.time_c1_fp32(10)
print('$side', round(r['ms_per_layer'], 4))" 2>/dev/null)
  done
done
