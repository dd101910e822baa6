#!/bin/bash
# Same-box A/B of the full-block training step (bench.time_train_step, C3):
# the current tree against scratch/old, alternating, three times each.
for i in 1 2 3; do
  for side in new old; do
    dir=$([ $side = new ] && echo . || echo scratch/old)
    (cd $dir && timeout 600 python -c "
import sys; sys.path.insert(0, '.')
import bench
from paper_2604_05182_b200.layer import build_instance
r = bench.time_train_step(build_instance('c3'), steps=5)
print('$side', round(r['ms_per_step'], 3), 'fwd', round(r['forward_ms'], 3), 'bwd', round(r['backward_ms'], 3))" 2>/dev/null)
  done
done
