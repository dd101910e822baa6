"""Run bench.py's instance-setup kernels once at C3 (voxel mask, foreground
mask, compaction, partition, volume and image routing) and print their
event times; meant to run under ncu (`-k regex:route_image`)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    print(json.dumps(bench.time_setup(sys.argv[1] if len(sys.argv) > 1 else "c3", reps=2)))
