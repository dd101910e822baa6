"""One C1 fp32 reference-API layer timing (bench.time_c1_fp32), for ncu launch lists."""
import sys; sys.path.insert(0, ".")
import bench
print(bench.time_c1_fp32(3))
