"""One full Stage-2 block training step (bench.time_train_step) at C3, for an
ncu launch list:  ncu --metrics gpu__time_duration.sum --clock-control none
--csv --log-file X python tools/train_launches.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import bench
    from paper_2604_05182_b200.layer import build_instance
    print(bench.time_train_step(build_instance(sys.argv[1] if len(sys.argv) > 1 else "c3"),
                                steps=1))
