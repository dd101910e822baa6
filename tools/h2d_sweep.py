"""Time lsrm_h2d_rows on the GPU box per host-thread count (one subprocess
per LSRM_HOST_THREADS setting): ms for one C3-sized upload (16815 x 1024 f32
rows, permuted, to bf16).  The round-2 sweep of staging variants that chose
csrc/hostio.cu's 2 MiB / all-threads-per-chunk design is in DESIGN.md §6.

    python tools/h2d_sweep.py"""
import json
import os
import subprocess
import sys

CHILD = r'''
import time, numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2604_05182_b200._native import call
from paper_2604_05182_b200 import _dev as D
n, d = 16815, 1024
a = np.random.default_rng(0).standard_normal((n, d)).astype(np.float32)
idx = np.random.default_rng(1).permutation(n).astype(np.int64)
out = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
def f():
    call("lsrm_h2d_rows", 1, a.ctypes.data, d, idx.ctypes.data, n, d, out.data_ptr(), d, D.stream())
    torch.cuda.synchronize()
for _ in range(3): f()
ts = []
for _ in range(10):
    t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e3)
print(np.median(ts))
'''

res = []
for th in (1, 4, 8, 16):
    env = dict(os.environ, LSRM_HOST_THREADS=str(th))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    ms = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
    res.append({"threads": th, "ms": ms})
    print(json.dumps(res[-1]), flush=True)
