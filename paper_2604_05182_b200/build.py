"""Build the in-tree C-ABI library `_lib/liblsrm_b200.so` for sm_100a.

    python -m paper_2604_05182_b200.build        (or __graft_entry__.build())

Each csrc/*.cu is compiled by nvcc for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (ncu source mapping) and linked against the shared CUDA
runtime (so the library shares torch's current-device state) and cuBLAS.
The router / mask / partition translation units are compiled with
--fmad=false on top of their explicit round-to-nearest intrinsics: their
outputs must be bit-exact with the reference's f64 NumPy arithmetic.
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "liblsrm_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "-Xptxas", "-v", "--expt-relaxed-constexpr"]
EXACT_TUS = {"routing.cu", "tokens.cu", "partition.cu", "raymarch.cu", "camera.cu",
             "decode.cu"}
# LSRM_NVCC_FLAGS="-DLSRM_TRACE" builds the per-chunk event trace of the fused
# attention kernel (tools/attn_trace.py); off by default.
EXTRA = os.environ.get("LSRM_NVCC_FLAGS", "").split()


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _compile(src):
    obj = os.path.join(OUT_DIR, src[:-3] + ".o")
    path = os.path.join(CSRC, src)
    deps = [path, os.path.join(CSRC, "common.cuh"),
            os.path.join(HERE, "..", "include", "lsrm_b200.h")]
    deps += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    stamp = obj + ".flags"
    same_flags = os.path.exists(stamp) and open(stamp).read() == " ".join(EXTRA)
    if same_flags and os.path.exists(obj) and \
            os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj, ""
    flags = ARCH + COMMON + EXTRA + (["--fmad=false"] if src in EXACT_TUS else [])
    cmd = [NVCC, *flags, "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    with open(stamp, "w") as fh:
        fh.write(" ".join(EXTRA))
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(f"--- {os.path.basename(o)}\n{log}", file=sys.stderr)
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", LIB, *objs,
               "-lcublas", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
