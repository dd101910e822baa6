"""Device plumbing: torch owns device memory and streams; compute goes through
the C ABI.  No CPU fallback: `require_cuda()` raises without a GPU."""

import numpy as np
import torch

from .errors import LsrmError


def require_cuda():
    if not torch.cuda.is_available():
        raise LsrmError("no CUDA device visible: paper_2604_05182_b200 has no "
                        "CPU fallback (the CPU oracle lives under oracle/, for tests)")


def device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def dev(x, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (optionally cast)."""
    require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        if t.device.type != "cuda":
            t = t.to(device(), non_blocking=False)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x)).to(device())
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def empty(shape, dtype):
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    return torch.zeros(shape, dtype=dtype, device=device())


def ptr(t):
    return None if t is None else t.data_ptr()


def stream():
    return torch.cuda.current_stream().cuda_stream


def host(t):
    return t.detach().cpu().numpy()


def is_device(x):
    return isinstance(x, torch.Tensor) and x.device.type == "cuda"


_WCACHE = {}


def weight(arr, dtype=torch.float32):
    """Device copy of a host weight array, made once per (array, dtype,
    device). Works for any weight container (this package's dataclasses or the
    reference's), which is what the drop-in needs."""
    key = (id(arr), dtype, torch.cuda.current_device())
    hit = _WCACHE.get(key)
    if hit is not None and hit[0] is arr:
        return hit[1]
    t = dev(arr, dtype)
    _WCACHE[key] = (arr, t)
    return t
