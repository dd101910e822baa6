"""Device plumbing: torch owns device memory and streams; compute goes through
the C ABI.  No CPU fallback: `require_cuda()` raises without a GPU."""

import weakref
from collections import OrderedDict

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


_WCACHE = OrderedDict()   # (id, dtype, device) -> (weakref to the array, snapshot, tensor)
_WCACHE_MAX = 256


def weight(arr, dtype=torch.float32):
    """Device copy of a host weight array.

    The reference functions are pure functions of their arguments, so a
    cached copy is only reused while the caller's array is alive AND still
    holds the same values (compared against a host snapshot: a weight updated
    in place is re-uploaded).  The cache is a bounded LRU, and it keeps the
    device copy alive past the launch that reads it.  Works for any weight
    container (this package's dataclasses or the reference's), which is what
    the drop-in needs."""
    if is_device(arr):
        return arr if arr.dtype == dtype else arr.to(dtype)
    a = np.asarray(arr)
    key = (id(arr), dtype, torch.cuda.current_device())
    hit = _WCACHE.get(key)
    if hit is not None:
        ref, snap, t = hit
        if ref() is arr and snap.shape == a.shape and snap.dtype == a.dtype and \
                np.array_equal(snap, a, equal_nan=snap.dtype.kind == "f"):
            _WCACHE.move_to_end(key)
            return t
        del _WCACHE[key]
    t = dev(a, dtype)
    try:
        ref = weakref.ref(arr)
    except TypeError:      # not weak-referenceable: no caching
        return t
    _WCACHE[key] = (ref, a.copy(), t)
    while len(_WCACHE) > _WCACHE_MAX:
        _WCACHE.popitem(last=False)
    return t
