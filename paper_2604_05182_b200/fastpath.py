"""bf16 tensor-core engines behind the reference API (`dropin.install(lsrm,
precision="bf16")`).

The reference-API functions default to the reference's own float contract
(fp32 CUDA-core kernels, ≤1e-5 of the reference). With precision "bf16",
these reference-API calls run on the bf16 tcgen05 engines that `bench.py`
measures:

  * `nsa_cross_attention` (`lsrm/nsa_attention.py:287-327`) -> a one-use
    `SparseLayerEngine` (fused projection GEMM, K/V prep, fused three-branch
    attention + gated merge, W_o);
  * `sparse_block_forward` (`lsrm/recon_pipeline.py:461-497`) ->
    `SparseBlockEngine`;
  * `sparse_stage_forward` (`lsrm/recon_pipeline.py:500-512`) ->
    `SparseStageEngine`.

The numeric contract is then the bf16 one stated in DESIGN.md §2 (rel-L2 ≤
1e-2 of the reference), not 1e-5. Calls the engines cannot take (score-mode
routing, head geometries outside DESIGN.md §3, a self use whose key stream is
not its query stream) stay on the fp32 GPU path.

Engines hold device copies of the routing and the weights. They are cached
per (partitions, routing, weights) object identity in a small LRU; a hit also
requires every weight array to be alive and unchanged on a strided sample of
its values (`_fingerprint`), so a weight set that is replaced or updated is
re-uploaded. (An in-place update that touches none of the sampled values is
not detected: call `clear_cache()` after such an update.)
"""

import os
import weakref
from collections import OrderedDict
from concurrent.futures import ThreadPoolExecutor
from dataclasses import fields, is_dataclass

import numpy as np
import torch

from . import _dev as D
from . import _ops
from ._native import call
from .errors import require

_STATE = {"precision": "fp32"}
_CACHE = OrderedDict()
_CACHE_MAX = 8
_SAMPLE = 1024     # values per weight array in the fingerprint


def set_precision(precision: str) -> None:
    require(precision in ("fp32", "bf16"), f"precision must be 'fp32' or 'bf16', got {precision!r}")
    _STATE["precision"] = precision
    if precision == "fp32":
        clear_cache()


def precision() -> str:
    return _STATE["precision"]


def active() -> bool:
    return _STATE["precision"] == "bf16"


def clear_cache() -> None:
    _CACHE.clear()


def supported(params) -> bool:
    """Head geometry the bf16 engine takes."""
    g = params.n_q_heads // params.n_kv_heads
    return (params.head_dim in (32, 64) and 4 <= g <= 128 and 128 % g == 0
            and params.n_kv_heads * params.head_dim in (64, 128))


def _arrays(obj, out):
    if isinstance(obj, np.ndarray):
        out.append(obj)
    elif is_dataclass(obj):
        for f in fields(obj):
            _arrays(getattr(obj, f.name), out)
    elif isinstance(obj, (list, tuple)):
        for o in obj:
            _arrays(o, out)
    return out


def _fingerprint(arrays) -> tuple:
    fp = []
    for a in arrays:
        flat = a.reshape(-1)
        step = max(1, flat.size // _SAMPLE)
        fp.append((a.shape, a.dtype.str, flat[::step].tobytes()))
    return tuple(fp)


def _cached(key, objs, weights, build):
    """LRU lookup: an entry is valid while every keyed object is alive and
    the weights' fingerprint is unchanged."""
    arrays = _arrays(weights, [])
    fp = _fingerprint(arrays)
    hit = _CACHE.get(key)
    if hit is not None:
        refs, fp_old, eng = hit
        if all(r() is o for r, o in zip(refs, objs)) and fp_old == fp:
            _CACHE.move_to_end(key)
            return eng
        del _CACHE[key]
    eng = build()
    try:
        refs = [weakref.ref(o) for o in objs]
    except TypeError:
        return eng
    _CACHE[key] = (refs, fp, eng)
    while len(_CACHE) > _CACHE_MAX:
        _CACHE.popitem(last=False)
    return eng


def _rows_of(sel, table, part_kv):
    from .nsa_attention import selection_rows
    if getattr(table, "rows", None) is not None:
        return table.rows, table.count
    return selection_rows(sel, part_kv)


def _same_buffer(a, b) -> bool:
    if a is b:
        return True
    if isinstance(a, np.ndarray) and isinstance(b, np.ndarray):
        return (a.shape == b.shape and a.dtype == b.dtype and a.strides == b.strides
                and a.__array_interface__["data"][0] == b.__array_interface__["data"][0])
    if D.is_device(a) and D.is_device(b):
        return a.shape == b.shape and a.dtype == b.dtype and a.data_ptr() == b.data_ptr()
    return False


_POOL = None


def _host_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[...] = src, row chunks on host threads (NumPy releases the GIL
    for plain copies): pageable <-> pinned staging at memory bandwidth."""
    global _POOL
    n = src.shape[0]
    if src.nbytes < (8 << 20) or n < 64:
        np.copyto(dst, src)
        return
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1)))
    k = _POOL._max_workers
    cuts = np.linspace(0, n, k + 1).astype(np.int64)
    list(_POOL.map(lambda i: np.copyto(dst[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]),
                   range(k)))


def _upload(a) -> torch.Tensor:
    """Host f32 rows -> device, through pinned staging (the caching host
    allocator keeps a staging block until its copy has completed)."""
    if isinstance(a, torch.Tensor) and a.device.type == "cuda":
        return a if a.dtype == torch.float32 else a.float()
    a = np.asarray(a)
    if a.dtype != np.float32 or not a.flags.c_contiguous:
        return D.dev(a, torch.float32)
    pin = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
    _host_copy(pin.numpy(), a)
    return pin.to(D.device(), non_blocking=True)


def _download(t: torch.Tensor) -> np.ndarray:
    """Device f32 -> a fresh NumPy array backed by pinned memory (DMA at
    full PCIe rate; the array owns its buffer)."""
    pin = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    pin.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return pin.numpy()


def _to_block_major(a, part, dtype):
    """token-order rows (host or device, any float) -> block-major device rows.
    Host rows go through `lsrm_h2d_rows`: the row permutation and the bf16
    rounding happen on host threads into pinned staging chunks that are
    copied while the next chunk is converted (csrc/hostio.cu)."""
    if not isinstance(a, torch.Tensor):
        a = np.asarray(a)
        if a.dtype != np.float32 or not a.flags.c_contiguous:
            a = np.ascontiguousarray(a, dtype=np.float32)
        require(a.ndim == 2 and a.shape[0] == part.n_tokens,
                "feature rows do not match the partition")
        idx = part.block_token_ids
        if idx.dtype != np.int64 or not idx.flags.c_contiguous:
            idx = np.ascontiguousarray(idx, dtype=np.int64)
        n, d = a.shape
        out = D.empty((n, d), dtype)
        call("lsrm_h2d_rows", int(dtype == torch.bfloat16), a.ctypes.data, d, idx.ctypes.data,
             n, d, out.data_ptr(), d, D.stream())
        return out
    t = _upload(a)
    g = _ops.gather_rows(t, part.dev("block_token_ids"))
    return g if dtype == torch.float32 else _ops.cast(g, dtype)


def _to_token_order(rows_bm, part, on_dev):
    r = rows_bm if rows_bm.dtype == torch.float32 else _ops.cast(rows_bm, torch.float32)
    out = D.empty(tuple(r.shape), torch.float32)
    _ops.scatter_rows(r, part.dev("block_token_ids"), out)
    return out if on_dev else _download(out)


def nsa_use(x, kv_feats, part_q, part_kv, sel, w, params, table):
    """One gated NSA use on a one-use bf16 engine; None if the engine cannot
    take this call (the caller then runs the fp32 path)."""
    from .engine import SparseLayerEngine
    if not supported(params) or (sel is None and getattr(table, "rows", None) is None):
        return None
    if not hasattr(part_q, "dev") or not hasattr(part_kv, "dev"):
        return None
    self_use = w.n_gates == 3
    if self_use and (part_q is not part_kv or not _same_buffer(x, kv_feats)):
        return None
    name = "v2v" if self_use else "v2i"
    routing = table if getattr(table, "rows", None) is not None else sel
    key = ("use", id(part_q), id(part_kv), id(routing), id(w), params, w.n_gates)

    def build():
        rows = _rows_of(sel, table, part_kv)
        return SparseLayerEngine(part_q, part_q if self_use else part_kv, {name: rows},
                                 {name: w}, params)
    eng = _cached(key, (part_q, part_kv, routing, w), w, build)
    xb = _to_block_major(x, part_q, torch.bfloat16)
    yb = xb if self_use else _to_block_major(kv_feats, part_kv, torch.bfloat16)
    out = eng.forward(xb, yb)[name]
    return _to_token_order(out, part_q, D.is_device(x))


def _ctx_rows(ctx):
    kv = {"v2v": ctx.part_vol, "v2i": ctx.part_img, "i2i": ctx.part_img, "i2v": ctx.part_vol}
    return {u: _rows_of(ctx.selections[u], (ctx.tables or {}).get(u), kv[u]) for u in kv}


def _block_uses(w) -> dict:
    return {"v2v": w.nsa_x_self, "v2i": w.nsa_x_cross, "i2i": w.nsa_y_self,
            "i2v": w.nsa_y_cross}


def _ctx_ok(ctx, params) -> bool:
    return (supported(params) and ctx.selections is not None
            and hasattr(ctx.part_vol, "dev") and hasattr(ctx.part_img, "dev"))


def sparse_block(x, y, x_inj, y_inj, w, ctx, params):
    """One Stage-2 block on `SparseBlockEngine`; None if not applicable."""
    from .recon_pipeline import SparseBlockEngine
    if not _ctx_ok(ctx, params):
        return None
    key = ("block", id(ctx), id(w), params)

    def build():
        return SparseBlockEngine(ctx.part_vol, ctx.part_img, _ctx_rows(ctx), w, params,
                                 uses=_block_uses(w))
    eng = _cached(key, (ctx, w), w, build)
    pv, pi = ctx.part_vol, ctx.part_img
    xs = [_to_block_major(a, pv, torch.float32) for a in (x, x_inj)]
    ys = [_to_block_major(a, pi, torch.float32) for a in (y, y_inj)]
    ox, oy = eng.forward(xs[0], ys[0], xs[1], ys[1])
    on_dev = D.is_device(x)
    return _to_token_order(ox, pv, on_dev), _to_token_order(oy, pi, on_dev)


def sparse_stage(x_up, y_up, weights, ctx, params):
    """The Stage-2 stage on `SparseStageEngine`; None if not applicable."""
    from .recon_pipeline import SparseStageEngine
    if not _ctx_ok(ctx, params) or len(weights) == 0:
        return None
    weights = list(weights)
    key = ("stage", id(ctx), tuple(id(w) for w in weights), params)

    def build():
        return SparseStageEngine(ctx.part_vol, ctx.part_img, _ctx_rows(ctx), weights, params,
                                 uses=[_block_uses(w) for w in weights])
    eng = _cached(key, (ctx, *weights), weights, build)
    xf = _to_block_major(x_up.features, ctx.part_vol, torch.float32)
    yf = _to_block_major(y_up.features, ctx.part_img, torch.float32)
    xs, ys = eng.forward(xf, yf)
    return _to_token_order(xs, ctx.part_vol, False), _to_token_order(ys, ctx.part_img, False)
