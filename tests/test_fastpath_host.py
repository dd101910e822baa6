"""Host logic of the bf16 drop-in (`fastpath.py`), no GPU: precision switch,
supported geometries, the weight fingerprint that invalidates cached engines,
and the same-buffer test that decides whether a self use can run on the
one-stream engine."""

import numpy as np
import pytest

from paper_2604_05182_b200 import fastpath as F
from paper_2604_05182_b200.errors import ConfigurationError
from paper_2604_05182_b200.tensor_core import AttentionParams


def test_precision_switch():
    assert F.precision() == "fp32" and not F.active()
    F.set_precision("bf16")
    assert F.active()
    F.set_precision("fp32")
    assert not F.active()
    with pytest.raises(ConfigurationError):
        F.set_precision("fp8")


def test_supported_geometries():
    assert F.supported(AttentionParams(32, 2, 32))      # paper heads
    assert F.supported(AttentionParams(16, 2, 64))
    assert not F.supported(AttentionParams(8, 1, 8))    # desk heads: fp32 path
    assert not F.supported(AttentionParams(4, 2, 32))   # group 2


def test_fingerprint_tracks_updates():
    from paper_2604_05182_b200.nsa_attention import init_nsa_weights
    w = init_nsa_weights(0, AttentionParams(8, 1, 8), 2, "fp")
    arrays = F._arrays(w, [])
    assert len(arrays) == 14      # w_q w_k w_v w_o gate_w gate_b + 2 ResBlocks x (w1 b1 w2 b2)
    fp = F._fingerprint(arrays)
    assert F._fingerprint(F._arrays(w, [])) == fp
    w.w_o *= 2.0
    assert F._fingerprint(F._arrays(w, [])) != fp
    w.w_o = w.w_o.reshape(-1)[:10].copy()
    assert F._fingerprint(F._arrays(w, [])) != fp


def test_cache_lru_and_identity():
    F.clear_cache()
    built = []

    class Obj:
        pass
    objs = [Obj() for _ in range(F._CACHE_MAX + 2)]
    wts = np.arange(16, dtype=np.float32)
    for i, o in enumerate(objs):
        F._cached(("t", i), (o,), wts, lambda i=i: built.append(i) or i)
    assert len(F._CACHE) == F._CACHE_MAX
    # hit: no rebuild
    assert F._cached(("t", len(objs) - 1), (objs[-1],), wts, lambda: built.append("x")) \
        == len(objs) - 1 and "x" not in built
    # a changed weight value rebuilds
    wts[3] = 7.0
    F._cached(("t", len(objs) - 1), (objs[-1],), wts, lambda: built.append("y") or 0)
    assert built[-1] == "y"
    F.clear_cache()


def test_same_buffer():
    a = np.zeros((4, 3), np.float32)
    assert F._same_buffer(a, a)
    assert F._same_buffer(a, a[:])
    assert not F._same_buffer(a, a.copy())
    assert not F._same_buffer(a, a[:2])
