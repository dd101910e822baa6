"""Oracle numerics: f32 storage, f64 accumulation (TEST INFRASTRUCTURE ONLY).

Restates `lsrm/tensor_core.py` (reference lines cited per function).
"""

import math
from dataclasses import dataclass

import numpy as np
from scipy.special import erf as _erf

DTYPE = np.float32
ACC = np.float64


class OracleError(Exception):
    """Raised where the reference raises one of its LsrmError subclasses.

    ``kind`` names the reference class (`lsrm/errors.py:8-59`)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


@dataclass(frozen=True)
class AttentionParams:
    """GQA head geometry (`lsrm/tensor_core.py:39-71`)."""
    n_q_heads: int
    n_kv_heads: int
    head_dim: int

    @property
    def model_dim(self) -> int:
        return self.n_q_heads * self.head_dim

    @property
    def group_size(self) -> int:
        return self.n_q_heads // self.n_kv_heads


def affine(x, w, b=None):
    """x @ w (+ b), f64 accumulation, f32 result (`tensor_core.py:100-116`).

    einsum keeps the per-row reduction independent of the batch."""
    y = np.einsum("...i,io->...o", np.asarray(x, ACC), np.asarray(w, ACC))
    if b is not None:
        y = y + np.asarray(b, ACC)
    return y.astype(DTYPE)


def gelu(x):
    """Exact-erf GELU in f64 (`tensor_core.py:82-86`)."""
    t = np.asarray(x, ACC)
    return (0.5 * t * (1.0 + _erf(t / math.sqrt(2.0)))).astype(DTYPE)


def sigmoid(x):
    """Branch-stable logistic in f64 (`tensor_core.py:89-94`)."""
    t = np.asarray(x, ACC)
    pos = 1.0 / (1.0 + np.exp(-np.where(t >= 0, t, 0.0)))
    e = np.exp(np.where(t < 0, t, 0.0))
    neg = e / (1.0 + e)
    return np.where(t >= 0, pos, neg).astype(DTYPE)


def layer_norm(x, gamma, beta, eps=1e-5):
    """Biased-variance LayerNorm in f64 (`tensor_core.py:139-146`)."""
    t = np.asarray(x, ACC)
    mu = t.mean(axis=-1, keepdims=True)
    c = t - mu
    var = (c * c).mean(axis=-1, keepdims=True)
    y = c / np.sqrt(var + eps) * np.asarray(gamma, ACC) + np.asarray(beta, ACC)
    return y.astype(DTYPE)


def dense_attention(q, k, v, params: AttentionParams, mask=None):
    """Grouped-query softmax attention, the oracle of every branch
    (`tensor_core.py:164-206`).  q [Nq,hq,dh], k/v [Nk,hkv,dh];
    mask [Nq,Nk] bool (True = attendable)."""
    if k.shape[0] == 0:
        raise OracleError("EmptyContextError", "attention over no keys")
    heads = np.arange(params.n_q_heads) // params.group_size
    q64 = np.asarray(q, ACC)
    k64 = np.asarray(k, ACC)[:, heads, :]
    v64 = np.asarray(v, ACC)[:, heads, :]
    s = np.einsum("qhd,khd->qhk", q64, k64) / math.sqrt(params.head_dim)
    if mask is not None:
        mask = np.asarray(mask, bool)
        if not mask.any(axis=1).all():
            raise OracleError("EmptyAttentionRowError", "row without keys")
        s = np.where(mask[:, None, :], s, -np.inf)
    s = s - s.max(axis=2, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=2, keepdims=True)
    return np.einsum("qhk,khd->qhd", p, v64).astype(DTYPE)
