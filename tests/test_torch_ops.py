"""torch.library ops (paper_2604_05182_b200.torch_ops): the fp32 branch op
and the differentiable bf16 sparse-attention op against a float64 masked
dense attention (autograd) on the same key sets, for cmp, sel and win."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _instance(seed=0, hq=4, hkv=2, dh=16):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import _dev as D
    from paper_2604_05182_b200.nsa_attention import resolve_rows, selection_rows
    g = np.random.default_rng(seed)
    coords = np.argwhere(g.random((16, 16, 16)) < 0.05)
    toks = L.TokenSet("volume", np.zeros((coords.shape[0], 4), np.float32), coords, (16,) * 3)
    part = L.partition(toks)
    n = toks.count
    lists = [np.sort(g.choice(part.occupied_ids, size=int(g.integers(1, 4)), replace=False))
             for _ in range(n)]
    rows, count = selection_rows(L.Selection(lists), part)
    rows, count, _, _, _ = resolve_rows(rows, count, part, part.block_of_token, True)
    f = lambda *s: torch.tensor(g.standard_normal(s), dtype=torch.float32, device="cuda")  # noqa
    q, k, v = f(n, hq, dh), f(n, hkv, dh), f(n, hkv, dh)      # k / v block-major
    kc, vc = f(part.n_occupied, hkv, dh), f(part.n_occupied, hkv, dh)
    offs = part.dev("block_offsets")
    own = part.dev("row_of_token")
    return dict(q=q, k=k, v=v, kc=kc, vc=vc, offs=offs, rows=rows, count=count, own=own,
                part=part, n=n)


def _mask(inst, mode):
    n, part = inst["n"], inst["part"]
    if mode == 0:
        return None
    offs = inst["offs"].cpu().numpy()
    row_of_key = np.repeat(np.arange(part.n_occupied), np.diff(offs))
    m = np.zeros((n, row_of_key.size), bool)
    if mode == 1:
        r, c = inst["rows"].cpu().numpy(), inst["count"].cpu().numpy()
        for i in range(n):
            m[i] = np.isin(row_of_key, r[i, :c[i]])
    else:
        own = inst["own"].cpu().numpy()
        m = row_of_key[None, :] == own[:, None]
    return torch.from_numpy(m)


def _ref(q, k, v, mask):
    hq, hkv, dh = q.shape[1], k.shape[1], q.shape[2]
    heads = torch.arange(hq) // (hq // hkv)
    s = torch.einsum("nhd,mhd->nhm", q, k[:, heads]) / math.sqrt(dh)
    if mask is not None:
        s = s.masked_fill(~mask[:, None, :], float("-inf"))
    return torch.einsum("nhm,mhd->nhd", torch.softmax(s, 2), v[:, heads])


def _args(inst, mode):
    k, v = (inst["kc"], inst["vc"]) if mode == 0 else (inst["k"], inst["v"])
    return k, v, mode, (None if mode == 0 else inst["offs"]), \
        (inst["rows"] if mode == 1 else None), (inst["count"] if mode == 1 else None), \
        (inst["own"] if mode == 2 else None)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_branch_attention_fp32(cuda, mode):
    import paper_2604_05182_b200.torch_ops  # noqa: F401  (registers the ops)
    inst = _instance(mode)
    k, v, *rest = _args(inst, mode)
    got = torch.ops.lsrm.branch_attention(inst["q"], k, v, *rest)
    want = _ref(inst["q"].double().cpu(), k.double().cpu(), v.double().cpu(), _mask(inst, mode))
    assert float((got.double().cpu() - want).abs().max()) < 1e-5


@pytest.mark.parametrize("heads", [(4, 2, 16), (32, 2, 32), (8, 1, 64)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_sparse_attention_forward_backward(cuda, mode, heads):
    import paper_2604_05182_b200.torch_ops  # noqa: F401
    inst = _instance(10 + mode, *heads)
    k, v, *rest = _args(inst, mode)
    q = inst["q"].clone().requires_grad_(True)
    kk = k.clone().requires_grad_(True)
    vv = v.clone().requires_grad_(True)
    out, lse = torch.ops.lsrm.sparse_attention(q, kk, vv, *rest)
    dout = torch.randn_like(out)
    out.backward(dout)
    q64, k64, v64 = (t.detach().double().cpu().requires_grad_(True) for t in (q, kk, vv))
    want = _ref(q64, k64, v64, _mask(inst, mode))
    want.backward(dout.double().cpu())

    def rel(a, b):
        return float((a.detach().double().cpu() - b).abs().max() / b.abs().max())
    assert rel(out, want.detach()) < 3e-2
    assert rel(q.grad, q64.grad) < 3e-2
    assert rel(kk.grad, k64.grad) < 3e-2
    assert rel(vv.grad, v64.grad) < 3e-2
