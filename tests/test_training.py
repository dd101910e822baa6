"""Backward of one gated NSA use (the reference has no
backward).  The oracle is `oracle/torch_nsa.py` (float64 torch autograd):

  * CPU: its forward is pinned to the NumPy oracle's `nsa_use` (which follows
    `nsa_attention.py:287-327`) and its gradients to finite differences
    (`torch.autograd.gradcheck`);
  * GPU: `training.NsaUseModule` (fp32 kernels) matches its forward and every
    gradient (inputs, projections, gate, compression ResBlocks) within
    GRAD_RTOL of the largest entry, for self (3 gates) and cross (2 gates) uses.
"""

import numpy as np
import pytest
import torch

import oracle as O
from oracle import torch_nsa as TN

GRAD_RTOL = 2e-4      # fp32 kernels vs f64 autograd, relative to max |grad|
FWD_ATOL = 2e-5       # NumPy oracle stores f32 between steps
FAST_RTOL = 3e-2      # tensor-core backward: bf16 q/k/v/dO/P/dS operands


def _coords(seed, side, keep):
    g = np.random.default_rng(seed)
    return np.argwhere(g.random((side, side, side)) < keep)


def _weights(seed, hq, hkv, dh, n_gates, scale=0.3):
    g = np.random.default_rng(seed)
    d, w = hq * dh, hkv * dh
    f = lambda *s: (g.standard_normal(s) * scale).astype(np.float32)   # noqa: E731
    rb = lambda: (f(w, w), f(w), f(w, w), f(w))                        # noqa: E731
    return dict(w_q=f(d, d), w_k=f(d, w), w_v=f(d, w), w_o=f(d, d), gate_w=f(d, n_gates * d),
                gate_b=f(n_gates * d), ck=rb(), cv=rb())


def _oracle_weights(w, n_gates):
    return O.NsaWeights(w["w_q"], w["w_k"], w["w_v"], w["w_o"], w["gate_w"], w["gate_b"],
                        (w["ck"], w["cv"]), n_gates)


def _t64(w, requires_grad=False):
    out = {}
    for k, v in w.items():
        if isinstance(v, tuple):
            out[k] = tuple(torch.tensor(a, dtype=torch.float64, requires_grad=requires_grad)
                           for a in v)
        else:
            out[k] = torch.tensor(v, dtype=torch.float64, requires_grad=requires_grad)
    return out


def _lists(seed, n, occupied, kmax=3):
    g = np.random.default_rng(seed)
    return [np.sort(g.choice(occupied, size=int(g.integers(1, min(kmax, occupied.size) + 1)),
                             replace=False)) for _ in range(n)]


def _instance(seed, self_use, side=16, keep=0.03, heads=(4, 2, 8), wscale=0.3):
    hq, hkv, dh = heads
    params = O.AttentionParams(hq, hkv, dh)
    cq = _coords(seed, side, keep)
    ckv = cq if self_use else _coords(seed + 100, side, keep)
    pq = O.partition_tokens("volume", cq, (side,) * 3)
    pkv = pq if self_use else O.partition_tokens("volume", ckv, (side,) * 3)
    g = np.random.default_rng(seed + 7)
    d = params.model_dim
    x = g.standard_normal((cq.shape[0], d)).astype(np.float32)
    kv = x if self_use else g.standard_normal((ckv.shape[0], d)).astype(np.float32)
    n_gates = 3 if self_use else 2
    w = _weights(seed + 3, hq, hkv, dh, n_gates, scale=wscale)
    lists = _lists(seed + 5, cq.shape[0], pkv.occupied_ids)
    return params, cq, ckv, pq, pkv, x, kv, w, lists, n_gates


@pytest.mark.parametrize("self_use", [True, False])
def test_torch_oracle_forward_matches_numpy_oracle(self_use):
    params, _, _, pq, pkv, x, kv, w, lists, ng = _instance(11, self_use)
    want = O.nsa_use(x, kv, pq, pkv, lists, _oracle_weights(w, ng), params)
    sel, win = TN.key_masks(pq, pkv, lists, self_use)
    got = TN.nsa_use(torch.tensor(x, dtype=torch.float64), torch.tensor(kv, dtype=torch.float64),
                     _t64(w), params, pkv, sel, win)
    err = np.max(np.abs(got.numpy() - want))
    assert err < FWD_ATOL * max(1.0, np.max(np.abs(want))), err


@pytest.mark.parametrize("self_use", [True, False])
def test_torch_oracle_gradcheck(self_use):
    """Finite differences on a tiny instance (2 q-heads, 1 kv-head, dh 2)."""
    params, _, _, pq, pkv, x, kv, w, lists, _ = _instance(12, self_use, side=8, keep=0.025,
                                                          heads=(2, 1, 2))
    sel, win = TN.key_masks(pq, pkv, lists, self_use)
    tw = _t64(w)
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    kvt = xt if self_use else torch.tensor(kv, dtype=torch.float64, requires_grad=True)
    flat = [tw["w_q"], tw["w_k"], tw["gate_b"], *tw["ck"], tw["cv"][2]]
    for t in flat:
        t.requires_grad_(True)

    def f(xx, kk, *ws):
        ww = dict(tw)
        ww["w_q"], ww["w_k"], ww["gate_b"] = ws[0], ws[1], ws[2]
        ww["ck"] = tuple(ws[3:7])
        ww["cv"] = (tw["cv"][0], tw["cv"][1], ws[7], tw["cv"][3])
        return TN.nsa_use(xx, xx if self_use else kk, ww, params, pkv, sel, win)
    assert torch.autograd.gradcheck(f, (xt, kvt, *flat), eps=1e-6, atol=1e-6, rtol=1e-4)


# ---------------------------------------------------------------------------
# GPU


def _our_weights(w, n_gates):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.block_partition import CompressWeights, ResBlockParams
    return L.NsaWeights(w["w_q"], w["w_k"], w["w_v"], w["w_o"], w["gate_w"], w["gate_b"],
                        CompressWeights(ResBlockParams(*w["ck"]), ResBlockParams(*w["cv"])),
                        n_gates)


def _rel(a, b, floor=1e-30):
    """max |a - b| / max(max |b|, floor)."""
    a = a.detach().double().cpu()
    b = b.detach().double().cpu()
    return float((a - b).abs().max() / max(float(b.abs().max()), floor))


def _gpu_vs_oracle(self_use, heads, wscale, fast):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.training import NsaUseModule
    params, cq, ckv, pq, pkv, x, kv, w, lists, ng = _instance(21, self_use, keep=0.05,
                                                              heads=heads, wscale=wscale)
    p = L.AttentionParams(*(params.n_q_heads, params.n_kv_heads, params.head_dim))
    side = 16
    tq = L.TokenSet("volume", x, cq, (side,) * 3)
    part_q = L.partition(tq)
    part_kv = part_q if self_use else L.partition(L.TokenSet("volume", kv, ckv, (side,) * 3))
    mod = NsaUseModule(p, ng, weights=_our_weights(w, ng), fast_backward=fast)
    xg = torch.tensor(x, device="cuda", requires_grad=True)
    kvg = xg if self_use else torch.tensor(kv, device="cuda", requires_grad=True)
    out = mod(xg, kvg, part_q, part_kv, sel=L.Selection(lists))
    g = np.random.default_rng(5)
    dout = g.standard_normal(out.shape).astype(np.float32)
    out.backward(torch.tensor(dout, device="cuda"))

    sel, win = TN.key_masks(pq, pkv, lists, self_use)
    tw = _t64(w, requires_grad=True)
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    kvt = xt if self_use else torch.tensor(kv, dtype=torch.float64, requires_grad=True)
    want = TN.nsa_use(xt, kvt, tw, params, pkv, sel, win)
    want.backward(torch.tensor(dout, dtype=torch.float64))
    assert _rel(out, want) < (FAST_RTOL if fast else 1e-5)
    pairs = [("x", xg.grad, xt.grad)]
    if not self_use:
        pairs.append(("kv", kvg.grad, kvt.grad))
    for name in ("w_q", "w_k", "w_v", "w_o", "gate_w", "gate_b"):
        pairs.append((name, getattr(mod, name).grad, tw[name].grad))
    for tag in ("ck", "cv"):
        for i, s in enumerate(("w1", "b1", "w2", "b2")):
            pairs.append((f"{tag}_{s}", getattr(mod, f"{tag}_{s}").grad, tw[tag][i].grad))
    # floor: 1% of the largest gradient, for gradients that vanish exactly
    # (the K compression's b2 shifts every compressed key of a head equally, so
    # the cmp softmax is invariant to it; fp32 leaves cancellation noise)
    floor = 1e-2 * max(float(b.abs().max()) for _, _, b in pairs)
    return {n: _rel(a, b, floor) for n, a, b in pairs}


@pytest.mark.gpu
@pytest.mark.parametrize("self_use", [True, False])
def test_gpu_backward_matches_f64_autograd(cuda, self_use):
    errs = _gpu_vs_oracle(self_use, (4, 2, 8), 0.3, False)
    bad = {n: e for n, e in errs.items() if e > GRAD_RTOL}
    assert not bad, bad


@pytest.mark.gpu
@pytest.mark.parametrize("self_use", [True, False])
@pytest.mark.parametrize("fast", [False, True])
def test_gpu_backward_paper_heads(cuda, self_use, fast):
    """Paper heads (32/2/32, group 16): the fp32 path within GRAD_RTOL, the
    fast path (mma.sync bf16 branch forward/backward, TF32 GEMMs) within
    FAST_RTOL."""
    errs = _gpu_vs_oracle(self_use, (32, 2, 32), 0.03, fast)
    tol = FAST_RTOL if fast else GRAD_RTOL
    bad = {n: e for n, e in errs.items() if e > tol}
    assert not bad, (bad, errs)


@pytest.mark.gpu
def test_gpu_training_steps_reduce_loss(cuda):
    """A few Adam steps on a fixed regression target lower the loss."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.training import NsaUseModule
    params, cq, _, _, _, x, _, w, lists, ng = _instance(31, True, keep=0.05)
    p = L.AttentionParams(params.n_q_heads, params.n_kv_heads, params.head_dim)
    part = L.partition(L.TokenSet("volume", x, cq, (16,) * 3))
    mod = NsaUseModule(p, ng, weights=_our_weights(w, ng))
    xg = torch.tensor(x, device="cuda")
    target = torch.tensor(np.random.default_rng(2).standard_normal(x.shape).astype(np.float32),
                          device="cuda")
    opt = torch.optim.Adam(mod.parameters(), lr=1e-2)
    sel = L.Selection(lists)
    losses = []
    for _ in range(20):
        opt.zero_grad()
        loss = ((mod(xg, xg, part, part, sel=sel) - target) ** 2).mean()
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    assert losses[-1] < 0.9 * losses[0], losses


@pytest.mark.gpu
def test_trained_weights_round_trip_to_reference_api(cuda):
    """module_weights() exports the module's parameters as NsaWeights; the
    reference-API forward with them equals the module's forward."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.training import NsaUseModule, module_weights
    params, cq, _, _, _, x, _, w, lists, ng = _instance(41, True, keep=0.05)
    p = L.AttentionParams(params.n_q_heads, params.n_kv_heads, params.head_dim)
    part = L.partition(L.TokenSet("volume", x, cq, (16,) * 3))
    mod = NsaUseModule(p, ng, weights=_our_weights(w, ng))
    with torch.no_grad():
        mod.w_o.mul_(1.5)                      # "trained": differs from the initial weights
    xg = torch.tensor(x, device="cuda")
    got = mod(xg, xg, part, part, sel=L.Selection(lists)).detach().cpu().numpy()
    ref = L.nsa_cross_attention(x, x, part, part, L.Selection(lists), module_weights(mod), p)
    assert np.max(np.abs(got - ref)) < 1e-5


# ---------------------------------------------------------------------------
# the full Stage-2 block (recon_pipeline.py:461-497)


def _block_instance(seed, heads, wscale, side=16, keep=0.03):
    hq, hkv, dh = heads
    params = O.AttentionParams(hq, hkv, dh)
    d = params.model_dim
    cx, cy = _coords(seed, side, keep), _coords(seed + 50, side, keep)
    px = O.partition_tokens("volume", cx, (side,) * 3)
    py = O.partition_tokens("volume", cy, (side,) * 3)
    g = np.random.default_rng(seed + 1)
    f = lambda *s, sc=wscale: (g.standard_normal(s) * sc).astype(np.float32)   # noqa: E731
    arrays = dict(x=f(cx.shape[0], d, sc=1.0), y=f(cy.shape[0], d, sc=1.0),
                  xi=f(cx.shape[0], d, sc=0.5), yi=f(cy.shape[0], d, sc=0.5))
    blk = {}
    for s_ in ("x", "y"):
        blk[f"ln_a{s_}"] = (1.0 + f(d, sc=0.2), f(d, sc=0.2))
        blk[f"ln_f{s_}"] = (1.0 + f(d, sc=0.2), f(d, sc=0.2))
        blk[f"gate_{s_}"] = (f(d, 2 * d), f(2 * d))
        blk[f"ffn_{s_}"] = (f(d, 4 * d), f(4 * d), f(4 * d, d), f(d))
    uses = {u: _weights(seed + 10 + i, hq, hkv, dh, 3 if u in ("v2v", "i2i") else 2, scale=wscale)
            for i, u in enumerate(("v2v", "v2i", "i2i", "i2v"))}
    kvp = {"v2v": px, "v2i": py, "i2i": py, "i2v": px}
    qn = {"v2v": cx.shape[0], "v2i": cx.shape[0], "i2i": cy.shape[0], "i2v": cy.shape[0]}
    lists = {u: _lists(seed + 20 + i, qn[u], kvp[u].occupied_ids)
             for i, u in enumerate(("v2v", "v2i", "i2i", "i2v"))}
    return params, cx, cy, px, py, arrays, blk, uses, lists


def _block_vs_oracle(heads, wscale, fast):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200 import recon_pipeline as R
    from paper_2604_05182_b200.nsa_attention import selection_rows
    from paper_2604_05182_b200.training import (BLOCK_PARAM_NAMES, SparseBlockModule,
                                                resolve_plan_rows)
    params, cx, cy, px, py, a, blk, uses, lists = _block_instance(41, heads, wscale)
    p = L.AttentionParams(params.n_q_heads, params.n_kv_heads, params.head_dim)
    part_x = L.partition(L.TokenSet("volume", a["x"], cx, (16,) * 3))
    part_y = L.partition(L.TokenSet("volume", a["y"], cy, (16,) * 3))
    kvp = {"v2v": part_x, "v2i": part_y, "i2i": part_y, "i2v": part_x}
    plan_rows = {u: selection_rows(L.Selection(lists[u]), kvp[u]) for u in lists}
    resolved = resolve_plan_rows(plan_rows, part_x, part_y)
    w = R.SparseBlockWeights(
        _our_weights(uses["v2v"], 3), _our_weights(uses["v2i"], 2), _our_weights(uses["i2i"], 3),
        _our_weights(uses["i2v"], 2), None, None, blk["gate_x"][0], blk["gate_x"][1],
        blk["gate_y"][0], blk["gate_y"][1], R.NormParams(*blk["ln_ax"]),
        R.NormParams(*blk["ln_ay"]), R.NormParams(*blk["ln_fx"]), R.NormParams(*blk["ln_fy"]),
        R.FfnWeights(*blk["ffn_x"]), R.FfnWeights(*blk["ffn_y"]))
    mod = SparseBlockModule(p, weights=w, fast_backward=fast)
    ins = {k: torch.tensor(v, device="cuda", requires_grad=True) for k, v in a.items()}
    x2, y2 = mod(ins["x"], ins["y"], ins["xi"], ins["yi"], part_x, part_y, resolved)
    g = np.random.default_rng(9)
    dx2 = g.standard_normal(x2.shape).astype(np.float32)
    dy2 = g.standard_normal(y2.shape).astype(np.float32)
    torch.autograd.backward([x2, y2], [torch.tensor(dx2, device="cuda"),
                                       torch.tensor(dy2, device="cuda")])
    # f64 oracle
    t = lambda v: torch.tensor(v, dtype=torch.float64, requires_grad=True)   # noqa: E731
    tw = {"uses": {u: _t64(uses[u], requires_grad=True) for u in uses}}
    for k, v in blk.items():
        tw[k] = tuple(t(z) for z in v)
    ta = {k: t(v) for k, v in a.items()}
    okv = {"v2v": px, "v2i": py, "i2i": py, "i2v": px}
    oq = {"v2v": px, "v2i": px, "i2i": py, "i2v": py}
    masks = {u: TN.key_masks(oq[u], okv[u], lists[u], u in ("v2v", "i2i")) for u in lists}
    rx, ry = TN.sparse_block(ta["x"], ta["y"], ta["xi"], ta["yi"], tw, params, okv, masks)
    torch.autograd.backward([rx, ry], [torch.tensor(dx2, dtype=torch.float64),
                                       torch.tensor(dy2, dtype=torch.float64)])
    fwd = max(_rel(x2, rx), _rel(y2, ry))
    pairs = [(k, ins[k].grad, ta[k].grad) for k in a]
    mp = {"ln_ax_g": tw["ln_ax"][0], "ln_ax_b": tw["ln_ax"][1], "ln_ay_g": tw["ln_ay"][0],
          "ln_ay_b": tw["ln_ay"][1], "gate_x_w": tw["gate_x"][0], "gate_x_b": tw["gate_x"][1],
          "gate_y_w": tw["gate_y"][0], "gate_y_b": tw["gate_y"][1], "ln_fx_g": tw["ln_fx"][0],
          "ln_fx_b": tw["ln_fx"][1], "ln_fy_g": tw["ln_fy"][0], "ln_fy_b": tw["ln_fy"][1]}
    for s_ in ("x", "y"):
        for i, nm in enumerate(("w1", "b1", "w2", "b2")):
            mp[f"f{s_}_{nm}"] = tw[f"ffn_{s_}"][i]
    for name in BLOCK_PARAM_NAMES:
        pairs.append((name, getattr(mod, name).grad, mp[name].grad))
    for u in lists:
        um = mod.layer.uses[u]
        for name in ("w_q", "w_k", "w_v", "w_o", "gate_w", "gate_b"):
            pairs.append((f"{u}.{name}", getattr(um, name).grad, tw["uses"][u][name].grad))
        for tag in ("ck", "cv"):
            for i, s_ in enumerate(("w1", "b1", "w2", "b2")):
                pairs.append((f"{u}.{tag}_{s_}", getattr(um, f"{tag}_{s_}").grad,
                              tw["uses"][u][tag][i].grad))
    floor = 1e-2 * max(float(b.abs().max()) for _, _, b in pairs)
    return fwd, {n: _rel(x_, y_, floor) for n, x_, y_ in pairs}


@pytest.mark.gpu
def test_gpu_block_backward_matches_f64_autograd(cuda):
    """SparseBlockModule (fp32 kernels): forward and every gradient (inputs,
    injections, LayerNorms, use gates, FFN, the four uses' weights) within
    GRAD_RTOL of the f64 autograd block."""
    fwd, errs = _block_vs_oracle((4, 2, 8), 0.3, False)
    bad = {n: e for n, e in errs.items() if e > GRAD_RTOL}
    print(f"block fp32: fwd {fwd:.2e}, worst grad {max(errs.values()):.2e}")
    assert fwd < 1e-5 and not bad, (fwd, bad)


@pytest.mark.gpu
def test_gpu_block_backward_paper_heads_fast(cuda):
    """Paper heads, fast path (bf16 tensor-core branches, TF32 GEMMs)."""
    fwd, errs = _block_vs_oracle((32, 2, 32), 0.03, True)
    bad = {n: e for n, e in errs.items() if e > FAST_RTOL}
    print(f"block fast: fwd {fwd:.2e}, worst grad {max(errs.values()):.2e}")
    assert fwd < FAST_RTOL and not bad, (fwd, bad)
