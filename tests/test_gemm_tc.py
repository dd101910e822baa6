"""The hand-written tcgen05 GEMM (csrc/gemm_tc.cu) against a plain PyTorch
fp32 reference of the same op, on the shapes the layer uses and on ragged
tails (m, n, k not multiples of the 128 x 256 x 64 tile), every epilogue
(bias bf16/f32, exact-erf gelu, residual bf16/f32, bf16/f32 out) and grouped
launches.

Tolerance: the operands are bf16 and the accumulation fp32 in both, so an
f32 output differs only by summation order (<= 1e-4 relative to the row
scale); a bf16 output adds one rounding (<= 2^-8 relative)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(a, bt, bias=None, res=None, gelu=False):
    y = a.float() @ bt.float().t()
    if bias is not None:
        y = y + bias.float()
    if gelu:
        y = torch.nn.functional.gelu(y)
    if res is not None:
        y = y + res.float()
    return y


def _close(got, want, out_dtype):
    scale = want.abs().amax().item() + 1e-6
    err = (got.float() - want).abs().amax().item() / scale
    bound = 1e-4 if out_dtype == torch.float32 else 8e-3
    assert err <= bound, f"max rel err {err:.3e} > {bound}"
    return err


def _mk(g, *shape, dtype=torch.bfloat16, scale=1.0):
    return (torch.randn(*shape, generator=g, device="cuda") * scale).to(dtype)


@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (1, 8, 8), (300, 264, 72), (1000, 520, 136),
                                   (16815, 1024, 1024), (257, 7424, 1024)])
def test_gemm_shapes(cuda, m, n, k):
    from paper_2604_05182_b200 import _ops
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n + k)
    a, bt = _mk(g, m, k), _mk(g, n, k, scale=0.05)
    got = _ops.gemm_bf16(a, bt)
    torch.cuda.synchronize()
    _close(got, _ref(a, bt), torch.bfloat16)
    got32 = _ops.gemm_bf16(a, bt, out_dtype=torch.float32)
    _close(got32, _ref(a, bt), torch.float32)


@pytest.mark.parametrize("bias_dt", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("res_dt", [None, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("gelu", [False, True])
def test_gemm_epilogues(cuda, bias_dt, res_dt, gelu):
    from paper_2604_05182_b200 import _ops
    g = torch.Generator(device="cuda").manual_seed(11)
    m, n, k = 517, 776, 264
    a, bt = _mk(g, m, k), _mk(g, n, k, scale=0.05)
    bias = _mk(g, n, dtype=bias_dt)
    res = _mk(g, m, n, dtype=res_dt) if res_dt is not None else None
    out_dt = res_dt or torch.bfloat16
    got = _ops.gemm_bf16(a, bt, out_dtype=out_dt, bias=bias, res=res, gelu=gelu)
    torch.cuda.synchronize()
    _close(got, _ref(a, bt, bias, res, gelu), out_dt)


def test_gemm_residual_in_place(cuda):
    """res may alias the output (the FFN's second GEMM adds into x1)."""
    from paper_2604_05182_b200 import _ops
    g = torch.Generator(device="cuda").manual_seed(5)
    a, bt = _mk(g, 333, 128), _mk(g, 256, 128, scale=0.05)
    x = _mk(g, 333, 256, dtype=torch.float32)
    want = _ref(a, bt, res=x)
    _ops.gemm_bf16(a, bt, out=x, res=x)
    torch.cuda.synchronize()
    _close(x, want, torch.float32)


def test_gemm_grouped_launch(cuda):
    """Several problems of different shapes in ONE persistent launch, with
    strided operand views (the engine reads column slices of its buffers)."""
    from paper_2604_05182_b200 import _ops
    from paper_2604_05182_b200._native import launch_count, reset_launch_count
    g = torch.Generator(device="cuda").manual_seed(3)
    big = _mk(g, 700, 2304)
    shapes = [(700, 1024, 1024), (129, 264, 512), (65, 8, 64), (1, 1024, 2048)]
    probs, refs, outs = [], [], []
    for i, (m, n, k) in enumerate(shapes):
        a = big[:m, 64 * i:64 * i + k]          # row stride 2304
        bt = _mk(g, n, k, scale=0.05)
        bias = _mk(g, n, dtype=torch.float32) if i % 2 else None
        out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        probs.append(_ops.gemm_problem(a, bt, out, bias=bias))
        refs.append(_ref(a, bt, bias))
        outs.append(out)
    reset_launch_count()
    _ops.gemm_tc(probs)
    assert launch_count() == 1
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        _close(o, r, torch.bfloat16)


def test_gemm_deterministic(cuda):
    from paper_2604_05182_b200 import _ops
    g = torch.Generator(device="cuda").manual_seed(9)
    a, bt = _mk(g, 2000, 1024), _mk(g, 1536, 1024, scale=0.05)
    r1 = _ops.gemm_bf16(a, bt, out_dtype=torch.float32)
    r2 = _ops.gemm_bf16(a, bt, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(r1, r2)


def test_gemm_rejects_bad_strides(cuda):
    from paper_2604_05182_b200 import _ops
    from paper_2604_05182_b200.errors import ConfigurationError
    a = torch.zeros(16, 12, dtype=torch.bfloat16, device="cuda")
    bt = torch.zeros(16, 12, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ConfigurationError):
        _ops.gemm_bf16(a, bt)


@pytest.mark.parametrize("a_mn,b_mn", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (1024, 1024, 16815), (300, 264, 72),
                                   (64, 128, 1000), (1000, 520, 137)])
def test_gemm_mn_major_operands(cuda, a_mn, b_mn, m, n, k):
    """A given as A^T [k,m] and/or B as W [k,n] (MN-major, no transposed copy):
    the weight-gradient form X^T . dY of the training path."""
    from paper_2604_05182_b200 import _ops
    if not (a_mn and b_mn) and k % 8:
        pytest.skip("a K-major operand needs k % 8 == 0")
    if (a_mn and m % 8) or n % 8:
        pytest.skip("row strides must be multiples of 8")
    g = torch.Generator(device="cuda").manual_seed(m + 3 * n + 5 * k + 7 * a_mn + 11 * b_mn)
    a, bt = _mk(g, m, k), _mk(g, n, k, scale=0.05)
    a_op = a.t().contiguous() if a_mn else a
    b_op = bt.t().contiguous() if b_mn else bt
    for out_dtype in (torch.float32, torch.bfloat16):
        out = torch.empty((m, n), dtype=out_dtype, device="cuda")
        _ops.gemm_tc([_ops.gemm_problem(a_op, b_op, out, a_mn=a_mn, b_mn=b_mn)])
        torch.cuda.synchronize()
        _close(out, _ref(a, bt), out_dtype)


@pytest.mark.parametrize("trans_a,trans_b", [(False, False), (False, True), (True, False),
                                             (True, True)])
@pytest.mark.parametrize("m,n,k", [(1000, 1024, 16815), (16815, 1024, 1024), (37, 64, 13),
                                   (64, 64, 16815)])
def test_gemm_train_all_transposes(cuda, trans_a, trans_b, m, n, k):
    """gemm_train (fp32 in/out, bf16 operands) for every op(a) / op(b)
    combination against torch on the bf16-rounded operands, incl. k % 8 != 0
    (zero-padded K), split K (outputs of few tiles with long K: partial
    products summed in slice order) and beta = 1 accumulation; the cast cache
    returns the same copy for a repeated operand."""
    from paper_2604_05182_b200 import _ops
    g = torch.Generator(device="cuda").manual_seed(m + n + k + 2 * trans_a + trans_b)
    A = torch.randn(m, k, generator=g, device="cuda")
    B = torch.randn(k, n, generator=g, device="cuda") * 0.05
    a = A.t().contiguous() if trans_a else A
    b = B.t().contiguous() if trans_b else B
    want = A.bfloat16().float() @ B.bfloat16().float()
    cache = {}
    got = _ops.gemm_train(a, b, trans_a=trans_a, trans_b=trans_b, cache=cache)
    n_cached = len(cache)
    acc = _ops.gemm_train(a, b, trans_a=trans_a, trans_b=trans_b, out=got.clone(), beta=1.0,
                          cache=cache)
    torch.cuda.synchronize()
    assert len(cache) == n_cached == 2
    _close(got, want, torch.float32)
    _close(acc, 2 * want, torch.float32)


@pytest.mark.parametrize("n", [8 * 12345, 8 * 12345 + 3])
def test_cast_vectorised_and_tail(cuda, n):
    from paper_2604_05182_b200 import _ops
    x = torch.randn(n, device="cuda") * 100
    x[:4] = torch.tensor([float("nan"), float("inf"), -0.0, 1e-40])
    y = _ops.cast(x, torch.bfloat16)
    assert torch.equal(y.view(torch.int16)[4:], x.bfloat16().view(torch.int16)[4:])
    assert torch.isnan(y[0]) and torch.isinf(y[1])
    z = _ops.cast(y, torch.float32)
    assert torch.equal(z[4:], y[4:].float())


def test_gemm_train_split_k_deterministic(cuda):
    """Split-K partial products are summed in slice order: two runs of the
    same weight-gradient GEMM give identical bytes."""
    from paper_2604_05182_b200 import _ops
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(16815, 1024, generator=g, device="cuda")
    dy = torch.randn(16815, 1024, generator=g, device="cuda")
    a = _ops.gemm_train(x, dy, trans_a=True)
    b = _ops.gemm_train(x, dy, trans_a=True)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
