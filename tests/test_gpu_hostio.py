"""`lsrm_h2d_rows` (csrc/hostio.cu): host rows -> device rows with the row
permutation and the bf16 rounding done on host threads into pinned staging
chunks. It must be bit-identical to uploading the f32 rows and running the
device gather + `lsrm_cast`, for every chunking (rows spanning several 8 MiB
staging slots, ragged last chunk, empty input) and for NaN / inf / subnormal
values."""

import numpy as np
import pytest
import torch

from paper_2604_05182_b200 import _dev as D
from paper_2604_05182_b200 import _ops
from paper_2604_05182_b200._native import call
from paper_2604_05182_b200.errors import ConfigurationError

pytestmark = pytest.mark.gpu


def _h2d(a, idx, to_bf16, ld_dst=None):
    n = 0 if idx is None else len(idx)
    n = a.shape[0] if idx is None else n
    d = a.shape[1]
    ld = ld_dst or d
    out = torch.zeros((n, ld), dtype=torch.bfloat16 if to_bf16 else torch.float32,
                      device="cuda")
    call("lsrm_h2d_rows", int(to_bf16), a.ctypes.data, a.shape[1],
         0 if idx is None else idx.ctypes.data, n, d, out.data_ptr(), ld, D.stream())
    torch.cuda.synchronize()
    return out


def _reference(a, idx, to_bf16):
    t = torch.from_numpy(a).cuda()
    if idx is not None:
        t = _ops.gather_rows(t, torch.from_numpy(idx).cuda())
    return _ops.cast(t, torch.bfloat16) if to_bf16 else t


@pytest.mark.parametrize("to_bf16", [True, False])
@pytest.mark.parametrize("n,d", [(1, 1024), (3000, 1024), (9000, 1024), (5, 96)])
def test_h2d_rows_bit_exact(to_bf16, n, d):
    rng = np.random.default_rng(n + d)
    a = (rng.standard_normal((n, d)) * 10 ** rng.uniform(-6, 6, (n, 1))).astype(np.float32)
    flat = a.reshape(-1)
    flat[:8] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1e-40, -3e-39, 3.3895314e38]
    idx = rng.permutation(n).astype(np.int64)
    got = _h2d(a, idx, to_bf16)
    ref = _reference(a, idx, to_bf16)
    assert torch.equal(got.view(torch.int16 if to_bf16 else torch.int32),
                       ref.view(torch.int16 if to_bf16 else torch.int32))
    got_id = _h2d(a, None, to_bf16)
    assert torch.equal(got_id.view(torch.int16 if to_bf16 else torch.int32),
                       _reference(a, None, to_bf16).view(torch.int16 if to_bf16 else torch.int32))


def test_h2d_rows_padded_destination_and_empty():
    a = np.arange(40 * 64, dtype=np.float32).reshape(40, 64)
    got = _h2d(a, None, True, ld_dst=80)
    assert torch.equal(got[:, :64], _ops.cast(torch.from_numpy(a).cuda(), torch.bfloat16))
    assert not got[:, 64:].any()
    empty = np.zeros((0, 64), np.float32)
    assert _h2d(empty, None, True).shape == (0, 64)
    with pytest.raises(ConfigurationError):
        call("lsrm_h2d_rows", 1, a.ctypes.data, 32, 0, 40, 64, 0, 64, D.stream())


def test_host_threads_pool():
    from paper_2604_05182_b200._native import lib
    assert 1 <= lib().lsrm_host_threads() <= 16
