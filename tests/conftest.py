import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def unflat(vals, lens):
    out, pos = [], 0
    for n in lens:
        out.append(vals[pos:pos + n])
        pos += n
    return out


@pytest.fixture(scope="session")
def ref_c1():
    return golden("ref_c1.npz")


@pytest.fixture(scope="session")
def ref_small():
    return golden("ref_small.npz")


@pytest.fixture(scope="session")
def cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback exists)"
    from paper_2604_05182_b200._native import lib
    lib()
    return torch.device("cuda", 0)
