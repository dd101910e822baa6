"""The pipelined host-API path (H2D | compute | D2H streams, double-buffered,
CUDA graphs) returns exactly what the serial `forward_host` returns."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_pipeline_matches_forward_host(cuda):
    from paper_2604_05182_b200.layer import HostPipeline, SparseAttentionLayer, build_instance
    from paper_2604_05182_b200.tensor_core import AttentionParams
    import torch
    inst = build_instance("c1", params=AttentionParams(32, 2, 32))
    layer = SparseAttentionLayer(inst)
    want = layer.forward_host(inst.x_hat, inst.y_hat)
    xp = torch.from_numpy(np.ascontiguousarray(inst.x_hat, np.float32)).pin_memory()
    yp = torch.from_numpy(np.ascontiguousarray(inst.y_hat, np.float32)).pin_memory()
    pipe = HostPipeline(layer, n_slots=2)
    ms = pipe.run(xp, yp, 3)
    assert ms > 0
    for slot in range(2):
        for u, w in want.items():
            assert np.array_equal(pipe.host_out[slot][u].numpy(), w), (slot, u)
