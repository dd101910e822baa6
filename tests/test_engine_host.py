"""Host-side tiling logic of the bf16 engine (no GPU needed): query tiles
cover every token exactly once, never straddle a query block, and carry the
block's own kv row for self uses (`engine.query_tiles`)."""

import numpy as np
import pytest

import oracle as O


@pytest.mark.parametrize("group,self_use", [(16, True), (16, False), (4, True)])
def test_query_tiles_cover_blocks(group, self_use):
    from paper_2604_05182_b200.engine import query_tiles
    g = np.random.default_rng(group)
    coords = np.argwhere(g.random((32, 32, 32)) < 0.08)
    part = O.partition_tokens("volume", coords, (32, 32, 32))
    tiles = query_tiles(part, group, self_use)
    T = 128 // group
    seen = np.zeros(part.block_of_token.size, int)
    for first, cnt, own, _ in tiles:
        assert 1 <= cnt <= T
        seen[first:first + cnt] += 1
        rows = np.searchsorted(part.block_offsets, [first, first + cnt - 1], side="right") - 1
        assert rows[0] == rows[1]                      # one query block per tile
        assert own == (rows[0] if self_use else -1)
    assert np.all(seen == 1)
