"""Edge cases the reference's own tests pin (tests/test_nsa_attention.py:117-184,
tests/test_block_routing.py:165-174, tests/test_tokenizer.py), on the GPU path:
selection fallbacks, empty rows / contexts, rejected configurations,
behind-camera queries, ragged and empty token sets, the C-ABI error mapping.
"""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _tokens(seed, side=16, keep=0.2, d=4):
    import paper_2604_05182_b200 as L
    g = np.random.default_rng(seed)
    coords = np.argwhere(g.random((side, side, side)) < keep)
    feats = g.standard_normal((coords.shape[0], d)).astype(np.float32)
    return L.TokenSet("volume", feats, coords, (side, side, side))


def _qkv(seed, n, n_kv, p):
    g = np.random.default_rng(seed)
    f = lambda *s: g.standard_normal(s).astype(np.float32)   # noqa: E731
    return f(n, p.n_q_heads, p.head_dim), f(n_kv, p.n_kv_heads, p.head_dim), \
        f(n_kv, p.n_kv_heads, p.head_dim)


def test_empty_selection_falls_back_to_own_block(cuda):
    import paper_2604_05182_b200 as L
    p = L.AttentionParams(4, 2, 8)
    toks = _tokens(1)
    part = L.partition(toks)
    n = toks.count
    q, k, v = _qkv(1, n, n, p)
    sel = L.Selection([np.zeros(0, np.int64)] * n)
    got = L.sel_attention(q, k, v, part, sel, p, own_block=part.block_of_token)
    want = L.win_attention(q, k, v, part, part, p)
    assert np.max(np.abs(got.astype(np.float64) - want.astype(np.float64))) < 1e-6


def test_empty_selection_falls_back_to_lowest_block(cuda):
    import paper_2604_05182_b200 as L
    p = L.AttentionParams(4, 2, 8)
    toks = _tokens(2)
    part = L.partition(toks)
    opart = O.partition_tokens("volume", toks.coords, toks.grid_res)
    n = toks.count
    q, k, v = _qkv(2, n, n, p)
    got = L.sel_attention(q, k, v, part, L.Selection([np.zeros(0, np.int64)] * n), p)
    lowest = [np.asarray([opart.occupied_ids[0]])] * n
    want = O.sel_attention(q, k, v, opart, lowest, O.AttentionParams(4, 2, 8))
    assert np.max(np.abs(got.astype(np.float64) - want)) < 1e-6


def test_empty_selection_without_fallback_raises(cuda):
    import paper_2604_05182_b200 as L
    p = L.AttentionParams(4, 2, 8)
    toks = _tokens(3)
    part = L.partition(toks)
    n = toks.count
    q, k, v = _qkv(3, n, n, p)
    with pytest.raises(L.EmptyAttentionRowError):
        L.sel_attention(q, k, v, part, L.Selection([np.zeros(0, np.int64)] * n), p,
                        fallback=False)


def test_query_count_and_cross_window_rejected(cuda):
    import paper_2604_05182_b200 as L
    p = L.AttentionParams(4, 2, 8)
    a, b = L.partition(_tokens(4)), L.partition(_tokens(5))
    q, k, v = _qkv(4, a.n_tokens, a.n_tokens, p)
    with pytest.raises(L.ConfigurationError):
        L.sel_attention(q[:-1], k, v, a, L.full_selection(a.n_tokens, a), p)
    qb, kb, vb = _qkv(5, a.n_tokens, b.n_tokens, p)
    with pytest.raises(L.ConfigurationError):
        L.win_attention(qb, kb, vb, a, b, p)


def test_cmp_without_blocks_raises(cuda):
    import paper_2604_05182_b200 as L
    p = L.AttentionParams(4, 2, 8)
    q, _, _ = _qkv(6, 5, 1, p)
    empty = np.zeros((0, 2, 8), np.float32)
    with pytest.raises(L.EmptyContextError):
        L.cmp_attention(q, empty, empty, p)


def test_single_token_blocks_match_oracle(cuda):
    """Ragged extreme: every block holds one token (tiles of one query, one key)."""
    import paper_2604_05182_b200 as L
    p = L.AttentionParams(4, 2, 8)
    coords = np.array([[0, 0, 0], [8, 8, 8], [15, 0, 8], [0, 15, 15]])
    toks = L.TokenSet("volume", np.zeros((4, 4), np.float32), coords, (16, 16, 16))
    part = L.partition(toks)
    opart = O.partition_tokens("volume", coords, (16, 16, 16))
    q, k, v = _qkv(7, 4, 4, p)
    got = L.win_attention(q, k, v, part, part, p)
    want = O.win_attention(q, k, v, opart, O.AttentionParams(4, 2, 8))
    assert np.max(np.abs(got.astype(np.float64) - want)) < 1e-6


def test_query_behind_all_cameras_gets_empty_image_list(cuda):
    """`tests/test_block_routing.py:165-174`: a point behind every camera sees
    no image block."""
    import paper_2604_05182_b200 as L
    from fixtures import load_workload
    wl = load_workload("c1")
    x_d = np.zeros(((wl.vol_mask.shape[0] // wl.factor_vol) ** 3, 8), np.float32)
    ic = np.argwhere(wl.img_mask)
    coords = np.stack([ic[:, 0], ic[:, 2], ic[:, 1]], 1)
    y = L.TokenSet("image", np.zeros((coords.shape[0], 8), np.float32), coords,
                   (wl.img_mask.shape[0], wl.img_mask.shape[1], wl.img_mask.shape[2]))
    part = L.partition(y)
    # one forward-looking camera for every view; the query sits behind it
    eye, tgt = np.array([0.5, 0.5, 0.2]), np.array([0.5, 0.5, 1.0])
    fwd = (tgt - eye) / np.linalg.norm(tgt - eye)
    right = np.cross(fwd, [1.0, 0.0, 0.0])
    right /= np.linalg.norm(right)
    R = np.stack([right, np.cross(fwd, right), fwd], axis=1)
    K = np.array([[120.0, 0, 96.0], [0, 120.0, 96.0], [0, 0, 1.0]])
    cams = [(K, R, eye)] * wl.img_mask.shape[0]
    pts = L.TokenCoords3D(wl.img_points, np.zeros(coords.shape[0], bool))
    sel = L.route_to_image_blocks(np.array([0.5, 0.5, 0.05]), cams, part, pts, 4, 3)
    assert len(sel) == 0
    del x_d


def test_empty_masks_give_empty_token_sets(cuda):
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import coarse_inputs
    from fixtures import load_workload
    wl = load_workload("c1")
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, 64)
    vm = np.zeros_like(wl.vol_mask)
    im = np.zeros_like(wl.img_mask)
    x_up, y_up = L.upsample_select_tokens(x_d, y_d, vm, im, pe_v, pe_i, wl.factor_vol,
                                          wl.factor_img)
    assert x_up.count == 0 and y_up.count == 0
    assert L.partition(x_up).n_occupied == 0


def test_c_abi_status_maps_to_reference_errors(cuda):
    """A bad head geometry through the C ABI surfaces as ConfigurationError
    with the library's message."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200._native import call
    with pytest.raises(L.ConfigurationError, match="not divisible"):
        call("lsrm_nsa_attention_tc", None, 8, 1, 6, 4, 32, None, None, None, None, 16,
             None, None, 1, None, 1, None, None, 8, None, 8, 0, None, 2, None,
             torch.cuda.current_stream().cuda_stream)


def test_reference_api_reads_current_weights(cuda):
    """The reference functions are pure: a NumPy weight updated in place
    between two calls must be seen by the second call (no stale device
    copies), and self uses reject mismatched partitions like win_attention."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.errors import ConfigurationError
    g = np.random.default_rng(5)
    params = L.AttentionParams(4, 2, 8)
    coords = np.stack(np.meshgrid(np.arange(12), np.arange(12), np.arange(4), indexing="ij"),
                      -1).reshape(-1, 3)[g.permutation(576)[:300]]
    toks = L.TokenSet("volume", np.zeros((300, 32), np.float32), coords, (16,) * 3)
    part = L.partition(toks)
    x = g.standard_normal((300, 32)).astype(np.float32)
    w = L.init_nsa_weights(0, params, 3, "t")
    sel = L.Selection([part.occupied_ids[:2].copy() for _ in range(300)])
    a = L.nsa_cross_attention(x, x, part, part, sel, w, params)
    w.w_o *= 2.0                       # in-place update of the caller's array
    b = L.nsa_cross_attention(x, x, part, part, sel, w, params)
    assert np.allclose(b, 2.0 * a, rtol=1e-6, atol=1e-7)
    toks2 = L.TokenSet("volume", np.zeros((300, 32), np.float32), coords[::-1].copy(), (16,) * 3)
    with pytest.raises(ConfigurationError):
        L.nsa_cross_attention(x, x, L.partition(toks2), part, sel, w, params)


@pytest.mark.parametrize("b_i", [1, 5, 16, 70, 200])
def test_image_router_dense_views_and_ties(cuda, b_i):
    """Image router against the oracle where views hold many occupied blocks
    (144 per view, more than a warp) and the shortlist cut b_i falls inside
    them, with duplicated token points so minimum distances tie (stable row
    order decides), queries in front of and behind the cameras."""
    import paper_2604_05182_b200 as L
    from paper_2604_05182_b200.workloads import orbit_cameras
    g = np.random.default_rng(b_i)
    views, side = 3, 96
    cams = orbit_cameras(views, 1.7, 20.0, (8 * side, 8 * side))
    ic = np.argwhere(g.random((views, side, side)) < 0.6)
    coords = np.stack([ic[:, 0], ic[:, 2], ic[:, 1]], 1)
    y = L.TokenSet("image", np.zeros((coords.shape[0], 4), np.float32), coords,
                   (views, side, side))
    part = L.partition(y)
    assert np.diff(np.searchsorted(part.block_views, np.arange(views + 1))).max() > 64
    pts = g.random((coords.shape[0], 3))
    pts[1::2] = pts[::2][: pts[1::2].shape[0]]          # duplicated points -> tied minima
    queries = np.concatenate([g.random((300, 3)), g.random((20, 3)) * 6.0 - 3.0])
    from paper_2604_05182_b200.block_routing import _route_points_to_image
    got = _route_points_to_image(queries, cams, part, L.TokenCoords3D(pts, np.zeros(
        pts.shape[0], bool)), b_i, 8)
    opart = O.partition_tokens("image", coords, (views, side, side))
    want = O.route_image(queries, [c[:3] for c in cams], opart, pts, b_i, 8)
    for a, b in zip(got.lists, want):
        assert np.array_equal(a, b)
