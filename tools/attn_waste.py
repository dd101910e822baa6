"""Where the fused attention kernel's exponentials go (C3, default block tiles):
per use, useful (row, key) pairs against what the streamed chunks cost at
three granularities - per row with 16-row block padding, per warp (the two
tokens a softmax warp's 32 rows cover; dead 32-key pieces are skipped), and
per tile (8 tokens, every row streams the tile's union) - plus the rows of
partial tiles (tokens past the block's end).

    python tools/attn_waste.py          # GPU box (builds the C3 instance)
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2604_05182_b200 import _dev as D
    from paper_2604_05182_b200.engine import USE_GEOM, _padded
    from paper_2604_05182_b200.layer import SparseAttentionLayer, build_instance
    inst = build_instance(sys.argv[1] if len(sys.argv) > 1 else "c3")
    eng = SparseAttentionLayer(inst).engine
    p = inst.params
    G = p.n_q_heads // p.n_kv_heads
    T = 128 // G
    out = {}
    for use in eng.uses:
        qs, ks, ng = USE_GEOM[use]
        mq, mk = eng.meta[qs], eng.meta[ks]
        occ = mk.part.occupancy.astype(np.int64)
        pad = _padded(occ)
        rows = D.host(eng.rows[use])
        cnt = D.host(eng.count[use])
        blk = np.repeat(np.arange(mq.loc_off_host.size - 1), np.diff(mq.loc_off_host))
        key = np.sort(np.where(rows >= 0, rows, np.iinfo(np.int32).max), axis=1)
        sig = tuple(key[:, j] for j in reversed(range(key.shape[1])))
        perm = np.lexsort(sig + (blk,))
        tiles = D.host(eng.tiles[use])
        B = mk.part.n_occupied
        cmp_pad = (B + 15) // 16 * 16
        qocc = mq.part.occupancy.astype(np.int64)
        useful = pad_row = warp2 = tile = 0
        empty_rows = 0
        for first, tc, own, _ in tiles:
            toks = perm[first:first + tc]
            sel = [set(rows[t, :cnt[t]].tolist()) for t in toks]
            own_k = pad[own] if (ng == 3 and own >= 0) else 0
            own_u = qocc[own] if ng == 3 and own >= 0 else 0
            for s in sel:
                useful += B + sum(occ[r] for r in s) + own_u
                pad_row += cmp_pad + sum(pad[r] for r in s) + own_k
            for w in range(0, T, 2):
                u = set().union(*sel[w:w + 2]) if w < tc else set()
                live = cmp_pad + sum(pad[r] for r in u) + own_k if w < tc else 0
                warp2 += 2 * live
            un = set().union(*sel)
            tile += T * (cmp_pad + sum(pad[r] for r in un) + own_k)
            empty_rows += T - tc
        out[use] = {"useful_Mpairs_per_head": useful / 1e6,
                    "row_padding_x": pad_row / useful, "warp_union_x": warp2 / useful,
                    "tile_union_x": tile / useful, "partial_tile_rows_frac":
                    empty_rows / (len(tiles) * T), "tiles": int(len(tiles))}
        print(use, json.dumps(out[use]), flush=True)
    tot_u = sum(v["useful_Mpairs_per_head"] for v in out.values())
    print("all uses: warp-union x", sum(v["warp_union_x"] * v["useful_Mpairs_per_head"]
                                        for v in out.values()) / tot_u,
          "tile-union x", sum(v["tile_union_x"] * v["useful_Mpairs_per_head"]
                              for v in out.values()) / tot_u)


if __name__ == "__main__":
    main()
