"""Block-aware sequence parallelism: sharding and collective accounting
(TEST INFRASTRUCTURE ONLY).

Restates `lsrm/seq_parallel.py:93-218`.  Data movement is the checker's
in-process copy; only the ownership rules and the (phase, kind, src, dst,
bytes) message log are reproduced.
"""

from dataclasses import dataclass, field

import numpy as np

TOKEN_COORD_BYTES = 12


@dataclass
class Topology:
    n_workers: int
    vol_rows: list
    img_rows: list
    vol_tokens: list
    img_tokens: list
    loads: np.ndarray
    message_log: list = field(default_factory=list)


def shard_blocks(part_vol, part_img, n_workers):
    """Greedy LPT over pooled blocks: occupancy descending, ties volume first
    then lower block id; lightest worker, ties lower id
    (`seq_parallel.py:93-131`)."""
    items = sorted((-int(p.occupancy[r]), m, int(p.occupied_ids[r]), r)
                   for m, p in enumerate((part_vol, part_img))
                   for r in range(p.n_occupied))
    loads = np.zeros(n_workers, np.int64)
    rows = [[[] for _ in range(n_workers)] for _ in range(2)]
    for neg, m, _, r in items:
        w = int(np.argmin(loads))
        loads[w] -= neg
        rows[m][w].append(r)
    rows = [[np.array(sorted(x), np.int64) for x in rm] for rm in rows]

    def toks(p, rr):
        return [np.concatenate([p.tokens_in_row(r) for r in x]) if x.size
                else np.zeros(0, np.int64) for x in rr]
    return Topology(n_workers, rows[0], rows[1], toks(part_vol, rows[0]),
                    toks(part_img, rows[1]), loads)


def naive_contiguous_shards(n_tokens, n_workers):
    """`seq_parallel.py:134-139`."""
    e = np.linspace(0, n_tokens, n_workers + 1).astype(np.int64)
    return [np.arange(a, b, dtype=np.int64) for a, b in zip(e[:-1], e[1:])]


def all_to_all_accounting(shards_in, shards_out, topo: Topology, phase,
                          bytes_per_token):
    """Per ordered pair byte log of a re-shard (`seq_parallel.py:146-178`)."""
    n = topo.n_workers
    owner = {}
    for w, ids in enumerate(shards_in):
        for t in ids.tolist():
            if t in owner:
                raise ValueError(f"ProtocolError: token {t} produced twice")
            owner[t] = w
    moved = np.zeros((n, n), np.int64)
    for dst, ids in enumerate(shards_out):
        for t in ids.tolist():
            if t not in owner:
                raise ValueError(f"ProtocolError: token {t} never produced")
            moved[owner[t], dst] += 1
    for s in range(n):
        for d in range(n):
            if s != d and moved[s, d]:
                topo.message_log.append((phase, "all_to_all", s, d,
                                         int(moved[s, d]) * bytes_per_token))
    return shards_out


def all_gather_kv_accounting(n_tok_per_worker, n_blocks_per_worker, width,
                             topo: Topology, phase):
    """Byte log of one All-gather-KV: 4*2*(|k| + |k_cmp|) from every source
    with data to every other worker (`seq_parallel.py:211-217`)."""
    n = topo.n_workers
    kv = [4 * 2 * (t * width + b * width)
          for t, b in zip(n_tok_per_worker, n_blocks_per_worker)]
    for s in range(n):
        for d in range(n):
            if s != d and kv[s]:
                topo.message_log.append((phase, "all_gather_kv", s, d, kv[s]))
