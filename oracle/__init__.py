"""CPU oracle for the LSRM sparse-attention hot path — TEST INFRASTRUCTURE ONLY.

This package is a plain NumPy restatement of the reference algorithm
(`/root/reference/pkg/src/lsrm`, lsrm 0.1.0) for exactly the functions on the
hot path named by BASELINE.json's north star.  Every function cites the
reference file:line it restates.

Rules (enforced by review):
  * only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
    ``--impl reference`` legs of ``bench.py`` may import this package;
  * it is the checker, never the thing measured or shipped: the product
    package ``paper_2604_05182_b200`` never imports it and has no CPU
    fallback.

Parity of this oracle is PINNED against the reference itself: the fixtures
under ``tests/golden/`` were produced by importing the real ``lsrm`` package
in the build container (script: ``tests/golden/make_golden.py``), and
``tests/test_oracle_golden.py`` checks the restatement against them
bit-for-bit (integer/index outputs) or to the reference's own tolerances
(floating-point outputs).

Numeric conventions follow the reference (`lsrm/tensor_core.py:1-12`):
float32 storage, float64 accumulation, head-split attention tensors, query
head g reads kv head g // group_size, logit scale 1/sqrt(head_dim).
"""

from .numerics import (ACC, DTYPE, AttentionParams, affine, dense_attention,
                       gelu, layer_norm, sigmoid)
from .rng import normal_f32, stream, tag_counter
from .partition import (Partition, compress_block_kv, partition_tokens,
                        res_block)
from .attention import (GatherTable, NsaWeights, build_gather_table,
                        cmp_attention, combine_branches, nsa_gates,
                        nsa_use, score_topk_blocks, sel_attention,
                        win_attention)
from .routing import (RoutingPlan, build_routing_plan, route_image,
                      route_volume)
from .tokens import (TokenSet, eval_sdf, factorized_pos_embed,
                     foreground_patch_mask, informative_voxel_mask,
                     upsample_select_tokens)
from .seqpar import (Topology, all_gather_kv_accounting, all_to_all_accounting,
                     naive_contiguous_shards, shard_blocks)
from .block import (SparseBlockWeights, ffn_forward, init_nsa_weights,
                    init_sparse_block, sparse_block_forward)
