"""B200-native drop-in for the LSRM sparse-attention hot path (arXiv 2604.05182).

Mirrors the reference `lsrm` module API for the hot path:
NSA three-branch attention, the 3D-aware router, foreground/voxel pruning and
compaction, block partition/compression and block-aware sequence parallelism.
All compute runs in the in-tree C-ABI library `_lib/liblsrm_b200.so`
(hand-written sm_100a CUDA + cuBLAS for plain GEMMs); there is no CPU fallback.
"""

from .errors import (BehindCameraError, ConfigurationError, EmptyAttentionRowError,
                     EmptyContextError, GoldenFormatError, LsrmError, OutOfDomainError,
                     ProtocolError, VerificationError)
from .tensor_core import AttentionParams, read_goldens, write_goldens
from .tokenizer import (PosEmbed, TokenSet, foreground_patch_mask, informative_voxel_mask,
                        init_pos_embed, upsample_select_tokens)
from .block_partition import (BlockPartition, CompressWeights, compress_block_kv,
                              init_compress_weights, occupancy_stats, partition, res_block)
from .nsa_attention import (GatherTable, NsaWeights, Selection, build_gather_table,
                            cmp_attention, combine_nsa_branches, full_selection,
                            init_nsa_weights, nsa_cross_attention, nsa_gates,
                            read_selection, score_topk_blocks, sel_attention,
                            win_attention, write_selection)
from .block_routing import (RoutingBudgets, RoutingPlan, TokenCoords3D, build_routing_plan,
                            route_to_image_blocks, route_to_volume_blocks,
                            image_token_coords, volume_token_coords, write_plan)

from .seq_parallel import (TOKEN_COORD_BYTES, WorkerTopology, all_gather_kv, all_to_all,
                           imbalance_report, makespan_ratio, message_log_to_csv,
                           naive_contiguous_shards, naive_split_loads, parallel_sparse_stage,
                           shard_blocks, shard_blocks_by_cost)
from .recon_pipeline import (DecodeWeights, DecoderHeads, DenseBlockWeights, FeatureVolume,
                             MhaWeights, build_sparse_context, build_sparse_features,
                             decode_feature_volume, decode_point, decode_points,
                             dense_block_forward, dense_stage_forward, init_decode,
                             init_decoder_heads, init_dense_block, mha_forward, query_field,
                             sparse_block_forward, sparse_stage_forward, affine_exact)
from .sdf import DecodedSdf, callable_field, decoded_sdf_field

__version__ = "0.1.0"
