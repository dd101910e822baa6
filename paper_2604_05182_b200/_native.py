"""ctypes binding of the in-tree C-ABI library (include/lsrm_b200.h).

There is deliberately no CPU fallback: if the library is missing or no CUDA
device is visible, every compute entry point raises.  `lib()` loads
`_lib/liblsrm_b200.so` once per process; `call(name, *args)` maps non-zero
status codes onto the reference exception classes.
"""

import ctypes as C
import os

from .errors import STATUS_CLASSES, LsrmError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "liblsrm_b200.so")

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int
F32 = C.c_float
F64 = C.c_double
SZ = C.c_size_t

# name -> (restype, argtypes); must match include/lsrm_b200.h
SIGNATURES = {
    "lsrm_abi_version": (I32, []),
    "lsrm_last_error": (C.c_char_p, []),
    "lsrm_launch_count": (I64, []),
    "lsrm_reset_launch_count": (None, []),
    "lsrm_partition_workspace": (SZ, [I64, I64]),
    "lsrm_partition": (I32, [I32, P, I64, I32, I32, I32, I32, P, P, P, P, P, P, P,
                             P, P, SZ, P]),
    "lsrm_compress_block": (I32, [I32, P, I64, I64, I32, P, P, P, P, P, P, I64, P,
                                  P, P]),
    "lsrm_route_volume": (I32, [P, I64, P, I64, I32, P, P, P]),
    "lsrm_route_image": (I32, [P, I64, P, I32, P, P, I64, P, P, P, I32, I32, I32, P, P, P]),
    "lsrm_block_bounds": (I32, [P, I64, P, I64, P, P]),
    "lsrm_build_gather_table": (I32, [P, P, I64, I32, P, I32, P, P, I64, P, P, P, P,
                                      P, P]),
    "lsrm_foreground_mask": (I32, [P, I32, I32, I32, I32, P, P]),
    "lsrm_voxel_mask": (I32, [P, I32, I32, F64, I32, P, P]),
    "lsrm_compact_workspace": (SZ, [I64]),
    "lsrm_compact_volume": (I32, [P, I32, I32, P, I32, P, P, P, P, P, I64, P, P, SZ,
                                  P]),
    "lsrm_compact_image": (I32, [P, I32, I32, I32, P, I32, P, P, P, P, I64, P, P,
                                 SZ, P]),
    "lsrm_attention_f32": (I32, [I32, P, I64, I32, I32, I32, P, P, I64, P, P, P,
                                 I32, P, P, P, I64, P, P]),
    "lsrm_gated_merge_f32": (I32, [P, I64, P, I32, P, P, P, I64, I32, P, P]),
    "lsrm_sigmoid_f32": (I32, [P, I64, P, I64, I32, P, P]),
    "lsrm_score_topk": (I32, [P, I64, I32, I32, I32, P, I64, I32, P, P, P]),
    "lsrm_gemm": (I32, [I32, I64, I64, I64, P, I64, P, I64, P, I64, P]),
    "lsrm_nsa_attention_tc": (I32, [P, I64, I64, I32, I32, I32, P, P, P, P, I64, P, P,
                                    I64, P, I64, P, P, I32, P, I64, I64, P, I32, P, P]),
    "lsrm_kv_interleave": (I32, [I32, P, I64, I64, I32, I32, I32, P, P, I64, P, I64,
                                 P, P]),
    "lsrm_debug_set_trace": (I32, [P]),
    "lsrm_copy_segments": (I32, [P, P, P, I64, P]),
    "lsrm_kv_prepare_jobs": (I32, [P, I32, I64, I32, I32, P]),
    "lsrm_nsa_attention_tc_multi": (I32, [P, I32, I32, I32, I32, P, I64, P, P]),
    "lsrm_image_token_points": (I32, [P, I64, P, P, I32, I32, P, I32, F64, P, P, P]),
    "lsrm_pluecker_rays": (I32, [P, P, I32, I32, I32, P, P]),
    "lsrm_silhouette_alpha": (I32, [P, P, I32, I32, I32, P, I32, P, P]),
    "lsrm_add_layer_norm": (I32, [I32, P, P, I32, I64, I32, P, P, F32, P, I32, P, P]),
    "lsrm_gate_mix_layer_norm": (I32, [I32, P, P, I64, I32, P, P, P, I32, I64, I32, P, P, P,
                                       F32, I32, P, P]),
    "lsrm_bias_act": (I32, [I32, P, I32, I64, P, I64, I32, I32, P, P, I32, I64, P]),
    "lsrm_gather_rows": (I32, [I32, P, I64, P, I64, I64, P, I64, P]),
    "lsrm_scatter_rows": (I32, [I32, P, I64, P, I64, I64, P, I64, P]),
    "lsrm_cast": (I32, [I32, P, P, I64, P]),
    "lsrm_layer_norm": (I32, [I32, P, I64, I32, P, P, F32, I32, P, P]),
    "lsrm_attention_bwd_workspace": (SZ, [I64, I32, I64, I32, I32, I32]),
    "lsrm_attention_bwd_f32": (I32, [I32, P, P, P, I64, I32, I32, I32, P, P, I64, P, I32, I32,
                                     P, P, I32, P, I32, P, P, P, P, SZ, P]),
    "lsrm_attention_bwd_mma": (I32, [I32, P, P, P, P, P, I64, I32, I32, I32, P, P, I64, P, I32, I32,
                                     P, P, I32, P, I32, P, P, P, P, P, P, SZ, P]),
    "lsrm_transpose_rows_workspace": (SZ, [I64, I32]),
    "lsrm_transpose_rows": (I32, [P, P, I64, I32, I32, P, P, P, SZ, P]),
    "lsrm_gate_merge_bwd_f32": (I32, [P, I64, P, I32, P, P, P, P, I64, I32, I32, P, P, P, P,
                                      P]),
    "lsrm_gated_merge_fast_f32": (I32, [P, I64, P, I32, P, P, P, I64, I32, P, P]),
    "lsrm_res_block_bwd_f32": (I32, [P, I64, I32, P, P, P, P, P, P, P, P, P, P, P]),
    "lsrm_decode_scatter": (I32, [P, I32, I32, I32, P, P]),
    "lsrm_sparse_features": (I32, [P, P, I64, I32, I32, I64, P, P, P]),
    "lsrm_decode_points": (I32, [P, I32, P, P, I32, I32, P, I64, P, I32, I32, P, P, P, P]),
    "lsrm_gemm_f32_ex": (I32, [I32, I32, I64, I64, I64, F32, P, I64, P, I64, F32, P, I64, I32,
                               P]),
    "lsrm_attention_fwd_mma": (I32, [I32, P, I64, I32, I32, I32, P, P, I64, P, P, P, I32, P, P, P,
                                     P]),
    "lsrm_check_field": (I32, [P]),
    "lsrm_image_token_points_field": (I32, [P, I64, P, P, I32, I32, P, F64, P, P, P]),
    "lsrm_ray_sample_points": (I32, [P, I64, P, P, I32, I32, P, P, P]),
    "lsrm_voxel_mask_field": (I32, [P, I32, F64, I32, I32, I32, P, P]),
    "lsrm_voxel_sample_points": (I32, [I32, I32, I32, I32, P, P]),
    "lsrm_affine_exact": (I32, [P, I64, I64, I32, P, P, I32, I32, P, I64, P]),
    "lsrm_gemm_tc": (I32, [P, I32, P]),
    "lsrm_compact_rows": (I32, [I32, P, I64, I64, I32, I32, I32, P, I32, P, P, P, P, P, P]),
    "lsrm_comm_unique_id": (I32, [P]),
    "lsrm_comm_init": (I32, [P, I32, I32, P]),
    "lsrm_comm_destroy": (I32, [P]),
    "lsrm_allgather_kv": (I32, [P, I32, I32, P, I64, P, P, P, P, P, I32, P]),
    "lsrm_all_to_all_v": (I32, [P, I32, I32, P, P, P, P, P]),
    "lsrm_colsum_parts": (I64, [I64]),
    "lsrm_layer_norm_bwd_f32": (I32, [P, I64, I64, I32, P, F32, P, I64, P, I64, I32, P, P, P, P]),
    "lsrm_colsum_f32": (I32, [P, I64, I64, I32, P, P, P]),
    "lsrm_gate_mix_bwd_f32": (I32, [P, I64, P, P, P, P, I64, I32, P, P, P, P]),
    "lsrm_gelu_bwd_f32": (I32, [P, P, P, I64, I32, P, P]),
    "lsrm_transpose_cast_bf16": (I32, [P, I64, I64, I64, P, I64, P]),
    "lsrm_host_threads": (I32, []),
    "lsrm_h2d_rows": (I32, [I32, P, I64, P, I64, I64, P, I64, P]),
    "lsrm_sum_slices_f32": (I32, [P, I32, I64, P, I32, P]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LsrmError(
                f"CUDA extension {LIB_PATH} is missing; run "
                "`python -m paper_2604_05182_b200.build` (there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols():
    return sorted(SIGNATURES)


def call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc:
        msg = lib().lsrm_last_error().decode(errors="replace")
        raise STATUS_CLASSES.get(rc, LsrmError)(msg)


def launch_count() -> int:
    return int(lib().lsrm_launch_count())


def reset_launch_count() -> None:
    lib().lsrm_reset_launch_count()
