"""Install this package as the reference `lsrm` package's hot path.

The reference has no plugin registry. Its callers import hot-path functions
by name at import time (`lsrm/recon_pipeline.py:29-30`,
`lsrm/seq_parallel.py:24-32`, `lsrm/runner.py:25-45`, `lsrm/cli.py:17`), so
patching only the defining module is not enough. `install()`
rebinds every hot-path name in EVERY loaded `lsrm.*` module that holds the
reference's object, and returns the list of (module, name) pairs it changed.
`uninstall()` restores them.

    import lsrm, paper_2604_05182_b200.dropin as d
    patched = d.install(lsrm)     # lsrm.run_scene(...) now routes/attends on the GPU
    d.install(lsrm, precision="bf16")   # + NSA uses / blocks / stage on the bf16 engines

precision="fp32" (default) keeps the reference's float contract (fp32 CUDA
kernels, <=1e-5); "bf16" sends `nsa_cross_attention`, `sparse_block_forward`
and `sparse_stage_forward` to the tcgen05 engines (fastpath.py; rel-L2 <=1e-2).
"""

import importlib
import pkgutil

# reference defining module -> names replaced (SURVEY.md §8b signature list)
HOT_PATH = {
    "nsa_attention": ("nsa_cross_attention", "cmp_attention", "sel_attention", "win_attention",
                      "build_gather_table", "score_topk_blocks", "nsa_gates",
                      "combine_nsa_branches"),
    "block_partition": ("partition", "compress_block_kv", "res_block"),
    "block_routing": ("build_routing_plan", "route_to_volume_blocks", "route_to_image_blocks",
                      "_route_points_to_volume", "_route_points_to_image",
                      "image_token_coords"),
    "tokenizer": ("informative_voxel_mask", "foreground_patch_mask", "upsample_select_tokens"),
    "seq_parallel": ("shard_blocks", "all_to_all", "all_gather_kv", "naive_contiguous_shards",
                     "parallel_sparse_stage"),
    "recon_pipeline": ("sparse_block_forward", "sparse_stage_forward", "build_sparse_context",
                       "ffn_forward",
                       "mha_forward", "dense_block_forward", "dense_stage_forward",
                       "decode_feature_volume", "build_sparse_features", "query_field",
                       "decode_points"),
    "camera_geometry": ("pluecker_rays", "silhouette_alpha"),
    "tensor_core": ("write_goldens", "read_goldens"),
}

_saved = []


def _ours(module: str, name: str):
    mod = importlib.import_module(f"{__package__}.{module}")
    return getattr(mod, name, None)


def install(lsrm_pkg, precision: str = "fp32") -> list:
    """Patch the hot-path names of an imported reference `lsrm` package."""
    from . import fastpath
    fastpath.set_precision(precision)
    mods = {}
    for info in pkgutil.iter_modules(lsrm_pkg.__path__):
        try:
            mods[info.name] = importlib.import_module(f"{lsrm_pkg.__name__}.{info.name}")
        except Exception:   # optional reference modules (e.g. CLI deps) may not import
            continue
    patched = []
    for defining, names in HOT_PATH.items():
        if defining not in mods:
            continue
        for name in names:
            ref_obj = getattr(mods[defining], name, None)
            new_obj = _ours(defining, name)
            if ref_obj is None or new_obj is None:
                continue
            for mname, mod in list(mods.items()) + [("", lsrm_pkg)]:
                if getattr(mod, name, None) is ref_obj:
                    _saved.append((mod, name, ref_obj))
                    setattr(mod, name, new_obj)
                    patched.append((mod.__name__, name))
    return patched


def uninstall() -> None:
    from . import fastpath
    fastpath.set_precision("fp32")
    while _saved:
        mod, name, obj = _saved.pop()
        setattr(mod, name, obj)
