"""Camera rays and silhouettes on the GPU (drop-in for the hot-path producers
in `lsrm/camera_geometry.py`): the Plücker rays of the image tokens and the
per-pixel silhouettes that feed `foreground_patch_mask`. f64 arithmetic in
NumPy's operation order (csrc/camera.cu)."""

import numpy as np
import torch

from . import _dev as D
from ._native import call
from .block_routing import pack_cameras
from .errors import require
from .sdf import callable_field, decoded_sdf_field, sdf_primitives  # noqa: F401


def _image_sizes(cameras):
    out = []
    for cam in cameras:
        size = getattr(cam, "image_size", None)
        if size is None and isinstance(cam, (tuple, list)) and len(cam) > 3:
            size = cam[3]
        require(size is not None, "camera needs an image size")
        out.append((int(size[0]), int(size[1])))
    return out


def pluecker_rays(camera, grid) -> np.ndarray:
    """[h, w, 6] float32 rows (d, o x d) through the centers of a (w, h) grid
    laid over the full image (`camera_geometry.py:91-107`)."""
    gw, gh = int(grid[0]), int(grid[1])
    require(gw >= 1 and gh >= 1, "ray grid must be at least 1x1")
    cams = D.dev(pack_cameras([camera]))
    wh = D.dev(np.asarray(_image_sizes([camera]), np.int32))
    out = D.empty((gh, gw, 6), torch.float32)
    call("lsrm_pluecker_rays", cams.data_ptr(), wh.data_ptr(), 1, gw, gh, out.data_ptr(),
         D.stream())
    return D.host(out)


def silhouette_alpha(field, camera) -> np.ndarray:
    """[H, W] float32: 1 where the pixel ray hits the analytic field
    (`camera_geometry.py:344-350`)."""
    return silhouettes(field, [camera])[0]


def silhouettes(field, cameras, as_device: bool = False):
    """Silhouettes of all views in one launch: [V, H, W] float32 (views of
    different sizes are zero-padded to the largest)."""
    sizes = _image_sizes(cameras)
    mw, mh = max(s[0] for s in sizes), max(s[1] for s in sizes)
    cams = D.dev(pack_cameras(cameras))
    wh = D.dev(np.asarray(sizes, np.int32))
    prims = D.dev(sdf_primitives(field))
    out = D.zeros((len(cameras), mh, mw), torch.float32)
    call("lsrm_silhouette_alpha", cams.data_ptr(), wh.data_ptr(), len(cameras), mw, mh,
         prims.data_ptr(), int(prims.shape[0]), out.data_ptr(), D.stream())
    return out if as_device else D.host(out)
