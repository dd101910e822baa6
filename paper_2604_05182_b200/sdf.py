"""SDF fields on the device (csrc/field.cuh): the analytic scene, the decoded
coarse volume, and opaque callables.

The reference's coarse-to-fine path scores voxel informativeness and marches
the image-token rays on the SDF DECODED from the coarse stage
(`runner.py:301-306`):

    geo_field = callable_field(lambda pts: decode_points(
        FeatureVolume(dense_grid), heads, pts)[1].astype(np.float64))

`decoded_sdf_field(dense_grid, heads)` builds that field as a `DecodedSdf`
callable, which `informative_voxel_mask` and `image_token_coords` evaluate
INSIDE their kernels (trilinear lookup, SDF head and bounding-sphere offset
per sample, with the reference's f32 rounding points and einsum reduction
order).  Any other callable field (e.g. the reference runner's own lambda
after `dropin.install`) is evaluated by calling it on the sample points the
GPU generates -- in the reference's layout -- with the reductions on the GPU.
"""

import ctypes as C

import numpy as np
import torch

from . import _dev as D
from .errors import ConfigurationError, require

S_BIAS_RADIUS = 0.45   # camera_geometry.py:21

KIND_ANALYTIC, KIND_DECODED, KIND_VALUES = 0, 1, 2


class SdfFieldDesc(C.Structure):
    """Mirror of `lsrm_sdf_field` (include/lsrm_b200.h)."""
    _fields_ = [("kind", C.c_int32), ("n_prims", C.c_int32), ("prims", C.c_void_p),
                ("grid", C.c_void_p), ("side", C.c_int32), ("d_f", C.c_int32),
                ("hidden", C.c_int32), ("pad_", C.c_int32), ("w1", C.c_void_p),
                ("b1", C.c_void_p), ("w2", C.c_void_p), ("b2", C.c_void_p),
                ("radius", C.c_double), ("values", C.c_void_p)]


def _get(node, key):
    return node.get(key) if isinstance(node, dict) else getattr(node, key, None)


class DecodedSdf:
    """s(p) of the decoded coarse volume: `decode_points(FeatureVolume(grid),
    heads, p)[1]` as float64 (`recon_pipeline.py:349-365`, dense part only).
    Callable on [N,3] points like the reference's lambda; the mask and march
    kernels evaluate it in-kernel."""

    def __init__(self, dense_grid, heads):
        g = D.dev(dense_grid, torch.float32)
        require(g.dim() == 4 and g.shape[0] == g.shape[1] == g.shape[2],
                f"decoded field: dense grid must be [S,S,S,d_f], got {tuple(g.shape)}")
        require(int(g.shape[0]) >= 2, "trilinear needs side >= 2")
        (w1, b1, a1), (w2, b2, a2) = heads.s_layers
        require(a1 == "gelu" and a2 == "identity" and np.shape(w2)[1] == 1,
                "decoded field: the SDF head must be affine-gelu-affine to one channel")
        self.grid = g.contiguous()
        self.side, self.d_f = int(g.shape[0]), int(g.shape[3])
        self.w1, self.b1, self.w2, self.b2 = (D.dev(a, torch.float32).contiguous()
                                              for a in (w1, b1, w2, b2))
        self.hidden = int(self.w1.shape[1])
        require(int(self.w1.shape[0]) == self.d_f, "decoded field: head input width != d_f")
        self.heads = heads

    def __call__(self, points):
        from .recon_pipeline import FeatureVolume, decode_points
        _, s = decode_points(FeatureVolume(self.grid), self.heads, points)
        return s.double() if D.is_device(s) else np.asarray(s, np.float64)

    def desc(self) -> SdfFieldDesc:
        return SdfFieldDesc(KIND_DECODED, 0, None, self.grid.data_ptr(), self.side, self.d_f,
                            self.hidden, 0, self.w1.data_ptr(), self.b1.data_ptr(),
                            self.w2.data_ptr(), self.b2.data_ptr(), S_BIAS_RADIUS, None)


class CallableField:
    """`SdfField("callable", fn=...)` of this package (`camera_geometry.py:186-187`)."""
    kind = "callable"

    def __init__(self, fn):
        self.fn = fn


def callable_field(fn) -> CallableField:
    return CallableField(fn)


def decoded_sdf_field(dense_grid, heads) -> CallableField:
    """The reference runner's decoded geometry field (`runner.py:301-306`)."""
    return CallableField(DecodedSdf(dense_grid, heads))


def sdf_primitives(field) -> np.ndarray:
    """Flatten an SDF union tree into [n,8] rows (kind, center, radius |
    half sizes).  Accepts the reference SdfField objects or scene-json dicts;
    union is min, which is associative, so flattening is exact."""
    rows = []

    def visit(node):
        kind = _get(node, "kind")
        if kind == "union":
            for p in _get(node, "parts"):
                visit(p)
        elif kind == "sphere":
            c = np.asarray(_get(node, "center"), np.float64)
            rows.append([0.0, c[0], c[1], c[2], float(_get(node, "radius")), 0.0, 0.0, 0.0])
        elif kind == "box":
            c = np.asarray(_get(node, "center"), np.float64)
            h = np.asarray(_get(node, "half_sizes"), np.float64)
            rows.append([1.0, c[0], c[1], c[2], h[0], h[1], h[2], 0.0])
        elif kind == "callable":
            raise ConfigurationError("a callable field cannot be part of an analytic union")
        else:
            raise ConfigurationError(f"unknown SDF kind {kind!r}")
    visit(field)
    return np.asarray(rows, np.float64)


class DeviceField:
    """A field as the kernels see it: `desc` (ctypes struct) for analytic and
    decoded fields; `fn` (an opaque callable) otherwise."""

    def __init__(self, field):
        kind = _get(field, "kind")
        self.fn = None
        self._refs = []
        if kind == "callable":
            fn = _get(field, "fn")
            require(callable(fn), "callable field without a callable fn")
            if isinstance(fn, DecodedSdf):
                self.desc = fn.desc()
                self._refs.append(fn)
            else:
                self.desc = None
                self.fn = fn
        else:
            prims = D.dev(sdf_primitives(field))
            self._refs.append(prims)
            self.desc = SdfFieldDesc(KIND_ANALYTIC, int(prims.shape[0]), prims.data_ptr(), None,
                                     0, 0, 0, 0, None, None, None, None, 0.0, None)

    @property
    def opaque(self) -> bool:
        return self.fn is not None

    def values_desc(self, values: torch.Tensor) -> SdfFieldDesc:
        self._refs.append(values)
        return SdfFieldDesc(KIND_VALUES, 0, None, None, 0, 0, 0, 0, None, None, None, None, 0.0,
                            values.data_ptr())

    def eval_host(self, pts_dev: torch.Tensor) -> torch.Tensor:
        """The opaque callable on [N,3] device points -> [N] f64 device values
        (the callable sees NumPy f64 points, as the reference's eval_sdf_many
        hands them over)."""
        s = self.fn(D.host(pts_dev))
        s = np.asarray(D.host(s) if D.is_device(s) else s, np.float64).reshape(-1)
        require(s.size == int(pts_dev.shape[0]), "callable field returned the wrong count")
        return D.dev(s, torch.float64)


def ptr(desc) -> C.c_void_p:
    return C.cast(C.pointer(desc), C.c_void_p)
