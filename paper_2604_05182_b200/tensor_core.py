"""Head geometry and dtype conventions (`lsrm/tensor_core.py:1-71`).

Storage is float32 on the reference API surface; the device fast path stores
bf16 with fp32 accumulation (see DESIGN.md for the stated tolerances).
"""

from dataclasses import dataclass

import numpy as np

from .errors import require

DTYPE = np.float32
ACC = np.float64


@dataclass(frozen=True)
class AttentionParams:
    """GQA layout; query head g reads kv head g // (n_q_heads // n_kv_heads).
    hardware_faithful enforces (n_q_heads / n_kv_heads) % 16 == 0
    (`tensor_core.py:39-71`)."""
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    hardware_faithful: bool = False

    def __post_init__(self):
        require(self.n_q_heads >= 1 and self.n_kv_heads >= 1,
                "head counts must be positive")
        require(self.head_dim >= 1, "head_dim must be positive")
        require(self.n_q_heads % self.n_kv_heads == 0,
                f"n_q_heads={self.n_q_heads} not divisible by "
                f"n_kv_heads={self.n_kv_heads}")
        if self.hardware_faithful:
            ratio = self.n_q_heads // self.n_kv_heads
            require(ratio % 16 == 0,
                    f"hardware-faithful mode needs (n_q_heads/n_kv_heads) % 16"
                    f" == 0, got ratio {ratio}")

    @property
    def model_dim(self) -> int:
        return self.n_q_heads * self.head_dim

    @property
    def group_size(self) -> int:
        return self.n_q_heads // self.n_kv_heads


# ---------------------------------------------------------------------------
# golden-vector files (tensor_core.py:255-311)
#
# little-endian: magic "LSRMGV1\0" | u32 tensor count |
#   per tensor: u32 rank | u32 dims[rank] | f32 payload (row-major)

GOLDEN_MAGIC = b"LSRMGV1\x00"
GOLDEN_MAX_RANK = 16


def write_goldens(path, tensors) -> None:
    """Write f32 tensors (NumPy or CUDA) in the LSRMGV1 layout."""
    import struct
    with open(path, "wb") as fh:
        fh.write(GOLDEN_MAGIC)
        fh.write(struct.pack("<I", len(tensors)))
        for t in tensors:
            if hasattr(t, "detach"):
                t = t.detach().cpu().numpy()
            arr = np.ascontiguousarray(np.asarray(t, dtype=DTYPE))
            fh.write(struct.pack("<I", arr.ndim))
            fh.write(struct.pack(f"<{arr.ndim}I", *arr.shape))
            fh.write(arr.astype("<f4").tobytes())


def read_goldens(path) -> list:
    """Parse an LSRMGV1 file; malformed input raises GoldenFormatError with
    the byte offset of the first bad field."""
    import struct
    from .errors import GoldenFormatError
    blob = open(path, "rb").read()
    size = len(blob)

    def take(pos, n, what):
        if pos + n > size:
            raise GoldenFormatError(f"truncated golden file: {what} needs {n} bytes, file "
                                    f"ends at {size}", byte_offset=pos)
        return blob[pos:pos + n]

    if take(0, 8, "magic") != GOLDEN_MAGIC:
        raise GoldenFormatError(f"bad magic {blob[:8]!r}, expected {GOLDEN_MAGIC!r}",
                                byte_offset=0)
    (count,) = struct.unpack("<I", take(8, 4, "tensor count"))
    pos, out = 12, []
    for ti in range(count):
        (rank,) = struct.unpack("<I", take(pos, 4, f"tensor {ti} rank"))
        if rank > GOLDEN_MAX_RANK:
            raise GoldenFormatError(f"tensor {ti} rank {rank} exceeds limit {GOLDEN_MAX_RANK}",
                                    byte_offset=pos)
        pos += 4
        dims = struct.unpack(f"<{rank}I", take(pos, 4 * rank, f"tensor {ti} dims"))
        pos += 4 * rank
        n = int(np.prod(dims, dtype=np.int64)) if rank else 1
        data = take(pos, 4 * n, f"tensor {ti} payload")
        out.append(np.frombuffer(data, dtype="<f4").reshape(dims).astype(DTYPE))
        pos += 4 * n
    if pos != size:
        raise GoldenFormatError(f"{size - pos} trailing bytes after last tensor",
                                byte_offset=pos)
    return out
