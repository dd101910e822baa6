"""Tagged counter-based random streams, draw-for-draw equal to the
reference's (`lsrm/rng.py:16-41`), so synthetic weights and inputs built
here are the reference's bit for bit.

A stream is NumPy's Philox keyed by the integer seed, with counter word 0
set to the first 8 bytes (little-endian) of sha256 over the "/"-joined tag
path; the other counter words are 0.
"""

import hashlib

import numpy as np

_KEY_MASK = (1 << 64) - 1


def tag_counter(*tags) -> int:
    path = "/".join(map(str, tags)).encode("utf-8")
    return int.from_bytes(hashlib.sha256(path).digest()[:8], "little")


def stream(seed: int, *tags) -> np.random.Generator:
    if not isinstance(seed, (int, np.integer)):
        raise TypeError(f"stream seed has to be an integer (got {type(seed).__name__})")
    philox = np.random.Philox(key=int(seed) & _KEY_MASK, counter=(tag_counter(*tags), 0, 0, 0))
    return np.random.Generator(philox)


def normal_f32(seed: int, shape, scale: float = 1.0, *tags) -> np.ndarray:
    """N(0, scale^2) draws of `shape`, stored as float32."""
    draws = stream(seed, *tags).standard_normal(shape)
    return (draws * scale).astype(np.float32)
