"""Counter-based Philox streams keyed by a tag path (TEST INFRASTRUCTURE ONLY).

Restates `lsrm/rng.py:16-41`: the tag tuple joined with "/" is hashed with
sha256; the first 8 digest bytes (little-endian) become Philox counter word 0
and the integer seed becomes the Philox key.
"""

import hashlib

import numpy as np


def tag_counter(*tags) -> int:
    digest = hashlib.sha256("/".join(map(str, tags)).encode()).digest()
    return int.from_bytes(digest[:8], "little")


def stream(seed: int, *tags) -> np.random.Generator:
    bits = np.random.Philox(key=int(seed) & (2 ** 64 - 1),
                            counter=[tag_counter(*tags), 0, 0, 0])
    return np.random.Generator(bits)


def normal_f32(seed: int, shape, scale: float = 1.0, *tags) -> np.ndarray:
    return (stream(seed, *tags).standard_normal(shape) * scale).astype(
        np.float32)
