"""Deterministic tagged Philox streams, identical to `lsrm/rng.py:16-41`, so
weights and synthetic inputs built here equal the reference's bit for bit."""

import hashlib

import numpy as np


def tag_counter(*tags) -> int:
    h = hashlib.sha256("/".join(str(t) for t in tags).encode("utf-8")).digest()
    return int.from_bytes(h[:8], "little")


def stream(seed: int, *tags) -> np.random.Generator:
    if not isinstance(seed, (int, np.integer)):
        raise TypeError(f"seed must be an int, got {type(seed).__name__}")
    return np.random.Generator(np.random.Philox(
        key=int(seed) & 0xFFFFFFFFFFFFFFFF, counter=[tag_counter(*tags), 0, 0, 0]))


def normal_f32(seed: int, shape, scale: float = 1.0, *tags) -> np.ndarray:
    return (stream(seed, *tags).standard_normal(shape) * scale).astype(np.float32)
