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
