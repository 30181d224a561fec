"""Storage accounting closed forms (reference analysis.py:202-245) and the
KvStream container the replay harness consumes (reference stream.py:68-124;
the KVTR file format and its GPU ingestion live in trace.py)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import UsageError


def bits_per_token(config, head_dim: int, pattern_set_size: int, token_count: int, side: str) -> float:
    """codes + amortized group params + 16-bit index + amortized 16-bit patterns (analysis.py:202-237)."""
    if side not in ("k", "v"):
        raise UsageError(f"side must be 'k' or 'v', got {side!r}")
    if head_dim < 1 or token_count < 1 or pattern_set_size < 0:
        raise UsageError("head_dim and token_count must be >= 1, pattern_set_size >= 0")
    uses = config.use_k_patterns if side == "k" else config.use_v_patterns
    codes = config.bits * head_dim
    params = 32.0 * head_dim / config.group_size if side == "k" else 32.0
    index = 16.0 if uses else 0.0
    patterns = 16.0 * head_dim * pattern_set_size / token_count
    return codes + params + index + patterns


def fp16_reference_bits_per_token(head_dim: int) -> float:
    if head_dim < 1:
        raise UsageError(f"head_dim must be >= 1, got {head_dim}")
    return 16.0 * head_dim


@dataclass
class KvStream:
    """prefill_k/v [L, H, T, d], decode_k/v [L, H, S, d] (stream.py:68-124)."""

    prefill_k: np.ndarray
    prefill_v: np.ndarray
    decode_k: np.ndarray
    decode_v: np.ndarray
    token_ids: np.ndarray | None = None
    v_cluster_ids: np.ndarray | None = None

    def __post_init__(self) -> None:
        for name in ("prefill_k", "prefill_v", "decode_k", "decode_v"):
            arr = np.asarray(getattr(self, name))
            if arr.ndim != 4:
                raise UsageError(f"{name} must be 4-D (layers, heads, tokens, dim)")
            setattr(self, name, arr)
        if self.prefill_k.shape != self.prefill_v.shape or self.decode_k.shape != self.decode_v.shape:
            raise UsageError("K and V tensors must have matching shapes")
        if self.prefill_k.shape[2] < 1:
            raise UsageError("prefill length must be >= 1")

    @property
    def num_layers(self) -> int:
        return self.prefill_k.shape[0]

    @property
    def num_heads(self) -> int:
        return self.prefill_k.shape[1]

    @property
    def prefill_len(self) -> int:
        return self.prefill_k.shape[2]

    @property
    def decode_steps(self) -> int:
        return self.decode_k.shape[2]

    @property
    def head_dim(self) -> int:
        return self.prefill_k.shape[3]

    def head_slices(self, layer: int, head: int):
        return (self.prefill_k[layer, head], self.prefill_v[layer, head],
                self.decode_k[layer, head], self.decode_v[layer, head])
