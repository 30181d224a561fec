"""Flattening gate (reference gate.py:23-188).

z_quantile and contraction_threshold run in the C ABI (pkv_z_quantile,
pkv_threshold: Wichura AS241 + bisection to 1e-12, bit-identical to the
reference); the K1 encode kernel applies the same `flat / raw <= threshold`
test per token on the device.  decide() is the scalar form of that test for
API callers.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from functools import lru_cache

from . import _lib
from .errors import UsageError


def z_quantile(alpha: float) -> float:
    """Upper alpha quantile of N(0, 1) (gate.py:23-30)."""
    out = C.c_double()
    _lib.call("pkv_z_quantile", C.c_double(alpha), C.byref(out))
    return out.value


@lru_cache(maxsize=None)
def contraction_threshold(head_dim: int, alpha: float) -> float:
    """Largest contraction ratio the z-test accepts at level alpha (gate.py:74-106)."""
    out = C.c_double()
    _lib.call("pkv_threshold", int(head_dim), C.c_double(alpha), C.byref(out))
    return out.value


@dataclass(frozen=True)
class GateConfig:
    alpha: float
    head_dim: int
    z: float
    threshold: float

    @classmethod
    def create(cls, head_dim: int, alpha: float = 0.05) -> "GateConfig":
        return cls(alpha=alpha, head_dim=head_dim, z=z_quantile(alpha), threshold=contraction_threshold(head_dim, alpha))


@dataclass(frozen=True)
class GateDecision:
    """Outcome of gating one vector; ratio = +inf for a constant vector (gate.py:142-156)."""

    flatten: bool
    ratio: float
    raw_range: float
    flat_range: float


def expected_error_gain(raw_range: float, flat_range: float, bits: int, dim: int) -> tuple[float, float]:
    """Mean and variance of the per-vector squared-error advantage (gate.py:159-171)."""
    if raw_range < 0 or flat_range < 0:
        raise UsageError("ranges must be non-negative")
    if dim < 1:
        raise UsageError(f"dim must be >= 1, got {dim}")
    if bits < 1:
        raise UsageError(f"bits must be >= 1, got {bits}")
    levels = (1 << bits) - 1
    d_raw = raw_range / levels
    d_flat = flat_range / levels
    return (d_raw ** 2 - d_flat ** 2) / 12.0, (d_raw ** 4 + d_flat ** 4) / (180.0 * dim)


def decide(raw_range: float, flat_range: float, config: GateConfig) -> GateDecision:
    """Flatten exactly when flat/raw <= threshold; constant vectors never flatten (gate.py:174-188)."""
    if raw_range < 0 or flat_range < 0:
        raise UsageError("ranges must be non-negative")
    if raw_range == 0.0:
        return GateDecision(flatten=False, ratio=math.inf, raw_range=0.0, flat_range=flat_range)
    ratio = flat_range / raw_range
    return GateDecision(flatten=ratio <= config.threshold, ratio=ratio, raw_range=raw_range, flat_range=flat_range)
