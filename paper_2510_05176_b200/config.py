"""EngineConfig: the reference's static scheme knobs (engine.py:38-83), field
for field, validated by the C ABI (pkv_config_validate)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

from . import _lib


@dataclass(frozen=True)
class EngineConfig:
    """Static knobs of one cache scheme (engine.py:38-60).

    use_k_patterns / use_v_patterns control residualization per side; with
    both off the engine degrades to plain per-channel K and per-token V
    quantization. generate_new_patterns adds one midrange pattern per side on
    every decode flush (only for sides with patterns enabled). use_v_gate runs
    the flattening test per value vector; use_k_gate extends it to keys.
    """

    bits: int = 2
    pattern_count: int = 32
    group_size: int = 128
    residual_window: int = 128
    alpha: float = 0.05
    use_k_patterns: bool = True
    use_v_patterns: bool = True
    generate_new_patterns: bool = True
    use_v_gate: bool = True
    use_k_gate: bool = False
    seed: int = 0

    def __post_init__(self) -> None:
        from .cache import make_config_struct

        s = make_config_struct(self)
        _lib.check(_lib.load().pkv_config_validate(C.byref(s)))

    def raw_variant(self) -> "EngineConfig":
        """Same geometry with every pattern mechanism disabled (engine.py:77-79)."""
        return replace(self, use_k_patterns=False, use_v_patterns=False, generate_new_patterns=False)

    @property
    def is_raw(self) -> bool:
        return not (self.use_k_patterns or self.use_v_patterns or self.generate_new_patterns)
