"""B200-native PatternKV codec (arXiv 2510.05176): pattern-aligned residual
KV-cache quantization with hand-written sm_100a kernels behind a C ABI.

Production API: ``PatternKVCache`` (batched units on one GPU).
Drop-in API: the reference package's names (``prefill``,
``append_decode_token``, ``quantize_group``, ...) re-exported below with the
reference's signatures, argument meaning and error behaviour.
"""

from .errors import DataError, UsageError
from . import _lib  # noqa: F401  (fails loudly when libpkv_b200.so is missing)
from .cache import RAW_MARKER, PatternKVCache, first_seed_index

__version__ = "0.1.0"

__all__ = ["DataError", "UsageError", "PatternKVCache", "RAW_MARKER", "first_seed_index"]
