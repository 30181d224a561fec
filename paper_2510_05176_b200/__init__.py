"""B200-native PatternKV codec (arXiv 2510.05176): pattern-aligned residual
KV-cache quantization with hand-written sm_100a kernels behind a C ABI
(include/pkv.h, libpkv_b200.so).

Production API: ``PatternKVCache`` -- U independent (batch, layer, kv-head)
units on one GPU: prefill (mine + encode), append-and-refresh, decode
attention over the compressed cache, exact dequant.
Drop-in API: the reference package's hot-path names (pkg/src/patternkv/
__init__.py:10-94) with the reference's signatures, argument meaning and
error behaviour, executed on the GPU.
"""

import sys as _sys

from . import _lib

# fail loudly when libpkv_b200.so is missing -- except while `python -m
# paper_2510_05176_b200.build` is building it from a clean tree
if not any(a.endswith("paper_2510_05176_b200.build") for a in getattr(_sys, "orig_argv", ())):
    _lib.load()
from .analysis import KvStream, bits_per_token, fp16_reference_bits_per_token
from .cache import PatternKVCache, first_seed_index
from .config import EngineConfig
from .engine import (
    RAW_MARKER,
    CacheMetrics,
    CommittedKBlock,
    CommittedVToken,
    HeadCacheState,
    HeadReport,
    accounted_bits_per_token,
    append_decode_token,
    committed_matrices,
    prefill,
    reconstruct_token,
    replay_head,
    run_scheme_comparison,
)
from .errors import DataError, UsageError
from .gate import GateConfig, GateDecision, contraction_threshold, decide, expected_error_gain, z_quantile
from .patterns import (
    PatternMatch,
    PatternSet,
    lloyd_kmeans,
    match_many,
    match_pattern,
    midrange_center,
    mine_patterns,
    minmax_distance,
    reconstruct_vector,
)
from .quant import QuantizedGroup, QuantParams, dequantize_group, pack_codes, quantize_group, unpack_codes
from .trace import TraceHeader, ingest_trace, load_trace_device, read_trace, read_trace_header, write_trace
from . import verify
from .snapshot import (
    SNAPSHOT_MAGIC,
    SNAPSHOT_VERSION,
    cache_snapshot_bytes,
    load_snapshot,
    restore_cache,
    save_cache_snapshot,
    save_snapshot,
)

__version__ = "0.1.0"

__all__ = [
    "PatternKVCache", "first_seed_index", "KvStream", "bits_per_token", "fp16_reference_bits_per_token",
    "EngineConfig", "RAW_MARKER", "CacheMetrics", "CommittedKBlock", "CommittedVToken", "HeadCacheState",
    "HeadReport", "accounted_bits_per_token", "append_decode_token", "committed_matrices", "prefill",
    "reconstruct_token", "replay_head", "run_scheme_comparison", "DataError", "UsageError", "GateConfig",
    "GateDecision", "contraction_threshold", "decide", "expected_error_gain", "z_quantile", "PatternMatch",
    "PatternSet", "lloyd_kmeans", "match_many", "match_pattern", "midrange_center", "mine_patterns",
    "minmax_distance", "reconstruct_vector", "QuantizedGroup", "QuantParams", "dequantize_group", "pack_codes",
    "quantize_group", "unpack_codes", "SNAPSHOT_MAGIC", "SNAPSHOT_VERSION", "save_snapshot", "load_snapshot",
    "save_cache_snapshot", "cache_snapshot_bytes", "restore_cache", "TraceHeader", "write_trace", "read_trace",
    "read_trace_header", "load_trace_device", "ingest_trace", "verify",
]
