"""Reference-side binding of the B200 codec: the module a patternkv maintainer adds as
`patternkv/_b200.py` so the reference package itself calls libpkv_b200.so (INTEGRATION.md
section 2).  ctypes is the only FFI a numpy package has; every entry point of
include/pkv.h is declared here with its full prototype (restype + argtypes), status codes
map onto the reference's UsageError / DataError (errors.py:9-14).

Standalone on purpose: it depends on ctypes + numpy (+ torch only to hold device buffers),
not on this repository's Python package.  tests/test_integration_stub.py checks the
prototypes against include/pkv.h and, on a GPU, runs a prefill through it against the
package's own binding.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_LIB = os.path.join(os.path.dirname(_HERE), "paper_2510_05176_b200", "libpkv_b200.so")

PKV_OK, PKV_USAGE, PKV_DATA, PKV_CUDA = 0, 1, 2, 3
PKV_F16, PKV_F32, PKV_F64, PKV_BF16 = 1, 2, 3, 4
PKV_FLAG_DECISIONS, PKV_FLAG_STATS, PKV_FLAG_BRUTE_FORCE = 1, 2, 4


class pkv_config(C.Structure):
    """engine.py:38-83 EngineConfig, field for field."""
    _fields_ = [("bits", C.c_int32), ("pattern_count", C.c_int32), ("group_size", C.c_int32),
                ("residual_window", C.c_int32), ("alpha", C.c_double),
                ("use_k_patterns", C.c_int32), ("use_v_patterns", C.c_int32),
                ("generate_new_patterns", C.c_int32), ("use_v_gate", C.c_int32),
                ("use_k_gate", C.c_int32), ("seed", C.c_int64)]


class pkv_cache_info(C.Structure):
    _fields_ = [("n_units", C.c_int32), ("head_dim", C.c_int32), ("head_dim_padded", C.c_int32),
                ("in_dtype", C.c_int32), ("token_count", C.c_int64), ("committed_count", C.c_int64),
                ("window_len", C.c_int32), ("window_slot0", C.c_int32), ("n_blocks", C.c_int32),
                ("pattern_capacity", C.c_int32), ("token_capacity", C.c_int64), ("block_bytes", C.c_int32),
                ("n_refined", C.c_uint32), ("n_exact_div", C.c_uint32)]


i32, i64, f32, f64, vp = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_void_p
P = C.POINTER
H = vp  # opaque pkv_cache*

# include/pkv.h, declaration order: name -> (restype, argtypes)
SIGNATURES = {
    "pkv_version": (C.c_int, []),
    "pkv_last_error": (C.c_char_p, [P(i64)]),
    "pkv_z_quantile": (C.c_int, [f64, P(f64)]),
    "pkv_threshold": (C.c_int, [i32, f64, P(f64)]),
    "pkv_config_validate": (C.c_int, [P(pkv_config)]),
    "pkv_cache_create": (C.c_int, [P(pkv_config), i32, i32, i32, i64, i32, i32, P(H)]),
    "pkv_cache_destroy": (C.c_int, [H]),
    "pkv_cache_info_get": (C.c_int, [H, P(pkv_cache_info)]),
    "pkv_cache_reserve": (C.c_int, [H, i64, i32, vp]),
    "pkv_cache_reserve_mining": (C.c_int, [H, i64, vp]),
    "pkv_cache_reset": (C.c_int, [H, i32, vp]),
    "pkv_cache_check": (C.c_int, [H, i32, P(i64)]),
    "pkv_check_finite": (C.c_int, [vp, i32, i64, P(i64), vp]),
    "pkv_mine": (C.c_int, [H, i32, vp, i64, P(i64), P(f64), P(i32), vp, vp]),
    "pkv_set_patterns": (C.c_int, [H, i32, vp, i32, vp]),
    "pkv_prefill": (C.c_int, [H, vp, vp, i64, P(i64), P(i64), vp]),
    "pkv_append": (C.c_int, [H, vp, vp, vp]),
    "pkv_decode_attn": (C.c_int, [H, vp, i32, f32, vp, vp]),
    "pkv_decode_attn_partial": (C.c_int, [H, vp, i32, f32, i32, i32, i32, vp, vp, vp]),
    "pkv_cache_fork": (C.c_int, [H, P(i32), P(i32), i32, vp]),
    "pkv_cache_fork_from": (C.c_int, [H, H, P(i32), vp]),
    "pkv_dequant": (C.c_int, [H, i64, i64, vp, vp, vp]),
    "pkv_export_codes": (C.c_int, [H, i64, i64, vp, vp, vp]),
    "pkv_cache_import": (C.c_int, [H, i64, i32, P(i64), P(i32), i32, i32, i32, i32, P(i32), P(i32),
                                   vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "pkv_cache_buffer": (C.c_int, [H, C.c_char_p, P(vp), P(i64)]),
    "pkv_cache_read": (C.c_int, [H, C.c_char_p, i64, i64, vp, vp]),
    "pkv_quantize_groups": (C.c_int, [vp, vp, i32, i32, vp, vp, vp, vp]),
    "pkv_quantize_group_host": (C.c_int, [vp, i64, i32, P(f64), P(f64), vp]),
    "pkv_dequantize_group_host": (C.c_int, [vp, i64, i32, f64, f64, vp]),
    "pkv_pack_codes": (C.c_int, [vp, i64, i32, vp, vp]),
    "pkv_unpack_codes": (C.c_int, [vp, i64, i32, vp, vp]),
    "pkv_match": (C.c_int, [vp, i64, vp, i32, i32, vp, vp, vp, vp]),
    "pkv_midrange": (C.c_int, [vp, i64, i32, vp, vp]),
    "pkv_kmeans": (C.c_int, [vp, i64, i32, i32, i64, vp, vp, P(f64), P(i32), P(i32), vp]),
}


def load(path: str | None = None) -> C.CDLL:
    lib = C.CDLL(path or os.environ.get("PKV_LIB") or DEFAULT_LIB)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class B200Codec:
    """The reference engine's prefill / append / reconstruction on the GPU for a batch of heads."""

    def __init__(self, lib: C.CDLL, usage_error=ValueError, data_error=ValueError):
        self.lib, self.usage_error, self.data_error = lib, usage_error, data_error

    def check(self, rc: int) -> None:
        if rc == PKV_OK:
            return
        idx = C.c_int64(-1)
        msg = self.lib.pkv_last_error(C.byref(idx)).decode()
        raise {PKV_USAGE: self.usage_error, PKV_DATA: self.data_error}.get(rc, RuntimeError)(msg)

    def create(self, cfg, n_units: int, head_dim: int, dtype: int = PKV_F64, max_tokens: int = 4096,
               flags: int = PKV_FLAG_DECISIONS):
        s = pkv_config(cfg.bits, cfg.pattern_count, cfg.group_size, cfg.residual_window, cfg.alpha,
                       int(cfg.use_k_patterns), int(cfg.use_v_patterns), int(cfg.generate_new_patterns),
                       int(cfg.use_v_gate), int(cfg.use_k_gate), cfg.seed)
        h = H()
        self.check(self.lib.pkv_cache_create(C.byref(s), n_units, head_dim, dtype, max_tokens,
                                             cfg.pattern_count + 64, flags, C.byref(h)))
        return h

    def prefill(self, h, k_dev, v_dev, n_units: int, tokens: int, seed: int, stream=None):
        """engine.prefill for n_units heads whose K/V are device buffers [U][T][D]."""
        first = lambda s: (i64 * n_units)(*([int(np.random.default_rng(s).integers(tokens))] * n_units))  # noqa: E731
        self.check(self.lib.pkv_prefill(h, k_dev, v_dev, tokens, first(seed), first(seed + 1), stream))
        self.check(self.lib.pkv_cache_check(h, 1, None))

    def append(self, h, k_dev, v_dev, stream=None):
        self.check(self.lib.pkv_append(h, k_dev, v_dev, stream))

    def info(self, h) -> pkv_cache_info:
        i = pkv_cache_info()
        self.check(self.lib.pkv_cache_info_get(h, C.byref(i)))
        return i

    def destroy(self, h) -> None:
        self.lib.pkv_cache_destroy(h)
