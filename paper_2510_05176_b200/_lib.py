"""ctypes binding of libpkv_b200.so (include/pkv.h).

The library is the product: there is no CPU fallback.  Importing the package
fails loudly when the shared library is missing (``load()``, called by the
package ``__init__``; only ``python -m paper_2510_05176_b200.build`` skips it so
a clean tree can build); every compute entry point fails with UsageError when
no CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DataError, UsageError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PKV_LIB") or os.path.join(_HERE, "libpkv_b200.so")  # PKV_LIB: A/B builds only

lib = None  # the loaded CDLL (load())

PKV_OK, PKV_USAGE, PKV_DATA, PKV_CUDA = 0, 1, 2, 3
PKV_F16, PKV_F32, PKV_F64, PKV_BF16 = 1, 2, 3, 4
PKV_FLAG_DECISIONS, PKV_FLAG_STATS = 1, 2


class PkvConfig(C.Structure):
    _fields_ = [
        ("bits", C.c_int32), ("pattern_count", C.c_int32), ("group_size", C.c_int32),
        ("residual_window", C.c_int32), ("alpha", C.c_double),
        ("use_k_patterns", C.c_int32), ("use_v_patterns", C.c_int32),
        ("generate_new_patterns", C.c_int32), ("use_v_gate", C.c_int32), ("use_k_gate", C.c_int32),
        ("seed", C.c_int64),
    ]


class PkvCacheInfo(C.Structure):
    _fields_ = [
        ("n_units", C.c_int32), ("head_dim", C.c_int32), ("head_dim_padded", C.c_int32), ("in_dtype", C.c_int32),
        ("token_count", C.c_int64), ("committed_count", C.c_int64),
        ("window_len", C.c_int32), ("window_slot0", C.c_int32), ("n_blocks", C.c_int32),
        ("pattern_capacity", C.c_int32), ("token_capacity", C.c_int64), ("block_bytes", C.c_int32),
        ("n_refined", C.c_uint32), ("n_exact_div", C.c_uint32),
    ]


_vp, _i32, _i64, _f64, _f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_float
_P = C.POINTER

# name: (restype, argtypes) -- every symbol declared in include/pkv.h
PROTOTYPES = {
    "pkv_version": (C.c_int, []),
    "pkv_last_error": (C.c_char_p, [_P(_i64)]),
    "pkv_z_quantile": (C.c_int, [_f64, _P(_f64)]),
    "pkv_threshold": (C.c_int, [_i32, _f64, _P(_f64)]),
    "pkv_config_validate": (C.c_int, [_P(PkvConfig)]),
    "pkv_cache_create": (C.c_int, [_P(PkvConfig), _i32, _i32, _i32, _i64, _i32, _i32, _P(_vp)]),
    "pkv_cache_destroy": (C.c_int, [_vp]),
    "pkv_cache_info_get": (C.c_int, [_vp, _P(PkvCacheInfo)]),
    "pkv_cache_reserve": (C.c_int, [_vp, _i64, _i32, _vp]),
    "pkv_cache_reserve_mining": (C.c_int, [_vp, _i64, _vp]),
    "pkv_cache_reset": (C.c_int, [_vp, _i32, _vp]),
    "pkv_check_finite": (C.c_int, [_vp, _i32, _i64, _P(_i64), _vp]),
    "pkv_cache_check": (C.c_int, [_vp, _i32, _P(_i64)]),
    "pkv_mine": (C.c_int, [_vp, _i32, _vp, _i64, _P(_i64), _P(_f64), _P(_i32), _vp, _vp]),
    "pkv_set_patterns": (C.c_int, [_vp, _i32, _vp, _i32, _vp]),
    "pkv_prefill": (C.c_int, [_vp, _vp, _vp, _i64, _P(_i64), _P(_i64), _vp]),
    "pkv_append": (C.c_int, [_vp, _vp, _vp, _vp]),
    "pkv_decode_attn": (C.c_int, [_vp, _vp, _i32, _f32, _vp, _vp]),
    "pkv_decode_attn_partial": (C.c_int, [_vp, _vp, _i32, _f32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "pkv_cache_fork": (C.c_int, [_vp, _P(_i32), _P(_i32), _i32, _vp]),
    "pkv_cache_fork_from": (C.c_int, [_vp, _vp, _P(_i32), _vp]),
    "pkv_dequant": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "pkv_export_codes": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "pkv_cache_import": (C.c_int, [_vp, _i64, _i32, _P(_i64), _P(_i32), _i32, _i32, _i32, _i32, _P(_i32), _P(_i32),
                                   _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pkv_cache_buffer": (C.c_int, [_vp, C.c_char_p, _P(_vp), _P(_i64)]),
    "pkv_cache_read": (C.c_int, [_vp, C.c_char_p, _i64, _i64, _vp, _vp]),
    "pkv_quantize_groups": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "pkv_quantize_group_host": (C.c_int, [_vp, _i64, _i32, _P(_f64), _P(_f64), _vp]),
    "pkv_dequantize_group_host": (C.c_int, [_vp, _i64, _i32, _f64, _f64, _vp]),
    "pkv_pack_codes": (C.c_int, [_vp, _i64, _i32, _vp, _vp]),
    "pkv_unpack_codes": (C.c_int, [_vp, _i64, _i32, _vp, _vp]),
    "pkv_match": (C.c_int, [_vp, _i64, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "pkv_midrange": (C.c_int, [_vp, _i64, _i32, _vp, _vp]),
    "pkv_kmeans": (C.c_int, [_vp, _i64, _i32, _i32, _i64, _vp, _vp, _P(_f64), _P(_i32), _P(_i32), _vp]),
}


def load():
    """Load libpkv_b200.so and bind every prototype; ImportError when it is missing."""
    global lib
    if lib is not None:
        return lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2510_05176_b200.build` "
            "(the B200 codec has no CPU fallback)"
        )
    handle = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(handle, name)  # AttributeError here = the .so does not export a declared symbol
        fn.restype = res
        fn.argtypes = args
    lib = handle
    return lib


def last_error() -> tuple[str, int]:
    idx = C.c_int64(-1)
    msg = load().pkv_last_error(C.byref(idx))
    return (msg.decode() if msg else ""), idx.value


def check(rc: int) -> None:
    """Map a status code onto the reference error taxonomy (errors.py:9-14)."""
    if rc == PKV_OK:
        return
    msg, _ = last_error()
    if rc == PKV_USAGE:
        raise UsageError(msg)
    if rc == PKV_DATA:
        raise DataError(msg)
    raise RuntimeError(f"pkv CUDA failure: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
