"""Group quantizer API (reference quant.py:18-179) on the B200 kernels.

quantize_group -> pkv_quantize_groups (one warp per group, exact fp64
semantics: zero = min, scale = (max - min)/(2^b - 1), code =
clip(floor((v - lo)/scale + 0.5), 0, qmax)); pack_codes / unpack_codes ->
pkv_pack_codes / pkv_unpack_codes (little-endian, first code in the low bits).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cache import _ptr, _stream, require_cuda
from .errors import DataError, UsageError

SUPPORTED_BITS = (2, 4, 8)
PER_CHANNEL = "per-channel"
PER_TOKEN = "per-token"
_LAYOUTS = (PER_CHANNEL, PER_TOKEN)


@dataclass(frozen=True)
class QuantParams:
    """Affine parameters of one group (quant.py:28-40)."""

    scale: float
    zero_point: float
    bits: int


@dataclass(frozen=True)
class QuantizedGroup:
    """Parameters plus packed codes (quant.py:43-57)."""

    params: QuantParams
    codes: bytes
    length: int
    layout: str


def _check_bits(bits: int) -> None:
    if bits not in SUPPORTED_BITS:
        raise UsageError(f"unsupported bit width {bits}; expected one of {SUPPORTED_BITS}")


def _check_layout(layout: str) -> None:
    if layout not in _LAYOUTS:
        raise UsageError(f"unknown layout {layout!r}; expected one of {_LAYOUTS}")


def quantize_groups(values: list[np.ndarray], bits: int) -> list[tuple[float, float, np.ndarray]]:
    """Batched quantize_group: one launch for many groups -> [(scale, zero, codes)]."""
    _check_bits(bits)
    require_cuda()
    lens = [len(v) for v in values]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    vals = torch.from_numpy(np.concatenate([np.asarray(v, np.float64) for v in values])).cuda()
    offs_d = torch.from_numpy(offs).cuda()
    n = len(values)
    scale = torch.empty(n, dtype=torch.float64, device="cuda")
    zero = torch.empty_like(scale)
    codes = torch.empty(int(offs[-1]), dtype=torch.uint8, device="cuda")
    _lib.call("pkv_quantize_groups", _ptr(vals), _ptr(offs_d), n, bits, _ptr(scale), _ptr(zero), _ptr(codes),
              _stream())
    s, z, c = scale.cpu().numpy(), zero.cpu().numpy(), codes.cpu().numpy()
    return [(float(s[i]), float(z[i]), c[offs[i]:offs[i + 1]]) for i in range(n)]


def quantize_group(values: np.ndarray, bits: int, layout: str = PER_TOKEN) -> QuantizedGroup:
    """Encode one group of finite reals as n-bit codes (quant.py:70-111)."""
    _check_bits(bits)
    _check_layout(layout)
    vals = np.asarray(values, dtype=np.float64).ravel()
    if vals.size == 0:
        raise UsageError("cannot quantize an empty group")
    finite = np.isfinite(vals)
    if not finite.all():
        idx = int(np.flatnonzero(~finite)[0])
        raise DataError(f"non-finite value at index {idx}: {vals[idx]}")
    require_cuda()
    vals = np.ascontiguousarray(vals)
    packed = np.empty((vals.size * bits + 7) // 8, dtype=np.uint8)
    scale, zero = C.c_double(), C.c_double()
    _lib.call("pkv_quantize_group_host", vals.ctypes.data_as(C.c_void_p), vals.size, bits, C.byref(scale),
              C.byref(zero), packed.ctypes.data_as(C.c_void_p))
    return QuantizedGroup(params=QuantParams(scale=scale.value, zero_point=zero.value, bits=bits),
                          codes=packed.tobytes(), length=vals.size, layout=layout)


def dequantize_group(group: QuantizedGroup) -> np.ndarray:
    """scale * code + zero_point in float64 (quant.py:114-117), on the GPU."""
    bits, n = group.params.bits, group.length
    _check_bits(bits)
    expected = (n * bits + 7) // 8
    if len(group.codes) != expected:
        raise DataError(f"packed payload is {len(group.codes)} bytes, expected {expected} for {n} codes of {bits} bits")
    out = np.empty(n, dtype=np.float64)
    if n:
        require_cuda()
        src = np.frombuffer(bytes(group.codes), dtype=np.uint8)
        _lib.call("pkv_dequantize_group_host", src.ctypes.data_as(C.c_void_p), n, bits, C.c_double(group.params.scale),
                  C.c_double(group.params.zero_point), out.ctypes.data_as(C.c_void_p))
    return out


def pack_codes(codes: np.ndarray, bits: int) -> bytes:
    """Pack n-bit codes, first code in the lowest-order bits (quant.py:120-146)."""
    _check_bits(bits)
    arr = np.asarray(codes, dtype=np.int64).ravel()
    if arr.size == 0:
        return b""
    qmax = (1 << bits) - 1
    if arr.min() < 0 or arr.max() > qmax:
        bad = int(np.flatnonzero((arr < 0) | (arr > qmax))[0])
        raise UsageError(f"code {arr[bad]} at index {bad} does not fit in {bits} bits")
    require_cuda()
    src = torch.from_numpy(arr.astype(np.uint8)).cuda()
    out = torch.empty((arr.size * bits + 7) // 8, dtype=torch.uint8, device="cuda")
    _lib.call("pkv_pack_codes", _ptr(src), arr.size, bits, _ptr(out), _stream())
    return out.cpu().numpy().tobytes()


def unpack_codes(data: bytes, length: int, bits: int) -> np.ndarray:
    """Invert pack_codes (quant.py:149-179)."""
    _check_bits(bits)
    if length < 0:
        raise UsageError(f"negative code count {length}")
    expected = (length * bits + 7) // 8
    if len(data) != expected:
        raise DataError(
            f"packed payload is {len(data)} bytes, expected {expected} for {length} codes of {bits} bits"
        )
    if length == 0:
        return np.zeros(0, dtype=np.uint8)
    require_cuda()
    src = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    out = torch.empty(length, dtype=torch.uint8, device="cuda")
    _lib.call("pkv_unpack_codes", _ptr(src), length, bits, _ptr(out), _stream())
    return out.cpu().numpy()
