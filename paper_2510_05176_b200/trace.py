"""KVTR trace interchange (reference stream.py:1-236) and its GPU ingestion.

Format (little-endian, packed; stream.py:3-24):

    magic b"KVTR", version u32 = 1, num_layers u32, num_heads u32 (KV heads per
    layer), head_dim u32, dtype u8 (1 float16, 2 float32), prefill u32 (>= 1),
    steps u32; then the body in that element dtype, row-major:
        for each layer: K[heads, prefill, dim], V[heads, prefill, dim]
        for each step: for each layer: K[heads, 1, dim], V[heads, 1, dim]

write_trace / read_trace / read_trace_header keep the reference's names, host
fp64 results and DataError messages (byte offsets, the first non-finite
element's layer/head/token/dim).  The B200 path, load_trace_device, never
widens on the host: the raw payload goes to HBM in one pinned copy and is
rearranged there into the cache's unit-major layout (unit u = layer * heads +
head): prefill K/V [U][prefill][dim] and decode K/V [steps][U][dim], in the
trace's own dtype (fp16 traces feed the fp16 encoder directly); finiteness is
checked on the device (pkv_check_finite) and reported with the reference's
message.  ingest_trace runs prefill + every decode step through a
PatternKVCache.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np

from .analysis import KvStream
from .errors import DataError, UsageError

TRACE_MAGIC = b"KVTR"
TRACE_VERSION = 1
_HEADER_FMT = "<4sIIIIBII"
HEADER_SIZE = struct.calcsize(_HEADER_FMT)
DTYPE_F16 = 1
DTYPE_F32 = 2
_DTYPE_NP = {DTYPE_F16: np.dtype("<f2"), DTYPE_F32: np.dtype("<f4")}
_DTYPE_NAMES = {DTYPE_F16: "float16", DTYPE_F32: "float32"}


@dataclass(frozen=True)
class TraceHeader:
    num_layers: int
    num_heads: int
    head_dim: int
    dtype_code: int
    prefill_len: int
    decode_steps: int

    @property
    def dtype_name(self) -> str:
        return _DTYPE_NAMES.get(self.dtype_code, f"unknown({self.dtype_code})")

    @property
    def body_bytes(self) -> int:
        per = _DTYPE_NP[self.dtype_code].itemsize
        return 2 * self.num_layers * self.num_heads * self.head_dim * (self.prefill_len + self.decode_steps) * per


def write_trace(path: str, stream: KvStream, dtype_code: int = DTYPE_F32) -> None:
    """Serialize a stream to the binary trace format (stream.py:126-150)."""
    if dtype_code not in _DTYPE_NP:
        raise UsageError(f"unknown trace dtype code {dtype_code}")
    dt = _DTYPE_NP[dtype_code]
    L, H, S = stream.num_layers, stream.num_heads, stream.decode_steps
    header = struct.pack(_HEADER_FMT, TRACE_MAGIC, TRACE_VERSION, L, H, stream.head_dim, dtype_code,
                         stream.prefill_len, S)
    # prefill: [L][2][H][T][d]; decode: [S][L][2][H][d] -- one array per phase, one write each
    pre = np.stack([np.asarray(stream.prefill_k), np.asarray(stream.prefill_v)], axis=1).astype(dt)
    dec = np.stack([np.asarray(stream.decode_k), np.asarray(stream.decode_v)], axis=1)  # [L][2][H][S][d]
    dec = np.ascontiguousarray(np.transpose(dec, (3, 0, 1, 2, 4))).astype(dt)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(np.ascontiguousarray(pre).tobytes())
        fh.write(dec.tobytes())


def _parse_header(raw: bytes, file_size: int) -> TraceHeader:
    if len(raw) < HEADER_SIZE:
        raise DataError(f"trace truncated inside the header: file ends at byte offset {file_size}, "
                        f"header needs {HEADER_SIZE}")
    magic, version, layers, heads, dim, dtype_code, prefill, steps = struct.unpack(_HEADER_FMT, raw[:HEADER_SIZE])
    if magic != TRACE_MAGIC:
        raise DataError(f"bad magic {magic!r} at byte offset 0, expected {TRACE_MAGIC!r}")
    if version != TRACE_VERSION:
        raise DataError(f"unsupported trace version {version} at byte offset 4, expected {TRACE_VERSION}")
    if layers < 1:
        raise DataError("num_layers is 0 at byte offset 8")
    if heads < 1:
        raise DataError("num_heads is 0 at byte offset 12")
    if dim < 1:
        raise DataError("head_dim is 0 at byte offset 16")
    if dtype_code not in _DTYPE_NP:
        raise DataError(f"unknown dtype code {dtype_code} at byte offset 20")
    if prefill < 1:
        raise DataError("prefill length is 0 at byte offset 21")
    return TraceHeader(layers, heads, dim, dtype_code, prefill, steps)


def read_trace_header(path: str) -> TraceHeader:
    """Parse and validate only the fixed-size header (stream.py:153-157)."""
    with open(path, "rb") as fh:
        raw = fh.read(HEADER_SIZE)
    return _parse_header(raw, len(raw))


def _body(path: str):
    """(header, body as a read-only uint8 memmap) with the body length checked."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        header = _parse_header(fh.read(HEADER_SIZE), size)
    got, expected = size - HEADER_SIZE, header.body_bytes
    if got != expected:
        raise DataError(f"trace body is {got} bytes, expected {expected}; "
                        f"file diverges from the format at byte offset {HEADER_SIZE + min(got, expected)}")
    body = np.memmap(path, dtype=np.uint8, mode="r", offset=HEADER_SIZE, shape=(expected,)) if expected else \
        np.zeros(0, np.uint8)
    return header, body


def _first_nonfinite(name: str, arr4: np.ndarray) -> None:
    if not np.isfinite(arr4).all():
        loc = np.argwhere(~np.isfinite(arr4))[0]
        raise DataError(f"non-finite {name} element at layer {loc[0]}, head {loc[1]}, token {loc[2]}, dim {loc[3]}")


def read_trace(path: str) -> KvStream:
    """Load a trace file into a float64 KvStream (stream.py:188-236)."""
    h, body = _body(path)
    flat = np.frombuffer(body, dtype=_DTYPE_NP[h.dtype_code])
    L, H, T, S, d = h.num_layers, h.num_heads, h.prefill_len, h.decode_steps, h.head_dim
    npre = L * 2 * H * T * d
    pre = flat[:npre].reshape(L, 2, H, T, d).astype(np.float64)
    dec = flat[npre:].reshape(S, L, 2, H, d).astype(np.float64)
    pk, pv = pre[:, 0], pre[:, 1]
    dk = np.ascontiguousarray(np.transpose(dec[:, :, 0], (1, 2, 0, 3)))  # [L][H][S][d]
    dv = np.ascontiguousarray(np.transpose(dec[:, :, 1], (1, 2, 0, 3)))
    for name, arr in (("prefill K", pk), ("prefill V", pv), ("decode K", dk), ("decode V", dv)):
        _first_nonfinite(name, arr)
    return KvStream(prefill_k=np.ascontiguousarray(pk), prefill_v=np.ascontiguousarray(pv), decode_k=dk, decode_v=dv)


# ---- GPU ingestion ---------------------------------------------------------------------------
@dataclass
class DeviceTrace:
    """A trace resident in HBM in the cache's unit-major layout (unit u = layer * heads + head)."""

    header: TraceHeader
    prefill_k: "object"   # torch [U][T][d]
    prefill_v: "object"
    decode_k: "object"    # torch [S][U][d]
    decode_v: "object"

    @property
    def n_units(self) -> int:
        return self.header.num_layers * self.header.num_heads


def load_trace_device(path: str, device: str = "cuda") -> DeviceTrace:
    """One pinned H2D copy of the raw payload, rearranged on the device."""
    import torch

    from . import _lib
    from .cache import _ptr, _stream

    h, body = _body(path)
    tdt = torch.float16 if h.dtype_code == DTYPE_F16 else torch.float32
    L, H, T, S, d = h.num_layers, h.num_heads, h.prefill_len, h.decode_steps, h.head_dim
    host = torch.empty(len(body), dtype=torch.uint8, pin_memory=True)
    host.numpy()[:] = body
    raw = host.to(device, non_blocking=True).view(tdt)
    # device finiteness check in the reference's report order (prefill K, prefill V, decode K, decode V)
    import ctypes as C
    bad = C.c_int64(-1)
    dcode = _lib.PKV_F16 if h.dtype_code == DTYPE_F16 else _lib.PKV_F32
    _lib.call("pkv_check_finite", _ptr(raw), dcode, raw.numel(), C.byref(bad), _stream())
    npre = L * 2 * H * T * d
    pre = raw[:npre].view(L, 2, H, T, d)
    dec = raw[npre:].view(S, L, 2, H, d)
    if bad.value >= 0:  # locate the first non-finite element as read_trace reports it
        def first(t):
            idx = (~torch.isfinite(t)).nonzero()
            return None if idx.numel() == 0 else idx[0].tolist()
        for name, t in (("prefill K", pre[:, 0]), ("prefill V", pre[:, 1]),
                        ("decode K", dec[:, :, 0].permute(1, 2, 0, 3)), ("decode V", dec[:, :, 1].permute(1, 2, 0, 3))):
            loc = first(t)
            if loc is not None:
                raise DataError(f"non-finite {name} element at layer {loc[0]}, head {loc[1]}, token {loc[2]}, "
                                f"dim {loc[3]}")
    return DeviceTrace(h, pre[:, 0].reshape(L * H, T, d).contiguous(), pre[:, 1].reshape(L * H, T, d).contiguous(),
                       dec[:, :, 0].reshape(S, L * H, d).contiguous(), dec[:, :, 1].reshape(S, L * H, d).contiguous())


def ingest_trace(path: str, config, max_steps: int | None = None, record_decisions: bool = False):
    """KVTR -> HBM -> prefill + decode appends of every (layer, head) in one cache.
    Returns (cache, device_trace)."""
    from .cache import PatternKVCache

    tr = load_trace_device(path)
    h = tr.header
    steps = h.decode_steps if max_steps is None else min(max_steps, h.decode_steps)
    cache = PatternKVCache(config, tr.n_units, h.head_dim, dtype=tr.prefill_k.dtype,
                           max_tokens=h.prefill_len + steps + 2 * config.group_size,
                           record_decisions=record_decisions)
    cache.prefill(tr.prefill_k, tr.prefill_v)
    for s in range(steps):
        cache.append(tr.decode_k[s], tr.decode_v[s])
    return cache, tr
