"""PKVS binary snapshots of committed cache state (reference snapshot.py:1-243).

Same byte layout as the reference (little-endian, packed; snapshot.py:3-28):

    magic b"PKVS", version u32 = 1
    config  bits u8, pattern_count u32, group_size u32, residual_window u32,
            alpha f64, flags u8 (bit0 use_k_patterns, bit1 use_v_patterns,
            bit2 generate_new_patterns, bit3 use_v_gate, bit4 use_k_gate), seed i64
    head_dim u32, state count u32, then per (layer, head) in sorted order:
        layer u32, head u32, token_count u64
        K / V patterns: u32 count, per pattern origin u8 (0 prefill, 1 decode) + d f64
        K blocks: u32 count, per block start u64, length u32, length i32 indices,
                  then d x (scale f64, zero f64, ceil(length*bits/8) packed bytes)
        V tokens: u32 count, per token index u64, pattern i32, scale f64, zero f64,
                  ceil(d*bits/8) packed bytes
        window: u32 count, count*d f64 K rows, then the V rows
        V then K gate decisions: u32 count, per decision flatten u8, ratio f64,
                  raw_range f64, flat_range f64

save_snapshot / load_snapshot keep the reference's names, argument meaning and
errors (UsageError for an empty or mixed cache, DataError with the byte offset
for malformed input).  States backed by a B200 cache (engine.HeadCacheState,
or a whole PatternKVCache through save_cache_snapshot) are serialized from one
export of the device arenas per unit, with numpy building each section in bulk
instead of per-object loops.  restore_cache() is the resume half: it loads a
snapshot back into a device cache (cache.PatternKVCache.import_state).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

from .config import EngineConfig
from .errors import DataError, UsageError
from .gate import GateConfig, GateDecision
from .patterns import ORIGIN_DECODE, ORIGIN_PREFILL, PatternSet
from .quant import PER_CHANNEL, PER_TOKEN, QuantizedGroup, QuantParams

SNAPSHOT_MAGIC = b"PKVS"
SNAPSHOT_VERSION = 1
_ORIGIN_CODE = {ORIGIN_PREFILL: 0, ORIGIN_DECODE: 1}
_ORIGIN_NAME = {0: ORIGIN_PREFILL, 1: ORIGIN_DECODE}


def _flags(cfg: EngineConfig) -> int:
    return (int(cfg.use_k_patterns) | int(cfg.use_v_patterns) << 1 | int(cfg.generate_new_patterns) << 2
            | int(cfg.use_v_gate) << 3 | int(cfg.use_k_gate) << 4)


def _header(cfg: EngineConfig, head_dim: int, count: int) -> bytes:
    return (struct.pack("<4sI", SNAPSHOT_MAGIC, SNAPSHOT_VERSION)
            + struct.pack("<BIIIdBq", cfg.bits, cfg.pattern_count, cfg.group_size, cfg.residual_window, cfg.alpha,
                          _flags(cfg), cfg.seed)
            + struct.pack("<II", head_dim, count))


# ---- bulk section writers (arrays in, bytes out) ------------------------------------------
def _patterns_bytes(mat: np.ndarray, decode: np.ndarray) -> bytes:
    n, d = mat.shape
    if n == 0:
        return struct.pack("<I", 0)
    rec = np.zeros(n, dtype=np.dtype([("o", "u1"), ("v", "<f8", (d,))]))
    rec["o"] = decode.astype(np.uint8)
    rec["v"] = mat
    return struct.pack("<I", n) + rec.tobytes()


def _decisions_bytes(dec: np.ndarray) -> bytes:
    """dec: [n, 3] (raw_range, flat_range, flatten) -> ratio as the reference computes it."""
    n = len(dec)
    rec = np.zeros(n, dtype=np.dtype([("f", "u1"), ("r", "<f8"), ("raw", "<f8"), ("flat", "<f8")]))
    if n:
        raw, flat = dec[:, 0], dec[:, 1]
        with np.errstate(divide="ignore", invalid="ignore"):
            ratio = np.where(raw == 0.0, np.inf, flat / np.where(raw == 0.0, 1.0, raw))
        rec["f"] = dec[:, 2] != 0
        rec["r"] = ratio
        rec["raw"] = raw
        rec["flat"] = flat
    return struct.pack("<I", n) + rec.tobytes()


def _unit_bytes(layer: int, head: int, us, bits: int, d: int) -> bytes:
    """One state from an export.UnitState (device arenas already on the host)."""
    out = [struct.pack("<IIQ", layer, head, us.token_count)]
    nk, nv = len(us.kpat), len(us.vpat)
    out.append(_patterns_bytes(np.asarray(us.kpat, np.float64).reshape(nk, d), np.arange(nk) >= us.n_prefill_k))
    out.append(_patterns_bytes(np.asarray(us.vpat, np.float64).reshape(nv, d), np.arange(nv) >= us.n_prefill_v))
    nb = len(us.kb_start)
    out.append(struct.pack("<I", nb))
    for b in range(nb):
        s, n = int(us.kb_start[b]), int(us.kb_len[b])
        out.append(struct.pack("<QI", s, n))
        out.append(us.k_idx[s:s + n].astype("<i4").tobytes())
        pk = (n * bits + 7) // 8
        rec = np.zeros(d, dtype=np.dtype([("s", "<f8"), ("z", "<f8"), ("c", "u1", (pk,))]))
        rec["s"] = us.k_scale[b]
        rec["z"] = us.k_zero[b]
        rec["c"] = np.frombuffer(b"".join(us.k_bytes[b]), np.uint8).reshape(d, pk)
        out.append(rec.tobytes())
    C = len(us.v_idx)
    pv = (d * bits + 7) // 8
    rec = np.zeros(C, dtype=np.dtype([("t", "<u8"), ("p", "<i4"), ("s", "<f8"), ("z", "<f8"), ("c", "u1", (pv,))]))
    if C:
        rec["t"] = np.arange(C, dtype=np.uint64)
        rec["p"] = us.v_idx
        rec["s"] = us.v_scale
        rec["z"] = us.v_zero
        rec["c"] = np.frombuffer(b"".join(us.v_bytes), np.uint8).reshape(C, pv)
    out.append(struct.pack("<I", C) + rec.tobytes())
    out.append(struct.pack("<I", len(us.window_k)))
    out.append(np.ascontiguousarray(us.window_k, dtype="<f8").reshape(-1, d).tobytes())
    out.append(np.ascontiguousarray(us.window_v, dtype="<f8").reshape(-1, d).tobytes())
    out.append(_decisions_bytes(us.vdec))
    out.append(_decisions_bytes(us.kdec))
    return b"".join(out)


# ---- generic writer over the reference's HeadCacheState attribute API -----------------------
def _state_bytes(layer: int, head: int, st) -> bytes:
    out = [struct.pack("<IIQ", layer, head, st.token_count)]
    for ps in (st.k_patterns, st.v_patterns):
        n = len(ps)
        mat = np.array([ps.vector(i) for i in range(n)], dtype=np.float64).reshape(n, st.head_dim)
        out.append(_patterns_bytes(mat, np.array([ps.origin(i) == ORIGIN_DECODE for i in range(n)], bool)))
    out.append(struct.pack("<I", len(st.k_blocks)))
    for blk in st.k_blocks:
        out.append(struct.pack("<QI", blk.start_token, blk.length))
        out.append(np.asarray(blk.pattern_indices, dtype="<i4").tobytes())
        for g in blk.channel_groups:
            out.append(struct.pack("<dd", g.params.scale, g.params.zero_point))
            out.append(g.codes)
    out.append(struct.pack("<I", len(st.v_tokens)))
    for tok in st.v_tokens:
        out.append(struct.pack("<Qidd", tok.token_index, tok.pattern_index, tok.group.params.scale,
                               tok.group.params.zero_point))
        out.append(tok.group.codes)
    out.append(struct.pack("<I", len(st.window_k)))
    for rows in (st.window_k, st.window_v):
        for r in rows:
            out.append(np.asarray(r, dtype="<f8").tobytes())
    for decs in (st.v_decisions, st.k_decisions):
        out.append(struct.pack("<I", len(decs)))
        for dec in decs:
            out.append(struct.pack("<Bddd", int(dec.flatten), dec.ratio, dec.raw_range, dec.flat_range))
    return b"".join(out)


def snapshot_bytes(states: dict) -> bytes:
    """The PKVS image of {(layer, head): HeadCacheState} (snapshot.py:57-99)."""
    if not states:
        raise UsageError("cannot snapshot an empty cache")
    items = sorted(states.items())
    config = items[0][1].config
    head_dim = items[0][1].head_dim
    for _, st in items:
        if st.config != config or st.head_dim != head_dim:
            raise UsageError("all snapshot heads must share one config and head dimension")
    out = [_header(config, head_dim, len(items))]
    for (layer, head), st in items:
        export = getattr(st, "_export", None)
        us = export() if export is not None else None
        out.append(_unit_bytes(layer, head, us, config.bits, head_dim) if us is not None
                   else _state_bytes(layer, head, st))
    return b"".join(out)


def save_snapshot(path: str, states: dict) -> None:
    """Serialize a cache (one config, many heads) to the snapshot format."""
    blob = snapshot_bytes(states)
    with open(path, "wb") as fh:
        fh.write(blob)


def cache_snapshot_bytes(cache, keys=None) -> bytes:
    """PKVS image of every unit of a PatternKVCache; keys[u] = (layer, head) of unit u
    (default (0, u)).  One arena export per unit, bulk section writers."""
    from .export import export_unit

    keys = list(keys) if keys is not None else [(0, u) for u in range(cache.n_units)]
    if len(keys) != cache.n_units or len(set(keys)) != len(keys):
        raise UsageError("keys must name every unit of the cache exactly once")
    if cache.n_units == 0:
        raise UsageError("cannot snapshot an empty cache")
    order = sorted(range(cache.n_units), key=lambda u: keys[u])
    out = [_header(cache.config, cache.head_dim, cache.n_units)]
    for u in order:
        out.append(_unit_bytes(keys[u][0], keys[u][1], export_unit(cache, u), cache.config.bits, cache.head_dim))
    return b"".join(out)


def save_cache_snapshot(path: str, cache, keys=None) -> None:
    with open(path, "wb") as fh:
        fh.write(cache_snapshot_bytes(cache, keys))


# ---- reader ------------------------------------------------------------------------------
@dataclass
class SnapshotBlock:
    start_token: int
    length: int
    channel_groups: list
    pattern_indices: np.ndarray


@dataclass
class SnapshotToken:
    token_index: int
    group: QuantizedGroup
    pattern_index: int


@dataclass
class SnapshotState:
    """Host copy of one head's state with the reference's HeadCacheState attributes
    (engine.py:104-129); restore_cache() puts it back on the GPU."""

    config: EngineConfig
    head_dim: int
    token_count: int = 0
    k_patterns: PatternSet = None
    v_patterns: PatternSet = None
    k_blocks: list = field(default_factory=list)
    v_tokens: list = field(default_factory=list)
    window_k: list = field(default_factory=list)
    window_v: list = field(default_factory=list)
    v_decisions: list = field(default_factory=list)
    k_decisions: list = field(default_factory=list)
    _facade: object = field(default=None, repr=False, compare=False)

    @property
    def gate(self) -> GateConfig:
        return GateConfig.create(self.head_dim, self.config.alpha)

    def device_state(self):
        """This state resumed on the GPU as an engine.HeadCacheState (one-unit cache via
        pkv_cache_import), created once; the engine's functions route a loaded snapshot
        state through it (reconstruct_token, committed_matrices, append_decode_token ...)."""
        if self._facade is None:
            import torch

            from .engine import HeadCacheState
            cache, _ = restore_cache({(0, 0): self}, dtype=torch.float64)
            self._facade = HeadCacheState(self.config, self.head_dim, _cache=cache, _unit=0)
        return self._facade


    @property
    def committed_count(self) -> int:
        return len(self.v_tokens)


class _Reader:
    def __init__(self, blob: bytes):
        self.blob = blob
        self.pos = 0

    def take(self, fmt: str) -> tuple:
        size = struct.calcsize(fmt)
        if self.pos + size > len(self.blob):
            raise DataError(f"snapshot truncated at byte offset {self.pos}, needed {size} more bytes")
        vals = struct.unpack_from(fmt, self.blob, self.pos)
        self.pos += size
        return vals

    def take_bytes(self, size: int) -> bytes:
        if self.pos + size > len(self.blob):
            raise DataError(f"snapshot truncated at byte offset {self.pos}, needed {size} more bytes")
        chunk = self.blob[self.pos:self.pos + size]
        self.pos += size
        return chunk

    def take_f64(self, count: int) -> np.ndarray:
        return np.frombuffer(self.take_bytes(8 * count), dtype="<f8").astype(np.float64)


def _read_patterns(rd: _Reader, d: int) -> PatternSet:
    (n,) = rd.take("<I")
    vecs, origins = [], []
    for _ in range(n):
        (code,) = rd.take("<B")
        if code not in _ORIGIN_NAME:
            raise DataError(f"unknown pattern origin code {code} at byte offset {rd.pos - 1}")
        vecs.append(rd.take_f64(d))
        origins.append(_ORIGIN_NAME[code])
    return PatternSet.from_matrix(np.array(vecs).reshape(n, d), origins) if n else PatternSet(d)


def _read_decisions(rd: _Reader) -> list:
    (n,) = rd.take("<I")
    out = []
    for _ in range(n):
        fl, ratio, raw, flat = rd.take("<Bddd")
        out.append(GateDecision(flatten=bool(fl), ratio=ratio, raw_range=raw, flat_range=flat))
    return out


def parse_snapshot(blob: bytes):
    """(EngineConfig, {(layer, head): SnapshotState}) from a PKVS image (snapshot.py:148-220)."""
    rd = _Reader(blob)
    magic, version = rd.take("<4sI")
    if magic != SNAPSHOT_MAGIC:
        raise DataError(f"bad magic {magic!r} at byte offset 0, expected {SNAPSHOT_MAGIC!r}")
    if version != SNAPSHOT_VERSION:
        raise DataError(f"unsupported snapshot version {version} at byte offset 4")
    bits, pattern_count, group_size, residual_window, alpha, flags, seed = rd.take("<BIIIdBq")
    cfg = EngineConfig(bits=bits, pattern_count=pattern_count, group_size=group_size,
                       residual_window=residual_window, alpha=alpha, use_k_patterns=bool(flags & 1),
                       use_v_patterns=bool(flags & 2), generate_new_patterns=bool(flags & 4),
                       use_v_gate=bool(flags & 8), use_k_gate=bool(flags & 16), seed=seed)
    d, count = rd.take("<II")
    packed = lambda n: (n * bits + 7) // 8  # noqa: E731
    states = {}
    for _ in range(count):
        layer, head, token_count = rd.take("<IIQ")
        st = SnapshotState(cfg, d, token_count)
        st.k_patterns = _read_patterns(rd, d)
        st.v_patterns = _read_patterns(rd, d)
        (nb,) = rd.take("<I")
        for _ in range(nb):
            start, length = rd.take("<QI")
            idx = np.frombuffer(rd.take_bytes(4 * length), dtype="<i4").astype(np.int32)
            groups = []
            for _ in range(d):
                scale, zero = rd.take("<dd")
                groups.append(QuantizedGroup(QuantParams(scale, zero, bits), rd.take_bytes(packed(length)), length,
                                             PER_CHANNEL))
            st.k_blocks.append(SnapshotBlock(start, length, groups, idx))
        (nv,) = rd.take("<I")
        for _ in range(nv):
            ti, pi = rd.take("<Qi")
            scale, zero = rd.take("<dd")
            st.v_tokens.append(SnapshotToken(ti, QuantizedGroup(QuantParams(scale, zero, bits),
                                                                rd.take_bytes(packed(d)), d, PER_TOKEN), pi))
        (nw,) = rd.take("<I")
        st.window_k = [rd.take_f64(d) for _ in range(nw)]
        st.window_v = [rd.take_f64(d) for _ in range(nw)]
        st.v_decisions = _read_decisions(rd)
        st.k_decisions = _read_decisions(rd)
        states[(layer, head)] = st
    if rd.pos != len(rd.blob):
        raise DataError(f"unexpected {len(rd.blob) - rd.pos} trailing bytes at offset {rd.pos}")
    return cfg, states


def load_snapshot(path: str):
    """Load a snapshot back into per-head states (host copies)."""
    with open(path, "rb") as fh:
        return parse_snapshot(fh.read())


# ---- resume: snapshot states -> device cache ---------------------------------------------
def _unpack_le(blob: bytes, count: int, length: int, bits: int) -> np.ndarray:
    """count groups of `length` codes packed little-endian within a byte, first code in the
    lowest bits, each group ceil(length*bits/8) bytes (quant.py:120-146) -> uint8 [count, length]."""
    per = 8 // bits
    nbytes = (length * bits + 7) // 8
    raw = np.frombuffer(blob, np.uint8).reshape(count, nbytes)
    shifts = (np.arange(per, dtype=np.uint8) * bits)
    codes = (raw[:, :, None] >> shifts[None, None, :]) & ((1 << bits) - 1)
    return codes.reshape(count, nbytes * per)[:, :length].astype(np.uint8)


def restore_cache(states: dict, dtype=None, max_tokens: int | None = None, record_decisions: bool = True):
    """Resume: put {(layer, head): HeadCacheState} (e.g. from load_snapshot) back into one
    B200 cache, unit u = the u-th key in sorted order.  The heads must be in lockstep (same
    token count, block geometry and window), as the units of a PatternKVCache are.
    Returns (cache, keys)."""
    import torch

    from . import _lib
    from .cache import PatternKVCache, _ptr, _stream

    if not states:
        raise UsageError("cannot restore an empty snapshot")
    keys = sorted(states)
    sts = [states[k] for k in keys]
    cfg, d = sts[0].config, sts[0].head_dim
    bits = cfg.bits
    geo = [(b.start_token, b.length) for b in sts[0].k_blocks]
    for st in sts:
        if st.config != cfg or st.head_dim != d:
            raise UsageError("all restored heads must share one config and head dimension")
        if st.token_count != sts[0].token_count or [(b.start_token, b.length) for b in st.k_blocks] != geo \
                or len(st.window_k) != len(sts[0].window_k):
            raise UsageError("restored heads must be in lockstep (token count, blocks, window)")
    U, nb, C, win = len(sts), len(geo), sum(n for _, n in geo), len(sts[0].window_k)
    dtype = dtype or torch.float64
    tokens = sts[0].token_count
    cap = max(max_tokens or 0, tokens + 4 * cfg.group_size)
    nk = [len(st.k_patterns) for st in sts]
    nv = [len(st.v_patterns) for st in sts]
    Pk, Pv = max(nk), max(nv)
    cache = PatternKVCache(cfg, U, d, dtype=dtype, max_tokens=cap, max_patterns=max(Pk, Pv) + 64,
                           record_decisions=record_decisions)
    dev = lambda a, t: torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=t)  # noqa: E731
    kpat = np.zeros((U, max(Pk, 1), d))
    vpat = np.zeros((U, max(Pv, 1), d))
    for u, st in enumerate(sts):
        for i in range(nk[u]):
            kpat[u, i] = st.k_patterns.vector(i)
        for i in range(nv[u]):
            vpat[u, i] = st.v_patterns.vector(i)
    kparam = np.zeros((U, max(nb, 1), 2, d))
    kidx = np.full((U, max(C, 1)), -1, np.int32)
    vidx = np.full((U, max(C, 1)), -1, np.int32)
    vparam = np.zeros((U, max(C, 1), 2))
    kc = np.zeros((U, max(C, 1), d), np.uint8)
    vc = np.zeros((U, max(C, 1), d), np.uint8)
    for u, st in enumerate(sts):
        for b, blk in enumerate(st.k_blocks):
            s, n = blk.start_token, blk.length
            kparam[u, b, 0] = [g.params.scale for g in blk.channel_groups]
            kparam[u, b, 1] = [g.params.zero_point for g in blk.channel_groups]
            kidx[u, s:s + n] = blk.pattern_indices
            kc[u, s:s + n] = _unpack_le(b"".join(g.codes for g in blk.channel_groups), d, n, bits).T
        if C:
            vidx[u, :C] = [t.pattern_index for t in st.v_tokens]
            vparam[u, :C, 0] = [t.group.params.scale for t in st.v_tokens]
            vparam[u, :C, 1] = [t.group.params.zero_point for t in st.v_tokens]
            vc[u, :C] = _unpack_le(b"".join(t.group.codes for t in st.v_tokens), C, d, bits)
    wk = np.array([np.asarray(st.window_k, np.float64).reshape(win, d) for st in sts]).reshape(U, win, d)
    wv = np.array([np.asarray(st.window_v, np.float64).reshape(win, d) for st in sts]).reshape(U, win, d)
    kd = vd = None
    if record_decisions:
        nvd = len(sts[0].v_decisions)
        first = C - nvd
        if nvd and all(len(st.v_decisions) == nvd for st in sts):
            vd = np.zeros((U, max(C, 1), 2))
            for u, st in enumerate(sts):
                vd[u, first:C] = decisions_array(st.v_decisions)[:, :2]
        nkd = len(sts[0].k_decisions)
        if nkd and all(len(st.k_decisions) == nkd for st in sts):
            kd = np.zeros((U, max(C, 1), 2))
            for u, st in enumerate(sts):
                kd[u, C - nkd:C] = decisions_array(st.k_decisions)[:, :2]
        cache.first_decision_token = first if nvd else C
    t_kp, t_vp = dev(kpat, torch.float64), dev(vpat, torch.float64)
    t_par, t_vpar = dev(kparam, torch.float64), dev(vparam, torch.float64)
    t_ki, t_vi = dev(kidx, torch.int32), dev(vidx, torch.int32)
    t_kc, t_vc = dev(kc, torch.uint8), dev(vc, torch.uint8)
    t_wk, t_wv = dev(wk, dtype), dev(wv, dtype)
    t_kd = dev(kd, torch.float64) if kd is not None else None
    t_vd = dev(vd, torch.float64) if vd is not None else None
    import ctypes as C_
    bs = (C_.c_int64 * max(nb, 1))(*[s for s, _ in geo])
    bl = (C_.c_int32 * max(nb, 1))(*[n for _, n in geo])
    cnk = (C_.c_int32 * U)(*nk)
    cnv = (C_.c_int32 * U)(*nv)
    _lib.call("pkv_cache_import", cache._h, tokens, nb, bs, bl, nb, win, Pk, Pv, cnk, cnv, _ptr(t_kp), _ptr(t_vp),
              _ptr(t_par), _ptr(t_ki), _ptr(t_vi), _ptr(t_vpar), _ptr(t_kc), _ptr(t_vc), _ptr(t_wk), _ptr(t_wv),
              _ptr(t_kd), _ptr(t_vd), _stream())
    npk = [sum(st.k_patterns.origin(i) == ORIGIN_PREFILL for i in range(len(st.k_patterns))) for st in sts]
    npv = [sum(st.v_patterns.origin(i) == ORIGIN_PREFILL for i in range(len(st.v_patterns))) for st in sts]
    cache.prefill_pattern_counts = (npk, npv)
    torch.cuda.synchronize()
    return cache, keys


def decisions_array(decs: list) -> np.ndarray:
    return np.array([[d.raw_range, d.flat_range, float(d.flatten)] for d in decs], dtype=np.float64).reshape(-1, 3)


def ratio_of(raw: float, flat: float) -> float:
    return math.inf if raw == 0.0 else flat / raw
