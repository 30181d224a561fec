"""Per-head cache engine API of the reference (engine.py:35-471), as a facade
over the B200 cache (PatternKVCache, one unit, fp64 inputs so every value the
reference sees is reproduced exactly).

The state lives on the GPU; the reference's HeadCacheState attributes
(k_patterns, k_blocks, v_tokens, window_k, v_decisions, ...) are exported
lazily from the device arenas.  run_scheme_comparison batches every
(layer, head) of a stream into one multi-unit cache per scheme.
"""

from __future__ import annotations

import math
from bisect import bisect_right
from dataclasses import dataclass, field

import numpy as np
import torch

from .cache import PatternKVCache, require_cuda
from .config import EngineConfig
from .errors import DataError, UsageError
from .export import export_unit
from .gate import GateConfig, GateDecision
from .patterns import ORIGIN_DECODE, ORIGIN_PREFILL, PatternSet
from .quant import PER_CHANNEL, PER_TOKEN, QuantizedGroup, QuantParams

RAW_MARKER = -1

__all__ = [
    "RAW_MARKER", "EngineConfig", "CommittedKBlock", "CommittedVToken", "HeadCacheState", "prefill",
    "append_decode_token", "reconstruct_token", "committed_matrices", "accounted_bits_per_token", "replay_head",
    "run_scheme_comparison", "HeadReport", "CacheMetrics",
]


@dataclass
class CommittedKBlock:
    start_token: int
    length: int
    channel_groups: list
    pattern_indices: np.ndarray


@dataclass
class CommittedVToken:
    token_index: int
    group: QuantizedGroup
    pattern_index: int


class HeadCacheState:
    """Cache state of one attention head (engine.py:104-129), stored on the GPU."""

    def __init__(self, config: EngineConfig, head_dim: int, _cache: PatternKVCache | None = None, _unit: int = 0):
        self.config = config
        self.head_dim = head_dim
        self._cache = _cache
        self._unit = _unit
        self._snap = None
        self._snap_key = None
        self._gate = None
        self._tokens = 0

    # -- device cache, created on first use -------------------------------------------------
    def _device(self) -> PatternKVCache:
        if self._cache is None:
            require_cuda()
            self._cache = PatternKVCache(self.config, 1, self.head_dim, dtype=torch.float64, max_tokens=256,
                                         record_decisions=True)
        return self._cache

    def _export(self):
        if self._cache is None:
            return None
        key = self._cache.info().token_count
        if self._snap is None or self._snap_key != key:
            self._snap = export_unit(self._cache, self._unit)
            self._snap_key = key
        return self._snap

    # -- reference attributes -------------------------------------------------------------
    @property
    def token_count(self) -> int:
        return 0 if self._cache is None else self._cache.info().token_count

    @property
    def committed_count(self) -> int:
        return 0 if self._cache is None else self._cache.info().committed_count

    @property
    def gate(self) -> GateConfig:
        if self._gate is None:
            self._gate = GateConfig.create(self.head_dim, self.config.alpha)
        return self._gate

    def _patterns(self, side: int) -> PatternSet:
        s = self._export()
        if s is None:
            return PatternSet(self.head_dim)
        mat = s.kpat if side == 0 else s.vpat
        n0 = s.n_prefill_k if side == 0 else s.n_prefill_v
        return PatternSet.from_matrix(mat, [ORIGIN_PREFILL] * min(n0, len(mat)) + [ORIGIN_DECODE] * max(len(mat) - n0, 0))

    @property
    def k_patterns(self) -> PatternSet:
        return self._patterns(0)

    @property
    def v_patterns(self) -> PatternSet:
        return self._patterns(1)

    @property
    def k_blocks(self) -> list[CommittedKBlock]:
        s = self._export()
        if s is None:
            return []
        bits = self.config.bits
        out = []
        for b in range(len(s.kb_start)):
            st, n = int(s.kb_start[b]), int(s.kb_len[b])
            groups = [QuantizedGroup(QuantParams(float(s.k_scale[b, c]), float(s.k_zero[b, c]), bits), s.k_bytes[b][c],
                                     n, PER_CHANNEL) for c in range(self.head_dim)]
            out.append(CommittedKBlock(st, n, groups, s.k_idx[st:st + n].astype(np.int32)))
        return out

    @property
    def v_tokens(self) -> list[CommittedVToken]:
        s = self._export()
        if s is None:
            return []
        bits = self.config.bits
        return [CommittedVToken(t, QuantizedGroup(QuantParams(float(s.v_scale[t]), float(s.v_zero[t]), bits),
                                                  s.v_bytes[t], self.head_dim, PER_TOKEN), int(s.v_idx[t]))
                for t in range(len(s.v_idx))]

    @property
    def window_k(self) -> list[np.ndarray]:
        s = self._export()
        return [] if s is None else [r.copy() for r in s.window_k]

    @property
    def window_v(self) -> list[np.ndarray]:
        s = self._export()
        return [] if s is None else [r.copy() for r in s.window_v]

    @staticmethod
    def _decisions(arr: np.ndarray) -> list[GateDecision]:
        out = []
        for raw, flat, fl in arr:
            ratio = math.inf if raw == 0.0 else flat / raw
            out.append(GateDecision(flatten=bool(fl), ratio=ratio, raw_range=float(raw), flat_range=float(flat)))
        return out

    @property
    def v_decisions(self) -> list[GateDecision]:
        s = self._export()
        return [] if s is None else self._decisions(s.vdec)

    @property
    def k_decisions(self) -> list[GateDecision]:
        s = self._export()
        return [] if s is None else self._decisions(s.kdec)


def _as_matrix(arr, name: str) -> np.ndarray:
    mat = np.asarray(arr, dtype=np.float64)
    if mat.ndim != 2 or mat.shape[0] < 1:
        raise UsageError(f"{name} must be a non-empty (tokens, dim) matrix")
    if not np.isfinite(mat).all():
        loc = np.argwhere(~np.isfinite(mat))[0]
        raise DataError(f"non-finite {name} element at token {loc[0]}, dim {loc[1]}")
    return mat


def prefill(k_tensor, v_tensor, config: EngineConfig) -> HeadCacheState:
    """Mine, commit all but the newest min(T, W) tokens, keep the window (engine.py:142-169)."""
    k = _as_matrix(k_tensor, "prefill K")
    v = _as_matrix(v_tensor, "prefill V")
    if k.shape != v.shape:
        raise UsageError(f"prefill K {k.shape} and V {v.shape} must have equal shapes")
    state = HeadCacheState(config, k.shape[1])
    cache = state._device()
    cache.prefill(torch.from_numpy(k)[None], torch.from_numpy(v)[None])
    return state


def append_decode_token(k_vec, v_vec, state: HeadCacheState) -> HeadCacheState:
    """Append one token; flush the oldest group when the window reaches W + G (engine.py:172-198)."""
    state = _on_device(state)
    k = np.asarray(k_vec, dtype=np.float64).ravel()
    v = np.asarray(v_vec, dtype=np.float64).ravel()
    if k.shape != (state.head_dim,) or v.shape != (state.head_dim,):
        raise UsageError(f"decode vectors must have dimension {state.head_dim}")
    if not (np.isfinite(k).all() and np.isfinite(v).all()):
        raise DataError(f"non-finite decode vector at token {state.token_count}")
    state._device().append(torch.from_numpy(k)[None], torch.from_numpy(v)[None])
    return state


def _on_device(state):
    """A HeadCacheState as is; a loaded snapshot state (snapshot.SnapshotState) resumed on the GPU."""
    return state if isinstance(state, HeadCacheState) else state.device_state()


def reconstruct_token(state: HeadCacheState, token_index: int) -> tuple[np.ndarray, np.ndarray]:
    """One token's (K, V); exact for window tokens (engine.py:271-293)."""
    state = _on_device(state)
    if not 0 <= token_index < state.token_count:
        raise UsageError(f"token index {token_index} outside [0, {state.token_count})")
    committed = state.committed_count
    if token_index >= committed:
        s = state._export()
        off = token_index - committed
        return s.window_k[off].copy(), s.window_v[off].copy()
    k, v = state._cache.dequant(token_index, token_index + 1)
    return k[state._unit, 0].cpu().numpy(), v[state._unit, 0].cpu().numpy()


def committed_matrices(state: HeadCacheState) -> tuple[np.ndarray, np.ndarray]:
    """All committed tokens reconstructed (engine.py:296-303), exact fp64 on the GPU."""
    state = _on_device(state)
    d = state.head_dim
    if state.committed_count == 0:
        return np.empty((0, d)), np.empty((0, d))
    k, v = state._cache.dequant()
    return k[state._unit].cpu().numpy(), v[state._unit].cpu().numpy()


def _side_bit_totals(state: HeadCacheState, side: str) -> tuple[int, int, int, int]:
    """(codes, params, indices, patterns) bits held on one side (engine.py:306-321)."""
    cfg = state.config
    d = state.head_dim
    c = state.committed_count
    s = state._export()
    if side == "k":
        nblk = 0 if s is None else len(s.kb_start)
        npat = 0 if s is None else len(s.kpat)
        return c * cfg.bits * d, 32 * d * nblk, (16 * c if cfg.use_k_patterns else 0), 16 * d * npat
    npat = 0 if s is None else len(s.vpat)
    return c * cfg.bits * d, 32 * c, (16 * c if cfg.use_v_patterns else 0), 16 * d * npat


def accounted_bits_per_token(state: HeadCacheState, side: str) -> float:
    """Committed storage cost per token (engine.py:324-333)."""
    if side not in ("k", "v"):
        raise UsageError(f"side must be 'k' or 'v', got {side!r}")
    c = state.committed_count
    if c == 0:
        return 0.0
    codes, params, index, patterns = _side_bit_totals(state, side)
    return codes / c + params / c + index / c + patterns / c


@dataclass
class HeadReport:
    layer: int
    head: int
    committed_tokens: int
    k_mse: float
    v_mse: float
    mse: float
    v_gate_acceptance_rate: float
    k_pattern_count: int
    v_pattern_count: int


@dataclass
class CacheMetrics:
    scheme: str
    config: EngineConfig
    committed_tokens: int
    k_mse: float
    v_mse: float
    mse: float
    k_bits_per_token: float
    v_bits_per_token: float
    bits_per_token: float
    v_gate_acceptance_rate: float
    ratios: np.ndarray
    raw_ranges: np.ndarray
    flat_ranges: np.ndarray
    per_head: list = field(default_factory=list)


def replay_head(k_prefill, v_prefill, k_decode, v_decode, config: EngineConfig) -> HeadCacheState:
    """Prefill then append every decode step for one head (engine.py:369-380)."""
    state = prefill(k_prefill, v_prefill, config)
    kd = np.asarray(k_decode, dtype=np.float64)
    vd = np.asarray(v_decode, dtype=np.float64)
    if kd.shape[0]:
        if not (np.isfinite(kd).all() and np.isfinite(vd).all()):
            bad = int(np.argwhere(~(np.isfinite(kd).all(axis=1) & np.isfinite(vd).all(axis=1)))[0][0])
            # replay the finite prefix so the error carries the right token index
            for t in range(bad):
                append_decode_token(kd[t], vd[t], state)
            raise DataError(f"non-finite decode vector at token {state.token_count}")
        cache = state._device()
        kt = torch.from_numpy(np.ascontiguousarray(kd)).cuda()
        vt = torch.from_numpy(np.ascontiguousarray(vd)).cuda()
        for t in range(kd.shape[0]):
            cache.append(kt[t][None], vt[t][None])
    return state


def run_scheme_comparison(stream, schemes: list[tuple[str, EngineConfig]]) -> list[CacheMetrics]:
    """Replay one stream under every scheme plus a raw baseline (engine.py:383-471).

    All (layer, head) units of the stream advance together in one GPU cache per
    scheme; metrics are reduced on the device in fp64."""
    if not schemes:
        raise UsageError("at least one scheme is required")
    for name, config in schemes:
        if name == "raw" and not config.is_raw:
            raise UsageError("a scheme named 'raw' must have all pattern toggles off")
    if not any(config.is_raw for _, config in schemes):
        schemes = [("raw", schemes[0][1].raw_variant())] + list(schemes)
    require_cuda()
    L, H = stream.num_layers, stream.num_heads
    d = stream.head_dim
    U = L * H
    kp = torch.from_numpy(np.ascontiguousarray(stream.prefill_k, dtype=np.float64).reshape(U, -1, d)).cuda()
    vp = torch.from_numpy(np.ascontiguousarray(stream.prefill_v, dtype=np.float64).reshape(U, -1, d)).cuda()
    kd = torch.from_numpy(np.ascontiguousarray(stream.decode_k, dtype=np.float64).reshape(U, -1, d)).cuda()
    vd = torch.from_numpy(np.ascontiguousarray(stream.decode_v, dtype=np.float64).reshape(U, -1, d)).cuda()
    truth_k = torch.cat([kp, kd], dim=1)
    truth_v = torch.cat([vp, vd], dim=1)
    results = []
    for name, config in schemes:
        cache = PatternKVCache(config, U, d, dtype=torch.float64, max_tokens=truth_k.shape[1] + 256,
                               record_decisions=True)
        cache.prefill(kp, vp)
        for t in range(kd.shape[1]):
            cache.append(kd[:, t], vd[:, t])
        c = cache.info().committed_count
        rk, rv = cache.dequant()
        err_k = ((rk - truth_k[:, :c]) ** 2).sum(dim=(1, 2)).cpu().numpy()
        err_v = ((rv - truth_v[:, :c]) ** 2).sum(dim=(1, 2)).cpu().numpy()
        bit_totals = {"k": np.zeros(4, np.int64), "v": np.zeros(4, np.int64)}
        ratios, raws, flats, per_head = [], [], [], []
        flattened = gated = 0
        for u in range(U):
            st = HeadCacheState(config, d, _cache=cache, _unit=u)
            for side in ("k", "v"):
                bit_totals[side] += np.asarray(_side_bit_totals(st, side), dtype=np.int64)
            decs = st._export().vdec
            head_flat = int(decs[:, 2].sum()) if len(decs) else 0
            flattened += head_flat
            gated += len(decs)
            if len(decs):
                raws.append(decs[:, 0])
                flats.append(decs[:, 1])
                with np.errstate(divide="ignore", invalid="ignore"):
                    ratios.append(np.where(decs[:, 0] == 0.0, np.inf, decs[:, 1] / np.where(decs[:, 0] == 0, 1, decs[:, 0])))
            denom = max(c, 1) * d
            s = st._export()
            per_head.append(HeadReport(layer=u // H, head=u % H, committed_tokens=c, k_mse=float(err_k[u]) / denom,
                                       v_mse=float(err_v[u]) / denom, mse=float(err_k[u] + err_v[u]) / (2 * denom),
                                       v_gate_acceptance_rate=head_flat / len(decs) if len(decs) else 0.0,
                                       k_pattern_count=len(s.kpat), v_pattern_count=len(s.vpat)))
        committed_total = c * U
        denom = max(committed_total, 1) * d
        side_bits = {}
        for side in ("k", "v"):
            codes, params, index, patterns = (int(x) for x in bit_totals[side])
            cc = max(committed_total, 1)
            side_bits[side] = codes / cc + params / cc + index / cc + patterns / cc
        sse_k, sse_v = float(err_k.sum()), float(err_v.sum())
        results.append(CacheMetrics(
            scheme=name, config=config, committed_tokens=committed_total,
            k_mse=sse_k / denom, v_mse=sse_v / denom, mse=(sse_k + sse_v) / (2 * denom),
            k_bits_per_token=side_bits["k"], v_bits_per_token=side_bits["v"],
            bits_per_token=side_bits["k"] + side_bits["v"],
            v_gate_acceptance_rate=flattened / gated if gated else 0.0,
            ratios=np.concatenate(ratios) if ratios else np.empty(0),
            raw_ranges=np.concatenate(raws) if raws else np.empty(0),
            flat_ranges=np.concatenate(flats) if flats else np.empty(0),
            per_head=per_head,
        ))
    return results
