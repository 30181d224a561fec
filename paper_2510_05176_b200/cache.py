"""Batched B200 PatternKV cache: U independent (batch, layer, kv-head) units in
lockstep, backed by libpkv_b200.so.  This is the production entry point; the
reference-shaped per-head API (engine.py) is a thin facade over it.

torch supplies device memory and streams only; every computation runs in the
hand-written sm_100a kernels behind the C ABI (include/pkv.h).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DataError, UsageError

RAW_MARKER = -1

_DTYPES = {
    torch.float16: _lib.PKV_F16,
    torch.bfloat16: _lib.PKV_BF16,
    torch.float32: _lib.PKV_F32,
    torch.float64: _lib.PKV_F64,
}


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def require_cuda():
    if not torch.cuda.is_available():
        raise UsageError("no CUDA device: the PatternKV B200 codec has no CPU fallback")


def first_seed_index(n_points: int, seed: int) -> int:
    """np.random.default_rng(seed).integers(T): the reference's first k-means
    center (patterns.py:103, 135).  Host RNG, identical stream."""
    return int(np.random.default_rng(seed).integers(n_points))


def make_config_struct(cfg) -> _lib.PkvConfig:
    return _lib.PkvConfig(
        bits=cfg.bits, pattern_count=cfg.pattern_count, group_size=cfg.group_size,
        residual_window=cfg.residual_window, alpha=cfg.alpha,
        use_k_patterns=int(cfg.use_k_patterns), use_v_patterns=int(cfg.use_v_patterns),
        generate_new_patterns=int(cfg.generate_new_patterns), use_v_gate=int(cfg.use_v_gate),
        use_k_gate=int(cfg.use_k_gate), seed=cfg.seed,
    )


@dataclass
class CacheInfo:
    n_units: int
    head_dim: int
    token_count: int
    committed_count: int
    window_len: int
    window_slot0: int
    n_blocks: int
    pattern_capacity: int
    token_capacity: int
    block_bytes: int
    n_refined: int
    n_exact_div: int


class PatternKVCache:
    """U-unit PatternKV cache on one GPU.

    Args:
        config: EngineConfig-shaped object (bits, pattern_count, group_size,
            residual_window, alpha, toggles, seed).
        n_units: independent (batch, layer, kv-head) units.
        head_dim: d <= 128.
        dtype: element type of the K/V the caller feeds (fp16 for serving,
            fp64 for the reference-exact drop-in path).
        record_decisions: keep per-token gate ranges (GateDecision records).
        stats: count fp64 re-matches and exact-division fallbacks.
    """

    def __init__(self, config, n_units: int, head_dim: int, dtype=torch.float16, max_tokens: int = 4096,
                 max_patterns: int | None = None, record_decisions: bool = False, stats: bool = False):
        require_cuda()
        if dtype not in _DTYPES:
            raise UsageError(f"unsupported dtype {dtype}")
        self.config = config
        self.n_units = n_units
        self.head_dim = head_dim
        self.dtype = dtype
        flags = (_lib.PKV_FLAG_DECISIONS if record_decisions else 0) | (_lib.PKV_FLAG_STATS if stats else 0)
        self._cfg = make_config_struct(config)
        h = C.c_void_p()
        mp = max_patterns if max_patterns is not None else config.pattern_count + 64
        _lib.call("pkv_cache_create", C.byref(self._cfg), n_units, head_dim, _DTYPES[dtype], max_tokens, mp, flags,
                  C.byref(h))
        self._h = h
        self.record_decisions = record_decisions
        # per-unit pattern counts right after the last prefill (device snapshot, read lazily so
        # prefill never blocks the host) and the committed count at that point
        self._npre_dev = None
        self._npre = (np.zeros(n_units, np.int64), np.zeros(n_units, np.int64))
        self._prefill_committed = 0
        self._first_decision = None
        self._part = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().pkv_cache_destroy(h)
            except Exception:  # interpreter shutdown: the module globals may already be gone
                pass
            self._h = None

    # ---- introspection --------------------------------------------------------
    def info(self) -> CacheInfo:
        i = _lib.PkvCacheInfo()
        _lib.call("pkv_cache_info_get", self._h, C.byref(i))
        return CacheInfo(i.n_units, i.head_dim, i.token_count, i.committed_count, i.window_len, i.window_slot0,
                         i.n_blocks, i.pattern_capacity, i.token_capacity, i.block_bytes, i.n_refined, i.n_exact_div)

    def read(self, name: str, dtype: torch.dtype, shape) -> torch.Tensor:
        """Copy the leading elements of a named device arena into a new tensor."""
        out = torch.empty(shape, dtype=dtype, device="cuda")
        nbytes = out.numel() * out.element_size()
        _lib.call("pkv_cache_read", self._h, name.encode(), 0, nbytes, _ptr(out), _stream())
        return out

    def arena_bytes(self, name: str) -> int:
        p = C.c_void_p()
        n = C.c_int64()
        _lib.call("pkv_cache_buffer", self._h, name.encode(), C.byref(p), C.byref(n))
        return n.value

    # ---- inputs -------------------------------------------------------------------
    def _as_input(self, x: torch.Tensor, ndim: int, name: str) -> torch.Tensor:
        if not isinstance(x, torch.Tensor):
            raise UsageError(f"{name} must be a torch tensor")
        if x.device.type != "cuda":
            x = x.to("cuda", non_blocking=True)
        if x.dtype != self.dtype:
            x = x.to(self.dtype)
        if x.dim() != ndim or x.shape[0] != self.n_units or x.shape[-1] != self.head_dim:
            raise UsageError(f"{name} must have shape [n_units={self.n_units}, ..., head_dim={self.head_dim}]")
        return x.contiguous()

    def check_finite(self, x: torch.Tensor) -> int:
        """Flat index of the first non-finite element or -1 (synchronous)."""
        bad = C.c_int64(-1)
        _lib.call("pkv_check_finite", _ptr(x), _DTYPES[x.dtype], x.numel(), C.byref(bad), _stream())
        return bad.value

    # ---- lifecycle ------------------------------------------------------------------
    def prefill(self, k: torch.Tensor, v: torch.Tensor, mine: bool = True, sync_check: bool = False) -> None:
        """engine.py:142-169 for every unit: k, v [U, T, D].

        Non-finite inputs are detected inside the kernels (no extra pass, no host sync) and
        raised as DataError by the next call that checks -- ``check()``, ``append`` -- once
        the GPU has run this prefill; ``sync_check=True`` waits for it and raises here."""
        k = self._as_input(k, 3, "prefill K")
        v = self._as_input(v, 3, "prefill V")
        if k.shape != v.shape:
            raise UsageError(f"prefill K {tuple(k.shape)} and V {tuple(v.shape)} must have equal shapes")
        T = k.shape[1]
        cfg = self.config
        fk = fv = None
        if mine and cfg.use_k_patterns:
            fk = (C.c_int64 * self.n_units)(*([first_seed_index(T, cfg.seed)] * self.n_units))
        if mine and cfg.use_v_patterns:
            fv = (C.c_int64 * self.n_units)(*([first_seed_index(T, cfg.seed + 1)] * self.n_units))
        _lib.call("pkv_prefill", self._h, _ptr(k), _ptr(v), T, fk, fv, _stream())
        # stream-ordered device copies of the per-unit counts: no host synchronisation here
        self._npre_dev = (self.read("nk", torch.int32, (self.n_units,)), self.read("nv", torch.int32, (self.n_units,)))
        self._prefill_committed = T - min(T, cfg.residual_window)
        self._first_decision = None
        if sync_check:
            self.check(wait=True)

    def check(self, wait: bool = True) -> None:
        """Raise DataError (the reference's message + unit) if a prefill / append fed a
        non-finite element (engine.py:136-138, 180-181); wait=False only looks at work the
        GPU has already finished."""
        _lib.call("pkv_cache_check", self._h, int(bool(wait)), None)

    # ---- prefill bookkeeping (read lazily) ------------------------------------------------
    @property
    def prefill_pattern_counts(self):
        """Per-unit (K, V) pattern counts as of the last prefill / restore: patterns below these
        indices have origin "prefill", the rest "decode" (patterns.py:25-60 origins)."""
        if self._npre_dev is not None:
            self._npre = tuple(t.cpu().numpy().astype(np.int64) for t in self._npre_dev)
            self._npre_dev = None
        return self._npre

    @prefill_pattern_counts.setter
    def prefill_pattern_counts(self, counts):
        self._npre_dev = None
        self._npre = tuple(np.asarray(c, np.int64).reshape(self.n_units) for c in counts)

    @property
    def n_prefill_patterns(self):
        """Largest per-unit prefill pattern count per side."""
        nk, nv = self.prefill_pattern_counts
        return int(nk.max(initial=0)), int(nv.max(initial=0))

    @property
    def first_decision_token(self) -> int:
        """Committed tokens before this index carry no gate record (V had no patterns yet)."""
        if self._first_decision is not None:
            return self._first_decision
        if self.config.use_v_patterns and self.n_prefill_patterns[1] == 0:
            return self._prefill_committed
        return 0

    @first_decision_token.setter
    def first_decision_token(self, t: int):
        self._first_decision = int(t)

    def reserve_mining(self, max_tokens: int) -> None:
        """Preallocate the k-means scratch for prefills of up to max_tokens tokens (no
        allocation inside later prefill / mine calls)."""
        _lib.call("pkv_cache_reserve_mining", self._h, int(max_tokens), _stream())

    def reset(self, keep_patterns: bool = True) -> None:
        """Empty the cache (token_count = 0); keep the pattern tables for a re-prefill."""
        _lib.call("pkv_cache_reset", self._h, int(keep_patterns), _stream())

    def set_patterns(self, side: int, patterns: torch.Tensor) -> None:
        """Install fp64 pattern tables [U, P, D] for side 0 (K) or 1 (V)."""
        p = patterns.to(device="cuda", dtype=torch.float64).contiguous()
        if p.dim() != 3 or p.shape[0] != self.n_units or p.shape[2] != self.head_dim:
            raise UsageError("patterns must have shape [n_units, P, head_dim]")
        _lib.call("pkv_set_patterns", self._h, side, _ptr(p), p.shape[1], _stream())

    def commit_prefill(self, k: torch.Tensor, v: torch.Tensor) -> None:
        """Prefill with the installed pattern tables (no mining)."""
        self.prefill(k, v, mine=False)

    def append(self, k: torch.Tensor, v: torch.Tensor, sync_check: bool = False) -> None:
        """engine.py:172-198 for every unit: k, v [U, D].  A non-finite row is flagged inside
        the window copy and raised by a later check()/append (or here with sync_check=True)."""
        k = self._as_input(k, 2, "decode K")
        v = self._as_input(v, 2, "decode V")
        _lib.call("pkv_append", self._h, _ptr(k), _ptr(v), _stream())
        if sync_check:
            self.check(wait=True)

    def mine(self, side: int, x: torch.Tensor, seed: int, labels: bool = False):
        """mine_patterns for every unit (patterns.py:145-158); returns (history [U, 25], niter [U])
        and, with labels=True, the final assignment [U, T] int32 on the device (patterns.py:84-85)."""
        x = self._as_input(x, 3, "mining input")
        T = x.shape[1]
        first = (C.c_int64 * self.n_units)(*([first_seed_index(T, seed)] * self.n_units))
        hist = np.zeros((self.n_units, 25))
        nit = np.zeros(self.n_units, np.int32)
        lab = torch.empty((self.n_units, T), dtype=torch.int32, device="cuda") if labels else None
        _lib.call("pkv_mine", self._h, side, _ptr(x), T, first,
                  hist.ctypes.data_as(C.POINTER(C.c_double)), nit.ctypes.data_as(C.POINTER(C.c_int32)), _ptr(lab),
                  _stream())
        return (hist, nit, lab) if labels else (hist, nit)

    # ---- reads --------------------------------------------------------------------------
    def decode_attention(self, q: torch.Tensor, sm_scale: float | None = None, out: torch.Tensor | None = None):
        """softmax(q K^T * scale) V per unit over committed + window tokens.
        q: [U, G, D] (G query heads share the unit's KV head) -> out fp32 [U, G, D]."""
        if q.dim() != 3 or q.shape[0] != self.n_units or q.shape[2] != self.head_dim:
            raise UsageError("q must have shape [n_units, G, head_dim]")
        q = q.to(device="cuda", dtype=torch.float32).contiguous()
        if sm_scale is None:
            sm_scale = 1.0 / float(np.sqrt(self.head_dim))
        if out is None:
            out = torch.empty_like(q)
        _lib.call("pkv_decode_attn", self._h, _ptr(q), q.shape[1], C.c_float(sm_scale), _ptr(out), _stream())
        return out

    def decode_attention_partial(self, q: torch.Tensor, blk0: int = 0, blk1: int | None = None,
                                 with_window: bool = True, sm_scale: float | None = None):
        """Unnormalised attention over committed blocks [blk0, blk1) (+ the exact window) for a
        sequence split across ranks: returns (o [U, G, D], m [U, G], l [U, G]) fp32 with
        o = sum_t e^(s_t - m) v_t and l = sum_t e^(s_t - m) (natural-log units); merge the
        ranks' partials with dist.gather_and_merge_partials."""
        if q.dim() != 3 or q.shape[0] != self.n_units or q.shape[2] != self.head_dim:
            raise UsageError("q must have shape [n_units, G, head_dim]")
        q = q.to(device="cuda", dtype=torch.float32).contiguous()
        if sm_scale is None:
            sm_scale = 1.0 / float(np.sqrt(self.head_dim))
        if blk1 is None:
            blk1 = self.info().n_blocks
        o = torch.empty_like(q)
        ml = torch.empty((self.n_units, q.shape[1], 2), dtype=torch.float32, device="cuda")
        _lib.call("pkv_decode_attn_partial", self._h, _ptr(q), q.shape[1], C.c_float(sm_scale), int(blk0), int(blk1),
                  int(bool(with_window)), _ptr(o), _ptr(ml), _stream())
        return o, ml[..., 0], ml[..., 1]

    def fork(self, src_units, dst_units) -> None:
        """Unit dst_units[i] becomes a copy of unit src_units[i] (parallel samples of one prompt)."""
        src = [int(x) for x in src_units]
        dst = [int(x) for x in dst_units]
        if len(src) != len(dst):
            raise UsageError("fork needs as many source as destination units")
        n = len(src)
        _lib.call("pkv_cache_fork", self._h, (C.c_int32 * max(n, 1))(*src), (C.c_int32 * max(n, 1))(*dst), n,
                  _stream())
        if self._npre_dev is not None:
            self.prefill_pattern_counts  # materialise before remapping  # noqa: B018
        nk, nv = (c.copy() for c in self._npre)
        nk[dst], nv[dst] = nk[src], nv[src]
        self._npre = (nk, nv)

    def fork_from(self, src: "PatternKVCache", src_units) -> None:
        """Every unit i of this cache becomes a copy of unit src_units[i] of `src` (parallel
        samples of one prompt: a prompt cache of L x H units -> S x L x H units)."""
        m = [int(x) for x in src_units]
        if len(m) != self.n_units:
            raise UsageError(f"fork_from needs one source unit per destination unit ({self.n_units})")
        _lib.call("pkv_cache_fork_from", self._h, src._h, (C.c_int32 * self.n_units)(*m), _stream())
        nk, nv = src.prefill_pattern_counts
        self._npre_dev = None
        self._npre = (nk[m].copy(), nv[m].copy())
        self._prefill_committed = src._prefill_committed
        self._first_decision = src._first_decision

    def dequant(self, t0: int = 0, t1: int | None = None):
        """Exact fp64 reconstruction of committed tokens [t0, t1): ([U,n,D], [U,n,D])."""
        if t1 is None:
            t1 = self.info().committed_count
        n = max(t1 - t0, 0)
        k = torch.empty((self.n_units, n, self.head_dim), dtype=torch.float64, device="cuda")
        v = torch.empty_like(k)
        _lib.call("pkv_dequant", self._h, t0, t1, _ptr(k), _ptr(v), _stream())
        return k, v

    def codes(self, t0: int = 0, t1: int | None = None):
        """Unpacked integer codes of committed tokens: (K [U,n,D], V [U,n,D]) uint8."""
        if t1 is None:
            t1 = self.info().committed_count
        n = max(t1 - t0, 0)
        k = torch.empty((self.n_units, n, self.head_dim), dtype=torch.uint8, device="cuda")
        v = torch.empty_like(k)
        _lib.call("pkv_export_codes", self._h, t0, t1, _ptr(k), _ptr(v), _stream())
        return k, v

    def pattern_counts(self):
        nk = self.read("nk", torch.int32, (self.n_units,)).cpu().numpy()
        nv = self.read("nv", torch.int32, (self.n_units,)).cpu().numpy()
        return nk, nv

    def pattern_counts_max(self):
        nk, nv = self.pattern_counts()
        return int(nk.max()), int(nv.max())

    def patterns(self, side: int) -> torch.Tensor:
        """fp64 pattern tables [U, Pcap, D] (rows beyond the unit's count are unused)."""
        cap = self.info().pattern_capacity
        return self.read("kpat64" if side == 0 else "vpat64", torch.float64, (self.n_units, cap, self.head_dim))

    def window(self):
        """Exact window rows in order: (K [U, Wn, D], V [U, Wn, D]) in the cache dtype."""
        inf = self.info()
        wcap = self.config.residual_window + self.config.group_size
        wk = self.read("wk", self.dtype, (self.n_units, wcap, self.head_dim))
        wv = self.read("wv", self.dtype, (self.n_units, wcap, self.head_dim))
        idx = (torch.arange(inf.window_len, device="cuda") + inf.window_slot0) % wcap
        return wk[:, idx], wv[:, idx]

    def block_table(self):
        inf = self.info()
        nbcap = self.arena_bytes("blk_len") // 4
        s = self.read("blk_start", torch.int64, (nbcap,)).cpu().numpy()[: inf.n_blocks]
        ln = self.read("blk_len", torch.int32, (nbcap,)).cpu().numpy()[: inf.n_blocks]
        return s, ln
