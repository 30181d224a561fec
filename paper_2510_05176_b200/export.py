"""Export of a GPU cache unit into the reference's HeadCacheState shapes
(engine.py:86-129): pattern tables, K blocks (per-channel groups), V tokens,
gate decisions and the exact window.  Used by the per-head facade
(engine.py in this package), the replay harness and the parity tests.

Codes leave the device unpacked (fragment layout decoded by a kernel) and are
re-packed into the reference byte layout (quant.py:120-146) on the device by
pkv_pack_codes.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cache import PatternKVCache, _ptr, _stream


def _arena(cache: PatternKVCache, name: str, dtype: torch.dtype, inner: tuple) -> torch.Tensor:
    nbytes = cache.arena_bytes(name)
    esz = torch.empty((), dtype=dtype).element_size()
    n = nbytes // esz
    out = torch.empty(n, dtype=dtype, device="cuda")
    _lib.call("pkv_cache_read", cache._h, name.encode(), 0, n * esz, _ptr(out), _stream())
    per_unit = n // cache.n_units
    return out.view(cache.n_units, per_unit)


def pack_rows(codes: torch.Tensor, bits: int) -> torch.Tensor:
    """Pack each row of a uint8 code matrix [R, L] into ceil(L*bits/8) bytes,
    rows concatenated (reference pack_codes per group)."""
    codes = codes.contiguous()
    R, L = codes.shape
    per = 8 // bits
    Lp = -(-L // per) * per
    if Lp != L:
        pad = torch.zeros((R, Lp - L), dtype=torch.uint8, device=codes.device)
        codes = torch.cat([codes, pad], dim=1).contiguous()
    out = torch.empty(R * Lp // per, dtype=torch.uint8, device=codes.device)
    _lib.call("pkv_pack_codes", _ptr(codes), codes.numel(), bits, _ptr(out), _stream())
    return out.view(R, Lp // per)


@dataclass
class UnitState:
    kpat: np.ndarray
    vpat: np.ndarray
    n_prefill_k: int
    n_prefill_v: int
    kb_start: np.ndarray
    kb_len: np.ndarray
    k_scale: np.ndarray     # [nb, D]
    k_zero: np.ndarray      # [nb, D]
    k_codes: np.ndarray     # [C, D] uint8
    k_idx: np.ndarray       # [C] int32
    v_scale: np.ndarray     # [C]
    v_zero: np.ndarray      # [C]
    v_codes: np.ndarray     # [C, D] uint8
    v_idx: np.ndarray       # [C]
    vdec: np.ndarray        # [n, 3] raw, flat, flatten
    kdec: np.ndarray        # [n, 3]
    window_k: np.ndarray
    window_v: np.ndarray
    token_count: int
    k_bytes: list           # per block: [D] bytes objects (reference layout)
    v_bytes: list           # per token bytes


def export_unit(cache: PatternKVCache, u: int, with_bytes: bool = True) -> UnitState:
    cfg = cache.config
    inf = cache.info()
    D = cache.head_dim
    Cn = inf.committed_count
    nk, nv = cache.pattern_counts()
    npre_k, npre_v = cache.prefill_pattern_counts
    kpat = cache.patterns(0)[u, : nk[u]].cpu().numpy() if cfg.use_k_patterns else np.zeros((0, D))
    vpat = cache.patterns(1)[u, : nv[u]].cpu().numpy() if cfg.use_v_patterns else np.zeros((0, D))
    kb_start, kb_len = cache.block_table()
    nb = len(kb_start)
    kp = _arena(cache, "kparam64", torch.float64, ()).view(cache.n_units, -1, 2, D)[u, :nb].cpu().numpy()
    vp = _arena(cache, "vparam64", torch.float64, ()).view(cache.n_units, -1, 2)[u, :Cn].cpu().numpy()
    gp = 16 * ((cfg.group_size + 15) // 16)
    slots = np.concatenate([b * gp + np.arange(int(n)) for b, n in enumerate(kb_len)]) if nb else np.zeros(0, np.int64)
    kidx = _arena(cache, "kidx", torch.int16, ())[u].cpu().numpy()[slots].astype(np.int32)
    vidx = _arena(cache, "vidx", torch.int16, ())[u].cpu().numpy()[slots].astype(np.int64)
    kc, vc = cache.codes(0, Cn)
    kc_u, vc_u = kc[u], vc[u]
    vdec = np.zeros((0, 3))
    kdec = np.zeros((0, 3))
    if cache.record_decisions:
        f0 = cache.first_decision_token
        if cfg.use_v_patterns:
            vd = _arena(cache, "vdiag", torch.float64, ()).view(cache.n_units, -1, 2)[u, f0:Cn].cpu().numpy()
            fl = (vidx[f0:Cn] != -1).astype(np.float64)
            vdec = np.concatenate([vd, fl[:, None]], axis=1)
        if cfg.use_k_patterns and cfg.use_k_gate:
            kd = _arena(cache, "kdiag", torch.float64, ()).view(cache.n_units, -1, 2)[u, f0:Cn].cpu().numpy()
            fl = (kidx[f0:Cn] != -1).astype(np.float64)
            kdec = np.concatenate([kd, fl[:, None]], axis=1)
    wk, wv = cache.window()
    k_bytes, v_bytes = [], []
    if with_bytes and Cn > 0:
        for b in range(nb):
            s, n = int(kb_start[b]), int(kb_len[b])
            rows = pack_rows(kc_u[s:s + n].t(), cfg.bits).cpu().numpy()
            k_bytes.append([rows[c].tobytes() for c in range(D)])
        vrows = pack_rows(vc_u, cfg.bits).cpu().numpy()
        v_bytes = [vrows[t].tobytes() for t in range(Cn)]
    return UnitState(
        kpat=kpat, vpat=vpat, n_prefill_k=int(npre_k[u]), n_prefill_v=int(npre_v[u]),
        kb_start=np.asarray(kb_start, np.int64), kb_len=np.asarray(kb_len, np.int64),
        k_scale=kp[:, 0, :], k_zero=kp[:, 1, :], k_codes=kc_u.cpu().numpy(), k_idx=kidx,
        v_scale=vp[:, 0], v_zero=vp[:, 1], v_codes=vc_u.cpu().numpy(), v_idx=vidx,
        vdec=vdec, kdec=kdec,
        window_k=wk[u].double().cpu().numpy(), window_v=wv[u].double().cpu().numpy(),
        token_count=inf.token_count, k_bytes=k_bytes, v_bytes=v_bytes,
    )
