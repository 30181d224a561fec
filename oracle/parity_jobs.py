"""Process-pool jobs for the BASELINE-config parity tests -- TEST INFRASTRUCTURE ONLY.

Each job regenerates one synthetic unit (oracle.synth_unit, the reference
generator restated) on a host core, rounds it to fp16 as the GPU side does,
runs the oracle restatement of the reference path and returns compact numpy
arrays for the GPU kernels to be compared against.  Only tests/ import this.

Reference lines followed (paths relative to pkg/src/patternkv/):
  mining    patterns.py:72-158 (oracle.kmeans)
  prefill   engine.py:142-169  (oracle.OracleHead.prefill / commit)
  decode    engine.py:172-198  (oracle.OracleHead.append)
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from . import pkv_oracle as O


def unit_inputs(seed: int, tokens: int, d: int = 128):
    """fp16-rounded K/V [tokens, d] (widened to fp64) of unit `seed`."""
    k, v = O.synth_unit(seed, tokens, d)
    return k.astype(np.float16).astype(np.float64), v.astype(np.float16).astype(np.float64)


def _flatten(h: O.OracleHead) -> dict:
    out = {"kpat": np.asarray(h.kpat, np.float64), "vpat": np.asarray(h.vpat, np.float64),
           "tokens": h.tokens, "committed": h.committed}
    if h.k_blocks:
        out["kb_start"] = np.array([b[0] for b in h.k_blocks], np.int64)
        out["kb_len"] = np.array([b[1] for b in h.k_blocks], np.int64)
        out["k_scale"] = np.stack([b[2] for b in h.k_blocks])
        out["k_zero"] = np.stack([b[3] for b in h.k_blocks])
        out["k_codes"] = np.concatenate([b[4] for b in h.k_blocks])
        out["k_idx"] = np.concatenate([b[5] for b in h.k_blocks]).astype(np.int32)
        out["v_scale"] = np.array([x[0] for x in h.v_tok])
        out["v_zero"] = np.array([x[1] for x in h.v_tok])
        out["v_codes"] = np.stack([x[2] for x in h.v_tok])
        out["v_idx"] = np.array([x[3] for x in h.v_tok], np.int64)
        out["vdec"] = np.array([x[2] for x in h.vdec], bool) if h.vdec else np.zeros(0, bool)
    wk, wv = h.window_kv()
    out["window_k"], out["window_v"] = wk, wv
    return out


def unit_job(args):
    """Mine once (K seed, V seed + 1), then prefill + decode for each bit width with
    the same tables.  args = (seed, prefill_tokens, decode_steps, d, pattern_count,
    bits_list, cfg_seed).  Returns {"hist_k", "hist_v", bits: flattened head}."""
    seed, tp, td, d, P, bits_list, cfg_seed = args
    k, v = unit_inputs(seed, tp + td, d)
    kc, lk, hk = O.kmeans(k[:tp], P, cfg_seed)
    vc, lv, hv = O.kmeans(v[:tp], P, cfg_seed + 1)
    res = {"hist_k": np.asarray(hk), "hist_v": np.asarray(hv), "lab_k": lk.astype(np.int32),
           "lab_v": lv.astype(np.int32), "margin_k": stop_margin(hk), "margin_v": stop_margin(hv)}
    for bits in bits_list:
        h = O.OracleHead(O.Knobs(bits=bits, pattern_count=P, seed=cfg_seed), d)
        h.kpat, h.vpat = kc.copy(), vc.copy()
        h.kpat_origin = ["prefill"] * len(kc)
        h.vpat_origin = ["prefill"] * len(vc)
        ncommit = tp - min(tp, h.cfg.residual_window)
        g = h.cfg.group_size
        for s in range(0, ncommit, g):
            h.commit(k[s:min(s + g, ncommit)], v[s:min(s + g, ncommit)], s)
        h.win_k = [r.copy() for r in k[ncommit:tp]]
        h.win_v = [r.copy() for r in v[ncommit:tp]]
        h.tokens = tp
        for t in range(tp, tp + td):
            h.append(k[t], v[t])
        res[bits] = _flatten(h)
    return res


def stop_margin(hist) -> float:
    """How close any round came to the stop rule's threshold (patterns.py:123,
    prev - obj < 1e-6 prev), as |relative improvement - 1e-6| / 1e-6 (SURVEY A.5:
    near-threshold stops are where a last-ulp objective difference could flip the
    iteration count)."""
    m = [abs((hist[i - 1] - hist[i]) / hist[i - 1] - O.KMEANS_TOL) / O.KMEANS_TOL
         for i in range(1, len(hist)) if hist[i - 1] > 0]
    return min(m) if m else math.inf


def run_pool(fn, jobs, workers: int | None = None):
    """Run oracle jobs on host cores (spawned workers: the parent may hold a CUDA context)."""
    workers = max(1, min(len(jobs), workers or os.cpu_count() or 1))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    with ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn")) as ex:
        return list(ex.map(fn, jobs))
