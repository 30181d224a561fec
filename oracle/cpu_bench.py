"""CPU timing of the oracle port (TEST/BENCH INFRASTRUCTURE ONLY).

Used by bench.py's `cpu_baseline` leg and `--impl reference` arm: the
reference's encode path (engine.py:201-252 _commit_span over the prefill
spans, restated in oracle/pkv_oracle.py) timed on host cores, one unit per
worker process (the reference loops units serially, engine.py:411-412; units
are independent).  Mining is excluded, exactly as on the GPU side
(patterns are mined before the timed region).
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from . import pkv_oracle as O


def _encode_unit(args):
    seed, tokens, d, bits, pcount, group, window = args
    k, v = O.synth_unit(seed, tokens, d)
    k = k.astype(np.float16).astype(np.float64)
    v = v.astype(np.float16).astype(np.float64)
    h = O.OracleHead(O.Knobs(bits=bits, pattern_count=pcount, group_size=group, residual_window=window), d)
    h.kpat = O.kmeans(k, pcount, 0)[0]
    h.vpat = O.kmeans(v, pcount, 1)[0]
    ncommit = tokens - min(tokens, window)
    t0 = time.perf_counter()
    for s in range(0, ncommit, group):
        h.commit(k[s:s + group], v[s:s + group], s)
    return ncommit, time.perf_counter() - t0


def encode_throughput(n_units: int, tokens: int, d: int = 128, bits: int = 2, pcount: int = 32,
                      group: int = 128, window: int = 128, workers: int | None = None, seed0: int = 0):
    """Encode n_units independent units on `workers` processes.
    Returns (committed token-units, wall seconds of the encode phase, workers)."""
    workers = workers or os.cpu_count() or 1
    jobs = [(O.unit_seed(seed0, 0, u), tokens, d, bits, pcount, group, window) for u in range(n_units)]
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    with ProcessPoolExecutor(workers) as ex:
        res = list(ex.map(_encode_unit, jobs))
    toks = sum(r[0] for r in res)
    # units run concurrently, `workers` at a time: the aggregate rate is
    # sum(tokens) / (sum(per-unit seconds) / workers)
    busy = sum(r[1] for r in res)
    return toks, busy / min(workers, n_units), min(workers, n_units)
