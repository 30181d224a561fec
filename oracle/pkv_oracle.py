"""CPU oracle for the PatternKV codec hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference's per-head codec
(``/root/reference/pkg/src/patternkv``) used as the *checker* for the
B200 kernels.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
it.  The product package never imports, links or calls anything here.

Pinning: every function below is checked against golden vectors that
``tests/golden/make_golden.py`` produced by importing the reference
itself (see ``tests/test_oracle_golden.py``), plus the reference test
suite's known-answer values.

All arithmetic is float64 with the reference's operation order; each
function cites the reference lines it restates (paths relative to
``pkg/src/patternkv/``).
"""

from __future__ import annotations

import math

import numpy as np

RAW = -1  # engine.py:35 RAW_MARKER
KMEANS_ITERS = 25  # patterns.py:21
KMEANS_TOL = 1e-6  # patterns.py:22


class OracleUsage(ValueError):
    """Caller error (reference errors.py:9 UsageError)."""


class OracleData(ValueError):
    """Bad data (reference errors.py:13 DataError)."""


# --------------------------------------------------------------------------
# quantizer (quant.py:70-179)
# --------------------------------------------------------------------------

def quantize(values, bits):
    """(scale, zero, codes[uint8]) -- quant.py:70-111.

    zero = min, scale = (max-min)/(2^b-1) by one IEEE division, codes =
    clip(floor((v-lo)/scale + 0.5), 0, qmax); scale == 0 gives all zeros.
    """
    if bits not in (2, 4, 8):
        raise OracleUsage(f"bits {bits}")
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    if v.size == 0:
        raise OracleUsage("empty group")
    bad = ~np.isfinite(v)
    if bad.any():
        raise OracleData(f"non-finite value at index {int(np.argmax(bad))}")
    qmax = (1 << bits) - 1
    lo = float(v.min())
    scale = (float(v.max()) - lo) / qmax
    if scale == 0.0:
        return scale, lo, np.zeros(v.size, np.uint8)
    q = np.floor((v - lo) / scale + 0.5)
    return scale, lo, np.clip(q, 0, qmax).astype(np.uint8)


def dequantize(scale, zero, codes):
    """scale * code + zero in float64 -- quant.py:114-117."""
    return scale * np.asarray(codes).astype(np.float64) + zero


def pack(codes, bits):
    """Little-endian within a byte, first code in the low bits -- quant.py:120-146."""
    c = np.asarray(codes, dtype=np.int64).reshape(-1)
    if c.size == 0:
        return b""
    per = 8 // bits
    nbytes = -(-c.size // per)
    buf = np.zeros(nbytes * per, np.int64)
    buf[: c.size] = c
    buf = buf.reshape(nbytes, per) << (np.arange(per) * bits)
    return buf.sum(axis=1).astype(np.uint8).tobytes()


def unpack(data, length, bits):
    """Inverse of pack -- quant.py:149-179."""
    if len(data) != (length * bits + 7) // 8:
        raise OracleData("packed byte count mismatch")
    per = 8 // bits
    raw = np.frombuffer(bytes(data), np.uint8).astype(np.int64)
    c = (raw[:, None] >> (np.arange(per) * bits)) & ((1 << bits) - 1)
    return c.reshape(-1)[:length].astype(np.uint8)


# --------------------------------------------------------------------------
# patterns (patterns.py:72-230)
# --------------------------------------------------------------------------

def minmax_match(x, pats):
    """Nearest pattern under d_mm(x,m) = max(x-m) - min(x-m), lowest index
    on ties (np.argmin) -- patterns.py:206-221.  Returns (idx, residual, dist)."""
    x = np.asarray(x, dtype=np.float64)
    m = np.asarray(pats, dtype=np.float64)
    r = x[:, None, :] - m[None, :, :]
    d = r.max(axis=2) - r.min(axis=2)
    i = np.argmin(d, axis=1)
    rows = np.arange(x.shape[0])
    return i, r[rows, i], d[rows, i]


def _sqd(pts, cen):
    # patterns.py:129-131 (einsum keeps the reference's reduction order on this CPU)
    diff = pts[:, None, :] - cen[None, :, :]
    return np.einsum("ijk,ijk->ij", diff, diff)


def first_seed_index(n_points, seed):
    """patterns.py:103/135: the first center index from numpy PCG64."""
    return int(np.random.default_rng(seed).integers(n_points))


def kmeans(points, k, seed):
    """Seeded farthest-point init + Lloyd -- patterns.py:72-126, 134-142.

    Returns (centers, labels, history)."""
    x = np.asarray(points, dtype=np.float64)
    uniq = np.unique(x, axis=0)
    if uniq.shape[0] <= k:  # patterns.py:95-101 distinct-rows shortcut
        return uniq, np.argmin(_sqd(x, uniq), axis=1), [0.0]
    n = x.shape[0]
    picks = [first_seed_index(n, seed)]
    near = _sqd(x, x[picks[0]][None])[:, 0]
    while len(picks) < k:
        j = int(np.argmax(near))
        picks.append(j)
        near = np.minimum(near, _sqd(x, x[j][None])[:, 0])
    cen = x[picks].copy()
    hist = []
    prev = math.inf
    for _ in range(KMEANS_ITERS):
        d2 = _sqd(x, cen)
        lab = np.argmin(d2, axis=1)
        own = d2[np.arange(n), lab]
        for e in np.setdiff1d(np.arange(k), lab):  # patterns.py:112-118 empty repair
            cnt = np.bincount(lab, minlength=k)
            far = int(np.argmax(np.where(cnt[lab] > 1, own, -1.0)))
            lab[far] = e
            cen[e] = x[far]
            own[far] = 0.0
        for j in range(k):
            cen[j] = x[lab == j].mean(axis=0)
        obj = float(_sqd(x, cen)[np.arange(n), lab].sum())
        hist.append(obj)
        if obj == 0.0 or (math.isfinite(prev) and prev - obj < KMEANS_TOL * prev):
            break
        prev = obj
    return cen, lab, hist


def midrange(rows):
    """0.5 * (min + max) per dimension -- patterns.py:161-171."""
    w = np.asarray(rows, dtype=np.float64)
    return 0.5 * (w.min(axis=0) + w.max(axis=0))


# --------------------------------------------------------------------------
# gate (gate.py:23-188)
# --------------------------------------------------------------------------

_A = (3.3871328727963666080e0, 1.3314166789178437745e2, 1.9715909503065514427e3, 1.3731693765509461125e4,
      4.5921953931549871457e4, 6.7265770927008700853e4, 3.3430575583588128105e4, 2.5090809287301226727e3)
_B = (1.0, 4.2313330701600911252e1, 6.8718700749205790830e2, 5.3941960214247511077e3,
      2.1213794301586595867e4, 3.9307895800092710610e4, 2.8729085735721942674e4, 5.2264952788528545610e3)
_C = (1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0, 3.64784832476320460504e0,
      1.27045825245236838258e0, 2.41780725177450611770e-1, 2.27238449892691845833e-2, 7.74545014278341407640e-4)
_D = (1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
      1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4, 1.05075007164441684324e-9)
_E = (6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0, 2.96560571828504891230e-1,
      2.65321895265761230930e-2, 1.24266094738807843860e-3, 2.71155556874348757815e-5, 2.01033439929228813265e-7)
_F = (1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
      7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7, 2.04426310338993978564e-15)


def _horner(coef, r):
    acc = coef[-1]
    for c in reversed(coef[:-1]):
        acc = acc * r + c
    return acc


def z_quantile(alpha):
    """Upper alpha point of N(0,1), Wichura AS241 -- gate.py:23-71."""
    if not 0.0 < alpha <= 0.5:
        raise OracleUsage("alpha")
    q = alpha - 0.5
    if abs(q) <= 0.425:
        r = 0.180625 - q * q
        return -(q * _horner(_A, r) / _horner(_B, r))
    r = math.sqrt(-math.log(alpha if q < 0 else 1.0 - alpha))
    if r <= 5.0:
        r -= 1.6
        z = _horner(_C, r) / _horner(_D, r)
    else:
        r -= 5.0
        z = _horner(_E, r) / _horner(_F, r)
    return z if q < 0 else -z


def threshold(head_dim, alpha):
    """Root of 1-rho^2 = (2z/sqrt(5d)) sqrt(1+rho^4) by bisection to 1e-12 -- gate.py:74-106."""
    z = z_quantile(alpha)
    if z <= 0.0:
        return 1.0
    c = 2.0 * z / math.sqrt(5.0 * head_dim)
    if c >= 1.0:
        raise OracleUsage("no significant ratio")
    lo, hi = 0.0, 1.0
    while hi - lo > 1e-12:
        mid = 0.5 * (lo + hi)
        if (1.0 - mid * mid) - c * math.sqrt(1.0 + mid ** 4) >= 0.0:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def flatten_decision(raw_range, flat_range, thr):
    """gate.py:174-188: flatten iff raw > 0 and flat/raw <= thr."""
    if raw_range == 0.0:
        return False, math.inf
    ratio = flat_range / raw_range
    return ratio <= thr, ratio


# --------------------------------------------------------------------------
# per-head engine (engine.py:38-333)
# --------------------------------------------------------------------------

class Knobs:
    """EngineConfig field-for-field (engine.py:50-60)."""

    def __init__(self, bits=2, pattern_count=32, group_size=128, residual_window=128, alpha=0.05,
                 use_k_patterns=True, use_v_patterns=True, generate_new_patterns=True,
                 use_v_gate=True, use_k_gate=False, seed=0):
        self.bits = bits
        self.pattern_count = pattern_count
        self.group_size = group_size
        self.residual_window = residual_window
        self.alpha = alpha
        self.use_k_patterns = use_k_patterns
        self.use_v_patterns = use_v_patterns
        self.generate_new_patterns = generate_new_patterns
        self.use_v_gate = use_v_gate
        self.use_k_gate = use_k_gate
        self.seed = seed


class OracleHead:
    """One head's cache, held as flat numpy arrays (engine.py:104-129).

    k_blocks: list of (start, length, scales[d], zeros[d], codes[length, d], idx[length])
    v_tok:    list of (scale, zero, codes[d], idx)
    vdec/kdec: list of (raw_range, flat_range, flatten)
    """

    def __init__(self, knobs, d):
        self.cfg = knobs
        self.d = d
        self.kpat = np.zeros((0, d))
        self.vpat = np.zeros((0, d))
        self.kpat_origin = []
        self.vpat_origin = []
        self.k_blocks = []
        self.v_tok = []
        self.win_k = []
        self.win_v = []
        self.tokens = 0
        self.vdec = []
        self.kdec = []
        self.thr = threshold(d, knobs.alpha)

    @property
    def committed(self):
        return self.tokens - len(self.win_k)

    # engine.py:142-169
    def prefill(self, k, v):
        k = np.asarray(k, np.float64)
        v = np.asarray(v, np.float64)
        cfg = self.cfg
        if cfg.use_k_patterns:
            self.kpat = kmeans(k, cfg.pattern_count, cfg.seed)[0]
            self.kpat_origin = ["prefill"] * len(self.kpat)
        if cfg.use_v_patterns:
            self.vpat = kmeans(v, cfg.pattern_count, cfg.seed + 1)[0]
            self.vpat_origin = ["prefill"] * len(self.vpat)
        n = k.shape[0]
        ncommit = n - min(n, cfg.residual_window)
        for s in range(0, ncommit, cfg.group_size):
            e = min(s + cfg.group_size, ncommit)
            self.commit(k[s:e], v[s:e], s)
        self.win_k = [r.copy() for r in k[ncommit:]]
        self.win_v = [r.copy() for r in v[ncommit:]]
        self.tokens = n
        return self

    # engine.py:172-198
    def append(self, kv, vv):
        cfg = self.cfg
        self.win_k.append(np.asarray(kv, np.float64).copy())
        self.win_v.append(np.asarray(vv, np.float64).copy())
        self.tokens += 1
        g = cfg.group_size
        if len(self.win_k) == cfg.residual_window + g:
            ks = np.stack(self.win_k[:g])
            vs = np.stack(self.win_v[:g])
            if cfg.generate_new_patterns:
                if cfg.use_k_patterns:
                    self.kpat = np.vstack([self.kpat, midrange(ks)[None]])
                    self.kpat_origin.append("decode")
                if cfg.use_v_patterns:
                    self.vpat = np.vstack([self.vpat, midrange(vs)[None]])
                    self.vpat_origin.append("decode")
            self.commit(ks, vs, self.committed)
            del self.win_k[:g]
            del self.win_v[:g]
        return self

    # engine.py:201-252
    def commit(self, ks, vs, start):
        cfg = self.cfg
        n = ks.shape[0]
        kidx = np.full(n, RAW, np.int32)
        keff = ks.copy()
        if cfg.use_k_patterns and len(self.kpat):
            i, res, dist = minmax_match(ks, self.kpat)
            if cfg.use_k_gate:
                raw = ks.max(axis=1) - ks.min(axis=1)
                for t in range(n):
                    fl, _ = flatten_decision(float(raw[t]), float(dist[t]), self.thr)
                    self.kdec.append((float(raw[t]), float(dist[t]), fl))
                    if fl:
                        kidx[t] = i[t]
                        keff[t] = res[t]
            else:
                kidx[:] = i
                keff = res
        sc = np.empty(self.d)
        ze = np.empty(self.d)
        codes = np.empty((n, self.d), np.uint8)
        for c in range(self.d):
            sc[c], ze[c], codes[:, c] = quantize(keff[:, c], cfg.bits)
        self.k_blocks.append((start, n, sc, ze, codes, kidx))

        if cfg.use_v_patterns and len(self.vpat):
            i, res, dist = minmax_match(vs, self.vpat)
            raw = vs.max(axis=1) - vs.min(axis=1)
            for t in range(n):
                if cfg.use_v_gate:
                    fl, _ = flatten_decision(float(raw[t]), float(dist[t]), self.thr)
                else:
                    fl = True
                self.vdec.append((float(raw[t]), float(dist[t]), fl))
                row, j = (res[t], int(i[t])) if fl else (vs[t], RAW)
                s, z, cd = quantize(row, cfg.bits)
                self.v_tok.append((s, z, cd, j))
        else:
            for t in range(n):
                s, z, cd = quantize(vs[t], cfg.bits)
                self.v_tok.append((s, z, cd, RAW))

    # engine.py:255-268, 296-303
    def committed_kv(self):
        if self.committed == 0:
            return np.zeros((0, self.d)), np.zeros((0, self.d))
        kk = []
        for (_, n, sc, ze, codes, idx) in self.k_blocks:
            m = sc[None, :] * codes.astype(np.float64) + ze[None, :]
            for t in range(n):
                if idx[t] != RAW:
                    m[t] += self.kpat[idx[t]]
            kk.append(m)
        vv = []
        for (s, z, cd, j) in self.v_tok:
            row = s * cd.astype(np.float64) + z
            if j != RAW:
                row = row + self.vpat[j]
            vv.append(row)
        return np.concatenate(kk, axis=0), np.stack(vv)

    def window_kv(self):
        if not self.win_k:
            return np.zeros((0, self.d)), np.zeros((0, self.d))
        return np.stack(self.win_k), np.stack(self.win_v)

    def k_block_ref_bytes(self, b):
        """Reference packed layout of K block b: list of d byte strings (engine.py:222)."""
        (_, n, _, _, codes, _) = self.k_blocks[b]
        return [pack(codes[:, c], self.cfg.bits) for c in range(self.d)]


def replay(kp, vp, kd, vd, knobs):
    """engine.py:369-380."""
    h = OracleHead(knobs, kp.shape[1]).prefill(kp, vp)
    for t in range(kd.shape[0]):
        h.append(kd[t], vd[t])
    return h


# --------------------------------------------------------------------------
# decode attention: absent from the reference; defined here
# as fp64 softmax attention over the reconstructed cache (engine.py:296-303)
# plus the exact residual window, GQA mapping q_head // (Hq / Hkv).
# --------------------------------------------------------------------------

def attention(q, k_all, v_all, sm_scale):
    """q [G, d], k_all/v_all [n, d] -> out [G, d] (float64)."""
    q = np.asarray(q, np.float64)
    s = (q @ np.asarray(k_all, np.float64).T) * sm_scale
    s = s - s.max(axis=1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=1, keepdims=True)
    return p @ np.asarray(v_all, np.float64)


def head_attention(head, q, sm_scale):
    kc, vc = head.committed_kv()
    kw, vw = head.window_kv()
    return attention(q, np.concatenate([kc, kw]), np.concatenate([vc, vw]), sm_scale)


# --------------------------------------------------------------------------
# synthetic KV generator (analysis.py:321-370), one (layer, head) unit per seed
# --------------------------------------------------------------------------

def synth_unit(seed, tokens, d, outlier=((3, 32.0),), drift=None, noise=0.05,
               clusters=32, spread=5.0, within=0.2, consistency=0.9, vocab=1024):
    """K/V [tokens, d] float64 for one unit, same draw order as the reference
    generator with layers=heads=1 (analysis.py:329-362)."""
    rng = np.random.default_rng(seed)
    if drift is None:
        drift = 1.0 / tokens
    tok = rng.integers(0, vocab, size=tokens)
    a = np.clip(np.arange(tokens) * drift, 0.0, 1.0)[:, None]
    p0 = rng.uniform(0.5, 1.5, size=d) * (rng.integers(0, 2, size=d) * 2 - 1)
    p1 = rng.uniform(0.5, 1.5, size=d) * (rng.integers(0, 2, size=d) * 2 - 1)
    for ch, mul in outlier:
        p0[ch] *= mul
        p1[ch] *= mul
    k = (1.0 - a) * p0[None, :] + a * p1[None, :]
    if noise > 0:
        k = k + rng.normal(0.0, noise, size=(tokens, d))
    cen = rng.normal(0.0, spread, size=(clusters, d))
    home = rng.integers(0, clusters, size=vocab)
    stray = rng.integers(0, clusters, size=tokens)
    keep = rng.random(tokens) <= consistency
    cl = np.where(keep, home[tok], stray)
    v = cen[cl]
    if within > 0:
        v = v + rng.normal(0.0, within, size=(tokens, d))
    return k, v


def unit_seed(b, layer, head):
    """Documented per-unit seed."""
    return 1_000_003 * b + 1_009 * layer + head
