"""Storage accounting closed forms (reference analysis.py:202-245), the
KvStream container the replay harness consumes (reference stream.py:68-124;
the KVTR file format and its GPU ingestion live in trace.py), and the two
host-side analysis checks the verify suites use (variance split, covering
bound; reference analysis.py:21-88, 119-199)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataError, UsageError

SUPPORTED_BITS = (2, 4, 8)


@dataclass(frozen=True)
class VarianceReport:
    """Per-dimension population variances: total = intra + inter (analysis.py:21-34)."""

    total: np.ndarray
    intra: np.ndarray
    inter: np.ndarray
    total_sum: float
    intra_sum: float
    inter_sum: float


def variance_decomposition(vectors: np.ndarray, assignment: np.ndarray, group_count: int | None = None) -> VarianceReport:
    """Law of total variance per dimension with divide-by-N variances (analysis.py:37-87):
    intra = sum_g w_g Var(rows of g), inter = sum_g w_g (mean_g - mean)^2, w_g = n_g / N."""
    pts = np.asarray(vectors, dtype=np.float64)
    lab = np.asarray(assignment)
    if pts.ndim != 2 or pts.shape[0] < 1:
        raise UsageError("variance decomposition expects a non-empty 2-D array")
    if lab.shape != (pts.shape[0],):
        raise UsageError("assignment must provide exactly one group id per vector")
    if not np.issubdtype(lab.dtype, np.integer):
        raise UsageError("assignment ids must be integers")
    k = int(lab.max()) + 1 if group_count is None else group_count
    out_of_range = (lab < 0) | (lab >= k)
    if out_of_range.any():
        row = int(np.argmax(out_of_range))
        raise UsageError(f"assignment id {lab[row]} at row {row} outside [0, {k})")
    n = pts.shape[0]
    mean = pts.mean(axis=0)
    total = ((pts - mean) ** 2).mean(axis=0)
    intra = np.zeros(pts.shape[1])
    inter = np.zeros(pts.shape[1])
    for grp in range(k):
        rows = pts[lab == grp]
        if rows.shape[0]:
            w = rows.shape[0] / n
            mu = rows.mean(axis=0)
            intra += w * ((rows - mu) ** 2).mean(axis=0)
            inter += w * (mu - mean) ** 2
    return VarianceReport(total, intra, inter, float(total.sum()), float(intra.sum()), float(inter.sum()))


@dataclass(frozen=True)
class CoveringReport:
    """Residual-range covering check (analysis.py:119-134)."""

    r_w_star: float
    epsilon: float
    epsilon_net_size: int
    net_size_estimate: float
    u_raw: float
    u_res: float
    bound_holds: bool


def covering_bound_check(points: np.ndarray, rho: float, bits: int) -> CoveringReport:
    """Grid net at radius eps = rho R_w* and the contraction u_res <= rho u_raw it implies
    (analysis.py:137-199).  R_w* = half the largest min-max width of the points around the
    per-dimension midrange; net points are centres of 2 eps cells over the bounding box."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[0] < 1:
        raise UsageError("covering check expects a non-empty 2-D array of row vectors")
    if not 0.0 < rho < 1.0:
        raise UsageError(f"rho must lie in (0, 1), got {rho}")
    if bits not in SUPPORTED_BITS:
        raise UsageError(f"unsupported bit width {bits}; expected one of {SUPPORTED_BITS}")
    if not np.isfinite(pts).all():
        raise DataError("covering check requires finite points")
    qmax = (1 << bits) - 1
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    res = pts - 0.5 * (lo + hi)
    r_w = 0.5 * float((res.max(axis=1) - res.min(axis=1)).max())
    eps = rho * r_w
    if eps == 0.0:  # every point on one diagonal line: each is its own net point
        n = int(np.unique(pts, axis=0).shape[0])
        return CoveringReport(0.0, 0.0, n, float(n), 0.0, 0.0, True)
    cells_per_dim = np.maximum(1, np.ceil((hi - lo) / (2.0 * eps)).astype(np.int64))
    cell = np.clip(np.floor((pts - lo) / (2.0 * eps)).astype(np.int64), 0, cells_per_dim - 1)
    snapped = pts - (lo + (2.0 * cell + 1.0) * eps)
    u_raw = r_w / qmax
    u_res = 0.5 * float((snapped.max(axis=1) - snapped.min(axis=1)).max()) / qmax
    r_inf = float(np.abs(pts).max())
    return CoveringReport(r_w, eps, int(np.prod(cells_per_dim)), float((1.0 + 2.0 * r_inf / eps) ** pts.shape[1]),
                          u_raw, u_res, bool(u_res <= rho * u_raw))


def bits_per_token(config, head_dim: int, pattern_set_size: int, token_count: int, side: str) -> float:
    """codes + amortized group params + 16-bit index + amortized 16-bit patterns (analysis.py:202-237)."""
    if side not in ("k", "v"):
        raise UsageError(f"side must be 'k' or 'v', got {side!r}")
    if head_dim < 1 or token_count < 1 or pattern_set_size < 0:
        raise UsageError("head_dim and token_count must be >= 1, pattern_set_size >= 0")
    uses = config.use_k_patterns if side == "k" else config.use_v_patterns
    codes = config.bits * head_dim
    params = 32.0 * head_dim / config.group_size if side == "k" else 32.0
    index = 16.0 if uses else 0.0
    patterns = 16.0 * head_dim * pattern_set_size / token_count
    return codes + params + index + patterns


def fp16_reference_bits_per_token(head_dim: int) -> float:
    if head_dim < 1:
        raise UsageError(f"head_dim must be >= 1, got {head_dim}")
    return 16.0 * head_dim


@dataclass
class KvStream:
    """prefill_k/v [L, H, T, d], decode_k/v [L, H, S, d] (stream.py:68-124)."""

    prefill_k: np.ndarray
    prefill_v: np.ndarray
    decode_k: np.ndarray
    decode_v: np.ndarray
    token_ids: np.ndarray | None = None
    v_cluster_ids: np.ndarray | None = None

    def __post_init__(self) -> None:
        for name in ("prefill_k", "prefill_v", "decode_k", "decode_v"):
            arr = np.asarray(getattr(self, name))
            if arr.ndim != 4:
                raise UsageError(f"{name} must be 4-D (layers, heads, tokens, dim)")
            setattr(self, name, arr)
        if self.prefill_k.shape != self.prefill_v.shape or self.decode_k.shape != self.decode_v.shape:
            raise UsageError("K and V tensors must have matching shapes")
        pk, dk = self.prefill_k.shape, self.decode_k.shape
        if (dk[0], dk[1], dk[3]) != (pk[0], pk[1], pk[3]):
            raise UsageError("decode tensors must match prefill layers/heads/dim")
        if self.prefill_k.shape[2] < 1:
            raise UsageError("prefill length must be >= 1")

    @property
    def num_layers(self) -> int:
        return self.prefill_k.shape[0]

    @property
    def num_heads(self) -> int:
        return self.prefill_k.shape[1]

    @property
    def prefill_len(self) -> int:
        return self.prefill_k.shape[2]

    @property
    def decode_steps(self) -> int:
        return self.decode_k.shape[2]

    @property
    def head_dim(self) -> int:
        return self.prefill_k.shape[3]

    def head_slices(self, layer: int, head: int):
        return (self.prefill_k[layer, head], self.prefill_v[layer, head],
                self.decode_k[layer, head], self.decode_v[layer, head])
