"""Pattern API (reference patterns.py:25-230) on the B200 kernels.

lloyd_kmeans / mine_patterns -> pkv_kmeans (K2), match_pattern / match_many /
minmax_distance -> pkv_match (IEEE fp64 d_mm, lowest index on ties),
midrange_center -> pkv_midrange.  PatternSet is the append-only host
container the reference exposes (patterns.py:25-60).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cache import _ptr, _stream, first_seed_index, require_cuda
from .errors import DataError, UsageError

ORIGIN_PREFILL = "prefill"
ORIGIN_DECODE = "decode"
KMEANS_MAX_ITERS = 25
KMEANS_REL_TOL = 1e-6


class PatternSet:
    """Append-only collection of pattern vectors of one fixed dimension."""

    def __init__(self, dim: int):
        if dim < 1:
            raise UsageError(f"pattern dimension must be >= 1, got {dim}")
        self.dim = dim
        self._matrix = np.empty((0, dim), dtype=np.float64)
        self._origins: list[str] = []

    def __len__(self) -> int:
        return self._matrix.shape[0]

    @property
    def matrix(self) -> np.ndarray:
        return self._matrix

    def origin(self, index: int) -> str:
        return self._origins[index]

    def vector(self, index: int) -> np.ndarray:
        if not 0 <= index < len(self):
            raise DataError(f"pattern index {index} out of range for set of {len(self)}")
        return self._matrix[index]

    def append(self, vector: np.ndarray, origin: str) -> int:
        vec = np.asarray(vector, dtype=np.float64).ravel()
        if vec.shape != (self.dim,):
            raise UsageError(f"pattern has dimension {vec.size}, set expects {self.dim}")
        if origin not in (ORIGIN_PREFILL, ORIGIN_DECODE):
            raise UsageError(f"unknown pattern origin {origin!r}")
        self._matrix = np.vstack([self._matrix, vec[None, :]])
        self._origins.append(origin)
        return len(self) - 1

    @classmethod
    def from_matrix(cls, matrix: np.ndarray, origins: list[str]) -> "PatternSet":
        ps = cls(matrix.shape[1])
        ps._matrix = np.array(matrix, dtype=np.float64).reshape(-1, matrix.shape[1])
        ps._origins = list(origins)
        return ps


@dataclass(frozen=True)
class PatternMatch:
    pattern_index: int
    residual: np.ndarray
    distance: float


def _as_points(vectors, what: str) -> np.ndarray:
    pts = np.asarray(vectors, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[0] < 1:
        raise UsageError(what)
    return pts


def lloyd_kmeans(vectors: np.ndarray, k: int, seed: int) -> tuple[np.ndarray, np.ndarray, list[float]]:
    """Seeded farthest-point init + Lloyd with empty-cluster repair (patterns.py:72-126) on the GPU."""
    pts = _as_points(vectors, "k-means expects a non-empty 2-D array of row vectors")
    if k < 1:
        raise UsageError(f"cluster count must be >= 1, got {k}")
    if not np.isfinite(pts).all():
        bad = np.argwhere(~np.isfinite(pts))[0]
        raise DataError(f"non-finite vector component at row {bad[0]}, dim {bad[1]}")
    require_cuda()
    T, D = pts.shape
    x = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    cen = torch.zeros((k, D), dtype=torch.float64, device="cuda")
    lab = torch.empty(T, dtype=torch.int32, device="cuda")
    hist = (C.c_double * 25)()
    nh = C.c_int32()
    nc = C.c_int32()
    _lib.call("pkv_kmeans", _ptr(x), T, D, k, first_seed_index(T, seed), _ptr(cen), _ptr(lab), hist, C.byref(nh),
              C.byref(nc), _stream())
    return cen[: nc.value].cpu().numpy(), lab.cpu().numpy().astype(np.int64), [hist[i] for i in range(nh.value)]


def mine_patterns(vectors: np.ndarray, pattern_count: int, seed: int) -> PatternSet:
    """Cluster prefill vectors into at most pattern_count patterns (patterns.py:145-158)."""
    pts = _as_points(vectors, "pattern mining expects a non-empty 2-D array of row vectors")
    centroids, _, _ = lloyd_kmeans(pts, pattern_count, seed)
    return PatternSet.from_matrix(centroids, [ORIGIN_PREFILL] * len(centroids))


def midrange_center(window: np.ndarray) -> np.ndarray:
    """Per-dimension 0.5 * (min + max) (patterns.py:161-171)."""
    win = _as_points(window, "window must be a non-empty 2-D array of row vectors")
    require_cuda()
    x = torch.from_numpy(np.ascontiguousarray(win)).cuda()
    out = torch.empty(win.shape[1], dtype=torch.float64, device="cuda")
    _lib.call("pkv_midrange", _ptr(x), win.shape[0], win.shape[1], _ptr(out), _stream())
    return out.cpu().numpy()


def _match(x: np.ndarray, m: np.ndarray):
    require_cuda()
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    md = torch.from_numpy(np.ascontiguousarray(m, dtype=np.float64)).cuda()
    n, D = x.shape
    idx = torch.empty(n, dtype=torch.int64, device="cuda")
    dist = torch.empty(n, dtype=torch.float64, device="cuda")
    res = torch.empty((n, D), dtype=torch.float64, device="cuda")
    _lib.call("pkv_match", _ptr(xd), n, _ptr(md), m.shape[0], D, _ptr(idx), _ptr(dist), _ptr(res), _stream())
    return idx.cpu().numpy(), res.cpu().numpy(), dist.cpu().numpy()


def minmax_distance(x: np.ndarray, pattern: np.ndarray) -> float:
    """max(x - m) - min(x - m) (patterns.py:174-186)."""
    xv = np.asarray(x, dtype=np.float64)
    mv = np.asarray(pattern, dtype=np.float64)
    if xv.shape != mv.shape:
        raise UsageError(f"dimension mismatch: {xv.shape} vs {mv.shape}")
    return float(_match(xv.reshape(1, -1), mv.reshape(1, -1))[2][0])


def match_pattern(x: np.ndarray, patterns: PatternSet) -> PatternMatch:
    """Nearest pattern under d_mm, lowest index on ties (patterns.py:189-203)."""
    if len(patterns) == 0:
        raise UsageError("cannot match against an empty pattern set")
    vec = np.asarray(x, dtype=np.float64).ravel()
    if vec.shape != (patterns.dim,):
        raise UsageError(f"vector has dimension {vec.size}, patterns expect {patterns.dim}")
    idx, res, dist = _match(vec[None, :], patterns.matrix)
    return PatternMatch(pattern_index=int(idx[0]), residual=res[0].copy(), distance=float(dist[0]))


def match_many(vectors: np.ndarray, patterns: PatternSet) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Batched match_pattern over rows: (indices, residuals, distances) (patterns.py:206-221)."""
    if len(patterns) == 0:
        raise UsageError("cannot match against an empty pattern set")
    pts = np.asarray(vectors, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != patterns.dim:
        raise UsageError(f"expected rows of dimension {patterns.dim}")
    if pts.shape[0] == 0:
        return np.zeros(0, np.int64), np.zeros((0, patterns.dim)), np.zeros(0)
    return _match(pts, patterns.matrix)


def reconstruct_vector(pattern_index: int, patterns: PatternSet, residual: np.ndarray) -> np.ndarray:
    """Pattern + residual (patterns.py:224-230)."""
    base = patterns.vector(pattern_index)
    res = np.asarray(residual, dtype=np.float64).ravel()
    if res.shape != (patterns.dim,):
        raise UsageError(f"residual has dimension {res.size}, patterns expect {patterns.dim}")
    require_cuda()
    return (torch.from_numpy(base.copy()).cuda() + torch.from_numpy(res.copy()).cuda()).cpu().numpy()
