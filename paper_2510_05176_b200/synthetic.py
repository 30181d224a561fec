"""Host-side synthetic KV streams and stream diagnostics of the drop-in API
(reference analysis.py:91-118 and 248-470): the KeyModel / ValueModel generator,
its flat `key = value` spec format, the consistency metric and the key-channel
statistics.  Not on the codec's hot path (the throughput benches draw the same
model family on the device, synth.py); kept so reference callers of
generate_synthetic_stream / parse_stream_spec keep working and so the parity
inputs can be regenerated from a seed.

The draw order of numpy's PCG64 stream is part of the contract (a seed names a
stream): token ids first, then per (layer, head): profile p0 (uniform
magnitudes, random signs), profile p1, key noise, value centers, home clusters,
stray clusters, the consistency coin, value noise (analysis.py:321-370).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .analysis import KvStream
from .errors import UsageError


@dataclass(frozen=True)
class KeyModel:
    """Keys: a per-head channel profile (outlier channels scaled up) drifting linearly
    from profile p0 to p1 at drift_rate per token, plus i.i.d. Gaussian noise."""

    outlier_channels: tuple[int, ...] = ()
    outlier_multipliers: tuple[float, ...] = ()
    drift_rate: float = 0.0
    noise_std: float = 0.0


@dataclass(frozen=True)
class ValueModel:
    """Values: Gaussian clusters; each token id has a home cluster it uses with
    probability `consistency`, otherwise a random cluster for that occurrence."""

    cluster_count: int = 8
    center_spread: float = 5.0
    within_std: float = 0.2
    consistency: float = 1.0
    vocab_size: int = 64


@dataclass(frozen=True)
class SyntheticStreamSpec:
    layers: int = 1
    heads: int = 1
    head_dim: int = 64
    prefill_len: int = 256
    decode_len: int = 256
    k_model: KeyModel = field(default_factory=KeyModel)
    v_model: ValueModel = field(default_factory=ValueModel)
    seed: int = 0


DEFAULT_STREAM_SPEC = SyntheticStreamSpec(
    layers=2, heads=2, head_dim=64, prefill_len=512, decode_len=512,
    k_model=KeyModel(outlier_channels=(3,), outlier_multipliers=(32.0,), drift_rate=1e-3, noise_std=0.05),
    v_model=ValueModel(cluster_count=8, center_spread=5.0, within_std=0.2, consistency=0.9, vocab_size=64),
)


def _check_spec(spec: SyntheticStreamSpec) -> None:
    km, vm = spec.k_model, spec.v_model
    problems = [
        (min(spec.layers, spec.heads, spec.head_dim) < 1, "layers, heads and head_dim must all be >= 1"),
        (spec.prefill_len < 1 or spec.decode_len < 0, "prefill_len must be >= 1 and decode_len >= 0"),
        (len(km.outlier_channels) != len(km.outlier_multipliers),
         "outlier_channels and outlier_multipliers must have equal length"),
        (any(c < 0 or c >= spec.head_dim for c in km.outlier_channels), "outlier channel index outside head_dim"),
        (km.noise_std < 0 or km.drift_rate < 0, "key noise_std and drift_rate must be non-negative"),
        (vm.cluster_count < 1 or vm.vocab_size < 1, "cluster_count and vocab_size must be >= 1"),
        (vm.within_std < 0 or vm.center_spread < 0, "value spreads must be non-negative"),
        (not (0.0 <= vm.consistency <= 1.0), "consistency must lie in [0, 1]"),
    ]
    for bad, msg in problems:
        if bad:
            raise UsageError(msg)


def _signed_profile(rng: np.random.Generator, d: int) -> np.ndarray:
    mags = rng.uniform(0.5, 1.5, size=d)
    signs = rng.integers(0, 2, size=d) * 2 - 1
    return mags * signs


def _one_head(rng, km: KeyModel, vm: ValueModel, alpha: np.ndarray, token_ids: np.ndarray, total: int, d: int):
    """(keys [total, d], values [total, d], clusters [total]) of one (layer, head)."""
    ends = [_signed_profile(rng, d), _signed_profile(rng, d)]
    for p in ends:
        for ch, mult in zip(km.outlier_channels, km.outlier_multipliers):
            p[ch] *= mult
    keys = ends[0][None, :] * (1.0 - alpha) + ends[1][None, :] * alpha
    if km.noise_std > 0:
        keys = keys + rng.normal(0.0, km.noise_std, size=(total, d))
    centers = rng.normal(0.0, vm.center_spread, size=(vm.cluster_count, d))
    home = rng.integers(0, vm.cluster_count, size=vm.vocab_size)
    stray = rng.integers(0, vm.cluster_count, size=total)
    loyal = rng.random(total) <= vm.consistency
    clusters = np.where(loyal, home[token_ids], stray)
    values = centers[clusters]
    if vm.within_std > 0:
        values = values + rng.normal(0.0, vm.within_std, size=(total, d))
    return keys, values, clusters


def generate_synthetic_stream(spec: SyntheticStreamSpec) -> KvStream:
    """Deterministic KV stream of the spec's seed (reference analysis.py:321-370);
    carries token_ids and per-head v_cluster_ids for the consistency metric."""
    _check_spec(spec)
    rng = np.random.default_rng(spec.seed)
    n_l, n_h, d = spec.layers, spec.heads, spec.head_dim
    total = spec.prefill_len + spec.decode_len
    token_ids = rng.integers(0, spec.v_model.vocab_size, size=total)
    alpha = np.clip(np.arange(total) * spec.k_model.drift_rate, 0.0, 1.0)[:, None]
    keys = np.empty((n_l, n_h, total, d))
    values = np.empty((n_l, n_h, total, d))
    clusters = np.empty((n_l, n_h, total), dtype=np.int64)
    for layer in range(n_l):
        for head in range(n_h):
            keys[layer, head], values[layer, head], clusters[layer, head] = _one_head(
                rng, spec.k_model, spec.v_model, alpha, token_ids, total, d)
    t = spec.prefill_len
    return KvStream(prefill_k=keys[:, :, :t], prefill_v=values[:, :, :t], decode_k=keys[:, :, t:],
                    decode_v=values[:, :, t:], token_ids=token_ids, v_cluster_ids=clusters)


# flat spec keys -> (section, field, converter); section None = top level
_SPEC_FIELDS = {
    "layers": (None, "layers", int), "heads": (None, "heads", int), "head_dim": (None, "head_dim", int),
    "prefill_len": (None, "prefill_len", int), "decode_len": (None, "decode_len", int), "seed": (None, "seed", int),
    "k_outlier_channels": ("k", "outlier_channels", int), "k_outlier_multipliers": ("k", "outlier_multipliers", float),
    "k_drift_rate": ("k", "drift_rate", float), "k_noise_std": ("k", "noise_std", float),
    "v_clusters": ("v", "cluster_count", int), "v_center_spread": ("v", "center_spread", float),
    "v_within_std": ("v", "within_std", float), "v_consistency": ("v", "consistency", float),
    "v_vocab_size": ("v", "vocab_size", int),
}


def parse_stream_spec(text: str) -> SyntheticStreamSpec:
    """`key = value` lines (blank lines and # comments skipped, comma-separated lists for
    the outlier keys) -> SyntheticStreamSpec (reference analysis.py:396-440); unknown keys
    and unparsable values are UsageErrors, missing keys keep the defaults."""
    found = {None: {}, "k": {}, "v": {}}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        key, sep, value = line.partition("=")
        if not sep:
            raise UsageError(f"spec line {lineno} is not `key = value`: {line!r}")
        key, value = key.strip(), value.strip()
        if key not in _SPEC_FIELDS:
            raise UsageError(f"unknown spec key {key!r} on line {lineno}")
        section, name, conv = _SPEC_FIELDS[key]
        try:
            if name.startswith("outlier"):
                found[section][name] = tuple(conv(p.strip()) for p in value.split(",") if p.strip())
            else:
                found[section][name] = conv(value)
        except ValueError as exc:
            raise UsageError(f"bad value for {key!r} on line {lineno}: {value!r}") from exc
    spec = SyntheticStreamSpec(**found[None])
    if found["k"]:
        spec = replace(spec, k_model=replace(spec.k_model, **found["k"]))
    if found["v"]:
        spec = replace(spec, v_model=replace(spec.v_model, **found["v"]))
    _check_spec(spec)
    return spec


@dataclass(frozen=True)
class ConsistencyReport:
    """Majority-cluster share per repeated token id (PAPER Eq. 2 C_t) and their mean
    (nan when no id repeats)."""

    per_token: dict
    aggregate: float


def consistency_metric(token_ids: np.ndarray, cluster_ids: np.ndarray) -> ConsistencyReport:
    """Reference analysis.py:103-117: ids seen once are skipped."""
    tok = np.asarray(token_ids).reshape(-1)
    cl = np.asarray(cluster_ids).reshape(-1)
    if tok.shape != cl.shape:
        raise UsageError("token_ids and cluster_ids must have equal length")
    ids, first, counts = np.unique(tok, return_index=True, return_counts=True)
    shares = {}
    for t, n in zip(ids, counts):
        if n >= 2:
            votes = np.bincount(cl[tok == t].astype(np.int64))
            shares[int(t)] = float(votes.max() / votes.sum())
    return ConsistencyReport(per_token=shares, aggregate=float(np.mean(list(shares.values()))) if shares else float("nan"))


def channel_statistics(stream: KvStream) -> list[dict]:
    """Per-layer key channel statistics over every head and token (reference
    analysis.py:443-463): mean |k|, min, max per channel and the median mean-|k|."""
    out = []
    for layer in range(stream.num_layers):
        flat = np.concatenate([stream.prefill_k[layer], stream.decode_k[layer]], axis=1).reshape(-1, stream.head_dim)
        mean_abs = np.abs(flat).mean(axis=0)
        out.append({"layer": layer, "mean_abs": mean_abs, "min": flat.min(axis=0), "max": flat.max(axis=0),
                    "median_mean_abs": float(np.median(mean_abs))})
    return out


def outlier_channels(stats_row: dict, threshold: float) -> list[int]:
    """Channels whose mean |k| exceeds `threshold` x the layer median."""
    return [int(c) for c in np.flatnonzero(stats_row["mean_abs"] > threshold * stats_row["median_mean_abs"])]
