"""The drop-in synthetic-stream API (reference analysis.py:248-470) on the host:
generate_synthetic_stream reproduces the reference generator's own output
(tests/golden/synth.npz, written by running the reference), parse_stream_spec
follows the flat spec format and its errors, consistency_metric its skipping rule."""

import math
import os

import numpy as np
import pytest

from paper_2510_05176_b200 import synthetic as S
from paper_2510_05176_b200.errors import UsageError

G = os.path.join(os.path.dirname(__file__), "golden")


def _spec(seed, tokens, d):
    return S.SyntheticStreamSpec(
        layers=1, heads=1, head_dim=d, prefill_len=tokens, decode_len=0, seed=seed,
        k_model=S.KeyModel(outlier_channels=(3,), outlier_multipliers=(32.0,), drift_rate=1.0 / tokens, noise_std=0.05),
        v_model=S.ValueModel(cluster_count=32, center_spread=5.0, within_std=0.2, consistency=0.9, vocab_size=1024))


def test_generator_matches_reference_golden():
    g = np.load(os.path.join(G, "synth.npz"))
    for i in range(2):
        k, v = g[f"c{i}_k"], g[f"c{i}_v"]
        s = S.generate_synthetic_stream(_spec(int(g[f"c{i}_seed"]), k.shape[0], k.shape[1]))
        assert np.array_equal(s.prefill_k[0, 0], k) and np.array_equal(s.prefill_v[0, 0], v)


def test_spec_parser_and_errors():
    spec = S.parse_stream_spec("layers = 3\n# comment\n\nk_outlier_channels = 1, 5\nk_outlier_multipliers = 2, 8.5\n"
                               "v_clusters = 4\nseed = 7\n")
    assert spec.layers == 3 and spec.seed == 7 and spec.v_model.cluster_count == 4
    assert spec.k_model.outlier_channels == (1, 5) and spec.k_model.outlier_multipliers == (2.0, 8.5)
    assert spec.heads == S.SyntheticStreamSpec().heads  # missing keys keep defaults
    for bad in ("layers 3", "bogus = 1", "layers = x", "k_outlier_channels = 1\nk_outlier_multipliers = 1, 2",
                "v_consistency = 1.5", "head_dim = 4\nk_outlier_channels = 9\nk_outlier_multipliers = 2"):
        with pytest.raises(UsageError):
            S.parse_stream_spec(bad)


def test_consistency_metric_and_channel_stats():
    rep = S.consistency_metric(np.array([0, 0, 0, 1, 2, 2]), np.array([1, 1, 2, 0, 3, 3]))
    assert rep.per_token == {0: 2 / 3, 2: 1.0} and math.isclose(rep.aggregate, (2 / 3 + 1.0) / 2)
    assert math.isnan(S.consistency_metric(np.array([1, 2]), np.array([0, 0])).aggregate)
    with pytest.raises(UsageError):
        S.consistency_metric(np.array([1, 2]), np.array([0]))
    s = S.generate_synthetic_stream(S.DEFAULT_STREAM_SPEC)
    rows = S.channel_statistics(s)
    assert len(rows) == 2 and S.outlier_channels(rows[0], 4.0) == [3]
    full = S.consistency_metric(s.token_ids, s.v_cluster_ids[0, 0])
    assert 0.85 <= full.aggregate <= 1.0
