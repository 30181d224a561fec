"""The reference's public API (pkg/src/patternkv/__init__.py:10-94) served by
the B200 package: known-answer values and behaviours of the reference test
suite (test_quant.py, test_patterns.py, test_engine.py, test_acceptance.py),
checked against the golden fixtures made by the reference itself."""

import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pkv_oracle as O  # noqa: E402

G = os.path.join(os.path.dirname(__file__), "golden")
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_05176_b200 as pkg
    return pkg


# ---- quant (test_quant.py) -------------------------------------------------------------

def test_quant_kats(P):
    g = P.quantize_group(np.array([0.0, 1.0, 2.0, 3.0]), bits=2)
    assert g.params.scale == 1.0 and g.params.zero_point == 0.0
    assert list(P.unpack_codes(g.codes, g.length, 2)) == [0, 1, 2, 3]
    g = P.quantize_group(np.array([5.0, 5.0, 5.0]), bits=2)
    assert g.params.scale == 0.0 and list(P.dequantize_group(g)) == [5.0, 5.0, 5.0]
    g = P.quantize_group(np.array([-1.0, 1.0]), bits=2)
    assert g.params.zero_point == -1.0 and list(P.unpack_codes(g.codes, 2, 2)) == [0, 3]
    g = P.quantize_group(np.array([0.0, 0.5, 1.5, 2.5, 15.0]), bits=4)
    assert list(P.unpack_codes(g.codes, g.length, 4)) == [0, 1, 2, 3, 15]
    assert P.pack_codes(np.array([1, 2, 3, 0]), bits=2) == bytes([0b00111001])
    assert P.pack_codes(np.array([], dtype=np.uint8), bits=4) == b""
    with pytest.raises(P.UsageError):
        P.quantize_group(np.array([]), bits=2)
    with pytest.raises(P.UsageError):
        P.quantize_group(np.array([1.0, 2.0]), bits=3)
    with pytest.raises(P.DataError, match="2"):
        P.quantize_group(np.array([0.0, 1.0, np.nan, 3.0]), bits=4)
    with pytest.raises(P.UsageError):
        P.pack_codes(np.array([4]), bits=2)
    with pytest.raises(P.DataError):
        P.unpack_codes(P.pack_codes(np.array([1, 2, 3]), 4), 5, 4)


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quant_golden_groups(P, bits):
    from paper_2510_05176_b200.quant import quantize_groups

    g = np.load(os.path.join(G, "quant.npz"))
    vals, offs = g[f"b{bits}_values"], g[f"b{bits}_offsets"]
    groups = [vals[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
    res = quantize_groups(groups, bits)
    codes = g[f"b{bits}_codes"]
    for i, (s, z, c) in enumerate(res):
        assert s == g[f"b{bits}_scale"][i] and z == g[f"b{bits}_zero"][i]
        assert np.array_equal(c, codes[offs[i]:offs[i + 1]])
    # pack of a few groups equals the reference bytes
    packed, poffs = g[f"b{bits}_packed"], g[f"b{bits}_packed_offsets"]
    for i in range(0, len(res), 37):
        assert P.pack_codes(res[i][2], bits) == packed[poffs[i]:poffs[i + 1]].tobytes()


# ---- patterns (test_patterns.py) ---------------------------------------------------------

def test_pattern_kats(P):
    assert P.minmax_distance(np.array([1.0, 2.0, 3.0]), np.zeros(3)) == 2.0
    assert P.minmax_distance(np.array([5.0, 1.0]), np.array([1.0, 1.0])) == 4.0
    ps = P.PatternSet(2)
    ps.append(np.array([0.0, 0.0]), "prefill")
    ps.append(np.array([0.0, 0.0]), "prefill")
    m = P.match_pattern(np.array([0.0, 2.0]), ps)
    assert m.pattern_index == 0 and m.distance == 2.0
    ps = P.PatternSet(2)
    ps.append(np.array([1.0, 1.0]), "prefill")  # constant offset ties the exact match
    ps.append(np.array([0.0, 0.0]), "prefill")
    m = P.match_pattern(np.array([0.0, 0.0]), ps)
    assert m.pattern_index == 0 and m.distance == 0.0 and list(m.residual) == [-1.0, -1.0]
    assert list(P.midrange_center(np.array([[0.0, 4.0], [2.0, 2.0]]))) == [1.0, 3.0]
    with pytest.raises(P.UsageError):
        P.match_pattern(np.zeros(2), P.PatternSet(2))


def test_match_many_golden(P):
    g = np.load(os.path.join(G, "match.npz"))
    for case in range(4):
        ps = P.PatternSet(g[f"c{case}_m"].shape[1])
        for row in g[f"c{case}_m"]:
            ps.append(row, "prefill")
        idx, res, dist = P.match_many(g[f"c{case}_x"], ps)
        assert np.array_equal(idx, g[f"c{case}_idx"])
        assert np.array_equal(dist, g[f"c{case}_dist"])
        assert np.array_equal(res, g[f"c{case}_res"])


def test_lloyd_kmeans_golden(P):
    """Mining parity: identical labels, centroids within 1e-12 (ulp-level
    einsum order differences only), objective history within 1e-12 rel."""
    g = np.load(os.path.join(G, "kmeans.npz"))
    for case in range(5):
        x = g[f"c{case}_x"]
        c, lab, hist = P.lloyd_kmeans(x, int(g[f"c{case}_k"]), int(g[f"c{case}_seed"]))
        assert np.array_equal(lab, g[f"c{case}_labels"]), case
        np.testing.assert_allclose(c, g[f"c{case}_centers"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(hist, g[f"c{case}_hist"], rtol=1e-12)
    ps = P.mine_patterns(g["c3_x"], 8, 5)  # 3 distinct rows <= k: sorted unique rows
    assert len(ps) == 3 and all(ps.origin(i) == "prefill" for i in range(3))


# ---- engine (test_engine.py) ------------------------------------------------------------------

def test_engine_geometry_and_reconstruct(P):
    rng = np.random.default_rng(2)
    k, v = rng.normal(size=(300, 8)), rng.normal(size=(300, 8))
    st = P.prefill(k, v, P.EngineConfig(pattern_count=4, group_size=128, residual_window=128))
    assert st.committed_count == 172
    assert [b.length for b in st.k_blocks] == [128, 44]
    rng = np.random.default_rng(12)
    k, v = rng.normal(size=(40, 8)), rng.normal(size=(40, 8))
    st = P.prefill(k, v, P.EngineConfig(pattern_count=4, group_size=16, residual_window=16))
    for t in range(24, 40):
        rk, rv = P.reconstruct_token(st, t)
        assert np.array_equal(rk, k[t]) and np.array_equal(rv, v[t])
    with pytest.raises(P.UsageError):
        P.reconstruct_token(st, 40)
    # exact-pattern vectors reconstruct exactly (test_engine.py:119-130)
    rng = np.random.default_rng(3)
    centers = rng.normal(size=(4, 8)) * 5
    idx = rng.integers(0, 4, size=64)
    st = P.prefill(centers[idx], centers[idx], P.EngineConfig(pattern_count=4, group_size=16, residual_window=16))
    rk, rv = P.committed_matrices(st)
    assert np.abs(rk - centers[idx][:48]).max() == 0.0 and np.abs(rv - centers[idx][:48]).max() == 0.0


def test_engine_append_and_errors(P):
    rng = np.random.default_rng(6)
    cfg = P.EngineConfig(pattern_count=4, group_size=32, residual_window=32, bits=4)
    st = P.prefill(rng.normal(size=(64, 8)), rng.normal(size=(64, 8)), cfg)
    kp, vp, committed = len(st.k_patterns), len(st.v_patterns), st.committed_count
    for _ in range(32):
        P.append_decode_token(rng.normal(size=8), rng.normal(size=8), st)
    assert st.committed_count == committed + 32 and len(st.window_k) == 32
    assert len(st.k_patterns) == kp + 1 and len(st.v_patterns) == vp + 1
    assert st.k_patterns.origin(len(st.k_patterns) - 1) == "decode"
    with pytest.raises(P.UsageError):
        P.append_decode_token(np.zeros(9), np.zeros(8), st)
    bad = np.zeros(8)
    bad[2] = np.nan
    with pytest.raises(P.DataError):
        P.append_decode_token(bad, np.zeros(8), st)
    k = np.zeros((10, 4))
    v = np.zeros((10, 4))
    v[3, 1] = np.inf
    with pytest.raises(P.DataError, match="token 3"):
        P.prefill(k, v, P.EngineConfig(group_size=4, residual_window=4, pattern_count=2))


def test_run_scheme_comparison_acceptance(P):
    """test_acceptance.py:354-381 through the GPU harness: MSE at rel 1e-9,
    gate acceptance, bits/token and pattern counts equal the reference."""
    with open(os.path.join(G, "acceptance.json")) as f:
        doc = json.load(f)
    k, v = O.synth_unit(11, 4096, 64, drift=1e-3, clusters=8, spread=10.0, within=0.1, consistency=1.0, vocab=64)
    stream = P.KvStream(prefill_k=k[None, None, :2048], prefill_v=v[None, None, :2048],
                        decode_k=k[None, None, 2048:], decode_v=v[None, None, 2048:])
    cfg = P.EngineConfig(bits=2, pattern_count=32, group_size=128, residual_window=128, seed=11)
    raw, pkv = P.run_scheme_comparison(stream, [("patternkv", cfg)])
    assert raw.scheme == "raw" and raw.config.is_raw
    assert math.isclose(pkv.mse, doc["mse"], rel_tol=1e-9)
    assert math.isclose(raw.mse, doc["raw_mse"], rel_tol=1e-9)
    assert pkv.committed_tokens == doc["committed"]
    assert pkv.v_gate_acceptance_rate == doc["gate_acceptance"]
    assert pkv.bits_per_token == doc["bits_per_token"] and raw.bits_per_token == doc["raw_bits_per_token"]
    assert pkv.per_head[0].k_pattern_count == doc["k_patterns"]
    assert pkv.mse < 0.5 * raw.mse
