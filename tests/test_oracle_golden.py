"""Pin the CPU oracle to the reference: golden fixtures (made by running the
reference itself, tests/golden/make_golden.py) and the reference test
suite's known-answer values."""

import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import pkv_oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, name))


# ---- known-answer values from the reference tests -------------------------

def test_quant_kats():
    s, z, c = O.quantize([0.0, 1.0, 2.0, 3.0], 2)  # test_quant.py:32-36
    assert s == 1.0 and z == 0.0 and list(c) == [0, 1, 2, 3]
    s, z, c = O.quantize([5.0, 5.0, 5.0], 2)  # :38-43
    assert s == 0.0 and z == 5.0 and list(c) == [0, 0, 0]
    s, z, c = O.quantize([-1.0, 1.0], 2)  # :45-49
    assert z == -1.0 and abs(s - 2.0 / 3.0) < 1e-15 and list(c) == [0, 3]
    _, _, c = O.quantize([0.0, 0.5, 1.5, 2.5, 15.0], 4)  # :180-187 round half up
    assert list(c) == [0, 1, 2, 3, 15]
    assert O.pack([1, 2, 3, 0], 2) == bytes([0b00111001])  # :105-107
    with pytest.raises(O.OracleData):
        O.quantize([0.0, 1.0, np.nan], 4)


def test_pattern_kats():
    i, r, d = O.minmax_match(np.array([[1.0, 2.0, 3.0]]), np.zeros((1, 3)))
    assert d[0] == 2.0
    i, r, d = O.minmax_match(np.array([[5.0, 1.0]]), np.array([[1.0, 1.0]]))
    assert d[0] == 4.0
    # tie -> lowest index (test_patterns.py:187-193)
    i, _, d = O.minmax_match(np.array([[0.0, 2.0]]), np.array([[0.0, 0.0], [0.0, 0.0]]))
    assert i[0] == 0 and d[0] == 2.0
    assert list(O.midrange(np.array([[0.0, 4.0], [2.0, 2.0]]))) == [1.0, 3.0]


def test_gate_kats():
    assert abs(O.z_quantile(0.05) - 1.644854) < 1e-6
    assert abs(O.z_quantile(0.025) - 1.959964) < 1e-6
    assert O.threshold(128, 0.05) == 0.9115533837525618  # library value
    assert O.flatten_decision(10.0, 9.0, O.threshold(128, 0.05))[0]


# ---- golden fixtures -------------------------------------------------------

@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quant_golden(bits):
    g = load("quant.npz")
    vals, offs = g[f"b{bits}_values"], g[f"b{bits}_offsets"]
    codes = g[f"b{bits}_codes"]
    packed, poffs = g[f"b{bits}_packed"], g[f"b{bits}_packed_offsets"]
    for i in range(len(offs) - 1):
        v = vals[offs[i]:offs[i + 1]]
        s, z, c = O.quantize(v, bits)
        assert s == g[f"b{bits}_scale"][i] and z == g[f"b{bits}_zero"][i]
        assert np.array_equal(c, codes[offs[i]:offs[i + 1]])
        pb = O.pack(c, bits)
        assert pb == packed[poffs[i]:poffs[i + 1]].tobytes()
        assert np.array_equal(O.unpack(pb, len(c), bits), c)


def test_match_golden():
    g = load("match.npz")
    for case in range(4):
        i, r, d = O.minmax_match(g[f"c{case}_x"], g[f"c{case}_m"])
        assert np.array_equal(i, g[f"c{case}_idx"])
        assert np.array_equal(d, g[f"c{case}_dist"])
        assert np.array_equal(r, g[f"c{case}_res"])


def test_kmeans_golden():
    g = load("kmeans.npz")
    for case in range(5):
        x = g[f"c{case}_x"]
        assert O.first_seed_index(len(x), int(g[f"c{case}_seed"])) == int(g[f"c{case}_first"])
        c, lab, hist = O.kmeans(x, int(g[f"c{case}_k"]), int(g[f"c{case}_seed"]))
        assert np.array_equal(lab, g[f"c{case}_labels"])
        np.testing.assert_allclose(c, g[f"c{case}_centers"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(hist, g[f"c{case}_hist"], rtol=1e-12)


def test_gate_golden():
    g = load("gate.npz")
    for j, a in enumerate(g["alphas"]):
        assert O.z_quantile(float(a)) == g["z"][j]
        for i, d in enumerate(g["dims"]):
            want = g["thr"][i, j]
            if np.isnan(want):
                with pytest.raises(O.OracleUsage):
                    O.threshold(int(d), float(a))
            else:
                assert O.threshold(int(d), float(a)) == want


def test_synth_golden():
    g = load("synth.npz")
    for i in range(2):
        k, v = g[f"c{i}_k"], g[f"c{i}_v"]
        kk, vv = O.synth_unit(int(g[f"c{i}_seed"]), k.shape[0], k.shape[1])
        assert np.array_equal(kk, k) and np.array_equal(vv, v)


def _engine_case(g, name):
    p = name + "__"
    cfg = json.loads(str(g[p + "config"]))
    seed, d, tp, td = (int(g[p + x]) for x in ("seed", "d", "prefill", "decode"))
    k, v = O.synth_unit(seed, tp + td, d)
    k = k.astype(np.float16).astype(np.float64)
    v = v.astype(np.float16).astype(np.float64)
    return cfg, k, v, tp, td


def compare_state(h, g, p):
    """Bit-exact comparison of an oracle head with a golden reference state."""
    assert np.array_equal(h.kpat, g[p + "kpat"].reshape(-1, h.d))
    assert np.array_equal(h.vpat, g[p + "vpat"].reshape(-1, h.d))
    assert [b[0] for b in h.k_blocks] == list(g[p + "kb_start"])
    assert [b[1] for b in h.k_blocks] == list(g[p + "kb_len"])
    if h.k_blocks:
        assert np.array_equal(np.concatenate([b[2] for b in h.k_blocks]), g[p + "k_scale"])
        assert np.array_equal(np.concatenate([b[3] for b in h.k_blocks]), g[p + "k_zero"])
        assert np.array_equal(np.concatenate([b[4] for b in h.k_blocks]), g[p + "k_codes"])
        assert np.array_equal(np.concatenate([b[5] for b in h.k_blocks]), g[p + "k_idx"])
        kb = b"".join(b"".join(h.k_block_ref_bytes(i)) for i in range(len(h.k_blocks)))
        assert kb == g[p + "k_bytes"].tobytes()
        assert np.array_equal(np.array([t[0] for t in h.v_tok]), g[p + "v_scale"])
        assert np.array_equal(np.array([t[1] for t in h.v_tok]), g[p + "v_zero"])
        assert np.array_equal(np.stack([t[2] for t in h.v_tok]), g[p + "v_codes"])
        assert np.array_equal(np.array([t[3] for t in h.v_tok]), g[p + "v_idx"])
        kc, vc = h.committed_kv()
        assert np.array_equal(kc, g[p + "k_hat"]) and np.array_equal(vc, g[p + "v_hat"])
    vd = np.array([[a, b, float(c)] for a, b, c in h.vdec]).reshape(-1, 3)
    assert np.array_equal(vd, g[p + "vdec"][:, :3])
    kd = np.array([[a, b, float(c)] for a, b, c in h.kdec]).reshape(-1, 3)
    assert np.array_equal(kd, g[p + "kdec"][:, :3])
    wk, wv = h.window_kv()
    assert np.array_equal(wk, g[p + "window_k"]) and np.array_equal(wv, g[p + "window_v"])
    assert h.tokens == int(g[p + "token_count"])


ENGINE_NAMES = ["default2", "four_bit", "g64", "k_gate", "no_vgate", "raw", "no_new", "eight_bit", "short"]


@pytest.mark.parametrize("name", ENGINE_NAMES)
def test_engine_golden(name):
    g = load("engine.npz")
    cfg, k, v, tp, td = _engine_case(g, name)
    knobs = O.Knobs(**cfg)
    h = O.OracleHead(knobs, k.shape[1]).prefill(k[:tp], v[:tp])
    compare_state(h, g, name + "__pre_")
    for t in range(tp, tp + td):
        h.append(k[t], v[t])
    compare_state(h, g, name + "__fin_")


def test_acceptance_instance():
    """test_acceptance.py:354-381 instance: MSEs, pattern counts and codes hash."""
    with open(os.path.join(G, "acceptance.json")) as f:
        doc = json.load(f)
    k, v = O.synth_unit(11, 4096, 64, drift=1e-3, clusters=8, spread=10.0, within=0.1, consistency=1.0, vocab=64)
    assert np.allclose(k[:2, :4], doc["kp_head"], rtol=0, atol=0)
    knobs = O.Knobs(bits=2, pattern_count=32, seed=11)
    h = O.replay(k[:2048], v[:2048], k[2048:], v[2048:], knobs)
    kc, vc = h.committed_kv()
    c = h.committed
    mse = (((kc - k[:c]) ** 2).sum() + ((vc - v[:c]) ** 2).sum()) / (2 * c * 64)
    assert math.isclose(mse, doc["mse"], rel_tol=1e-12)
    assert len(h.kpat) == doc["k_patterns"] and len(h.vpat) == doc["v_patterns"]
    hs = hashlib.sha256()
    for b in range(len(h.k_blocks)):
        hs.update(h.k_blocks[b][5].astype(np.int32).tobytes())
        for chunk in h.k_block_ref_bytes(b):
            hs.update(chunk)
    for (_, _, cd, j) in h.v_tok:
        hs.update(np.int32(j).tobytes())
        hs.update(O.pack(cd, 2))
    assert hs.hexdigest() == doc["sha256"]
