"""GPU parity at BASELINE.json's configurations.

* cfg1 end to end: U = 8 units x 4096 tokens, 4-bit, |M| = 16, GPU mining + K1-TC
  encode + 256 decode appends (two flushes with refresh), bit-exact against the
  oracle's prefill/append (engine.py:142-198, patterns.py:72-171).
* cfg2-shaped units: 32,768-token Llama-3.1-8B-shaped units, |M| = 32, 2-bit AND
  4-bit through K1-TC, then 256 decode appends: pattern tables, indices, codes,
  params, gate decisions and window bit-exact against the oracle.
* Mining at 32K tokens: the GPU's final label vector, iteration count and objective
  history against oracle.kmeans (patterns.py:72-126); the closest approach of any
  round to the 1e-6 stop threshold is logged.

The oracle runs on host cores in spawned worker processes (oracle/parity_jobs.py);
inputs are the reference generator family (oracle.synth_unit) rounded to fp16.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import parity_jobs as J  # noqa: E402
from oracle import pkv_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def pkv():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_05176_b200 as P
    return P


def _inputs(seeds, tokens, d=128):
    ks, vs = zip(*(J.unit_inputs(s, tokens, d) for s in seeds))
    return np.stack(ks), np.stack(vs)


def _assert_unit(st, want, what):
    np.testing.assert_array_equal(st.kpat, want["kpat"], err_msg=f"{what}: K patterns")
    np.testing.assert_array_equal(st.vpat, want["vpat"], err_msg=f"{what}: V patterns")
    np.testing.assert_array_equal(st.kb_start, want["kb_start"], err_msg=f"{what}: block starts")
    np.testing.assert_array_equal(st.kb_len, want["kb_len"], err_msg=f"{what}: block lengths")
    for key in ("k_idx", "v_idx", "k_codes", "v_codes"):
        got, exp = getattr(st, key), want[key]
        if not np.array_equal(got, exp):
            bad = np.argwhere(got != exp)
            raise AssertionError(f"{what}: {key} differs at {len(bad)} positions, first {bad[:5].tolist()}")
    np.testing.assert_array_equal(st.k_scale, want["k_scale"], err_msg=f"{what}: K scales")
    np.testing.assert_array_equal(st.k_zero, want["k_zero"], err_msg=f"{what}: K zeros")
    np.testing.assert_array_equal(st.v_scale, want["v_scale"], err_msg=f"{what}: V scales")
    np.testing.assert_array_equal(st.v_zero, want["v_zero"], err_msg=f"{what}: V zeros")
    if st.vdec.shape[0]:
        np.testing.assert_array_equal(st.vdec[:, 2].astype(bool), want["vdec"], err_msg=f"{what}: gate")
    np.testing.assert_array_equal(st.window_k, want["window_k"], err_msg=f"{what}: window K")
    np.testing.assert_array_equal(st.window_v, want["window_v"], err_msg=f"{what}: window V")
    assert st.token_count == want["tokens"]


def _run_gpu(pkv, cfg, k, v, tp, td, record=True):
    from paper_2510_05176_b200.export import export_unit

    U, d = k.shape[0], k.shape[2]
    cache = pkv.PatternKVCache(cfg, U, d, dtype=torch.float16, max_tokens=tp + td + 256, record_decisions=record)
    kt = torch.from_numpy(k).to("cuda", torch.float16)
    vt = torch.from_numpy(v).to("cuda", torch.float16)
    cache.prefill(kt[:, :tp], vt[:, :tp])
    for t in range(tp, tp + td):
        cache.append(kt[:, t], vt[:, t])
    torch.cuda.synchronize()
    return cache, [export_unit(cache, u, with_bytes=False) for u in range(U)]


def test_cfg1_end_to_end(pkv):
    """BASELINE configs[0]: 8 KV heads x 4096 tokens, d = 128, 4-bit, |M| = 16 -- GPU mining,
    K1-TC prefill and 256 decode appends == the reference path (oracle) bit for bit."""
    from paper_2510_05176_b200.config import EngineConfig

    seeds = [O.unit_seed(0, 0, h) for h in range(8)]
    tp, td = 4096, 256
    jobs = [(s, tp, td, 128, 16, [4], 0) for s in seeds]
    want = J.run_pool(J.unit_job, jobs)
    k, v = _inputs(seeds, tp + td)
    cache, states = _run_gpu(pkv, EngineConfig(bits=4, pattern_count=16), k, v, tp, td)
    for u in range(8):
        _assert_unit(states[u], want[u][4], f"cfg1 unit {u}")
        assert len(states[u].kpat) == 16 + 2 and len(states[u].vpat) == 16 + 2  # two flush refreshes
    # decode attention over the cfg1 cache (GQA 4) vs fp64 softmax over the oracle's reconstruction
    q = np.random.default_rng(1).normal(size=(8, 4, 128)).astype(np.float32)
    out = cache.decode_attention(torch.from_numpy(q).cuda()).cpu().numpy()
    for u in (0, 5):
        h = O.replay(k[u, :tp], v[u, :tp], k[u, tp:], v[u, tp:], O.Knobs(bits=4, pattern_count=16))
        ref = O.head_attention(h, q[u].astype(np.float64), 1.0 / math.sqrt(128))
        assert np.abs(out[u] - ref).max() / np.abs(ref).max() <= 1e-3


@pytest.fixture(scope="module")
def cfg2_oracle():
    seeds = [O.unit_seed(3, 17, 5), O.unit_seed(7, 31, 2), O.unit_seed(0, 0, 0), O.unit_seed(5, 9, 7)]
    tp, td = 32768, 256
    want = J.run_pool(J.unit_job, [(s, tp, td, 128, 32, [2, 4], 0) for s in seeds])
    return seeds, tp, td, want


@pytest.mark.parametrize("bits", [2, 4])
def test_cfg2_units_32k(pkv, cfg2_oracle, bits):
    """cfg2-shaped units (32,768-token prefill, d = 128, |M| = 32) through GPU mining + K1-TC,
    then 256 decode appends (two flushes, P 32 -> 34): bit-exact vs the oracle."""
    from paper_2510_05176_b200.config import EngineConfig

    seeds, tp, td, want = cfg2_oracle
    k, v = _inputs(seeds, tp + td)
    _, states = _run_gpu(pkv, EngineConfig(bits=bits, pattern_count=32), k, v, tp, td)
    for u in range(len(seeds)):
        _assert_unit(states[u], want[u][bits], f"cfg2 {bits}-bit unit {u}")
        assert len(states[u].kpat) == 34


def test_mining_32k_labels_history(pkv, cfg2_oracle):
    """K2 at 32K tokens: final labels, iteration count, objective history (rel 1e-12) and centers
    (bit-exact) per unit-side vs oracle.kmeans; logs the closest approach to the stop threshold."""
    from paper_2510_05176_b200.config import EngineConfig

    seeds, tp, td, want = cfg2_oracle
    k, v = _inputs(seeds, tp + td)  # the oracle mined the first tp rows of these units
    k, v = np.ascontiguousarray(k[:, :tp]), np.ascontiguousarray(v[:, :tp])
    cache = pkv.PatternKVCache(EngineConfig(bits=2, pattern_count=32), len(seeds), 128, dtype=torch.float16,
                               max_tokens=tp + 256)
    for side, x, key in ((0, k, "k"), (1, v, "v")):
        hist, nit, lab = cache.mine(side, torch.from_numpy(x).to("cuda", torch.float16), seed=side, labels=True)
        lab = lab.cpu().numpy()
        tabs = cache.patterns(side)[:, :32].cpu().numpy()
        for u in range(len(seeds)):
            w = want[u]
            hw = w["hist_" + key]
            print(f"unit {u} side {key}: {len(hw)} rounds, closest stop margin {w['margin_' + key]:.3g}")
            assert int(nit[u]) == len(hw), f"unit {u} {key}: {nit[u]} rounds vs oracle {len(hw)}"
            np.testing.assert_allclose(hist[u, :len(hw)], hw, rtol=1e-12, atol=0)
            ndiff = int((lab[u] != w["lab_" + key]).sum())
            assert ndiff == 0, f"unit {u} {key}: {ndiff} labels differ"
            np.testing.assert_array_equal(tabs[u], w[bits_key(w)]["kpat" if side == 0 else "vpat"][:32])


def bits_key(w):
    return 2 if 2 in w else 4
