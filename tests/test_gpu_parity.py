"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
golden states and the CPU oracle.  Bit-exact for indices, codes, gate
decisions, params and the fp64 reconstruction; attention within 1e-3 of the
fp64 oracle (relative to max |out|)."""

import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import pkv_oracle as O  # noqa: E402

G = os.path.join(os.path.dirname(__file__), "golden")
ENGINE_NAMES = ["default2", "four_bit", "g64", "k_gate", "no_vgate", "raw", "no_new", "eight_bit", "short"]


@pytest.fixture(scope="module")
def pkv():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_05176_b200 as P
    from paper_2510_05176_b200 import config, export  # noqa: F401
    return P


def _golden():
    return np.load(os.path.join(G, "engine.npz"))


def _case(g, name):
    p = name + "__"
    cfg = json.loads(str(g[p + "config"]))
    seed, d, tp, td = (int(g[p + x]) for x in ("seed", "d", "prefill", "decode"))
    k, v = O.synth_unit(seed, tp + td, d)
    return cfg, k.astype(np.float16).astype(np.float64), v.astype(np.float16).astype(np.float64), tp, td


def assert_state(st, g, p, d, bits):
    kpat = g[p + "kpat"].reshape(-1, d)
    vpat = g[p + "vpat"].reshape(-1, d)
    assert st.kpat.shape == kpat.shape and st.vpat.shape == vpat.shape
    np.testing.assert_array_equal(st.kpat, kpat)
    np.testing.assert_array_equal(st.vpat, vpat)
    np.testing.assert_array_equal(st.kb_start, g[p + "kb_start"])
    np.testing.assert_array_equal(st.kb_len, g[p + "kb_len"])
    if len(st.kb_start):
        np.testing.assert_array_equal(st.k_idx, g[p + "k_idx"])
        np.testing.assert_array_equal(st.v_idx, g[p + "v_idx"])
        np.testing.assert_array_equal(st.k_codes, g[p + "k_codes"])
        np.testing.assert_array_equal(st.v_codes, g[p + "v_codes"])
        np.testing.assert_array_equal(st.k_scale.reshape(-1), g[p + "k_scale"])
        np.testing.assert_array_equal(st.k_zero.reshape(-1), g[p + "k_zero"])
        np.testing.assert_array_equal(st.v_scale, g[p + "v_scale"])
        np.testing.assert_array_equal(st.v_zero, g[p + "v_zero"])
        kb = b"".join(b"".join(blk) for blk in st.k_bytes)
        assert kb == g[p + "k_bytes"].tobytes()
        assert b"".join(st.v_bytes) == g[p + "v_bytes"].tobytes()
    np.testing.assert_array_equal(st.vdec, g[p + "vdec"][:, :3])
    np.testing.assert_array_equal(st.kdec, g[p + "kdec"][:, :3])
    np.testing.assert_array_equal(st.window_k, g[p + "window_k"])
    np.testing.assert_array_equal(st.window_v, g[p + "window_v"])
    assert st.token_count == int(g[p + "token_count"])


@pytest.mark.parametrize("dtype", ["float64", "float16"])
@pytest.mark.parametrize("name", ENGINE_NAMES)
def test_engine_golden_gpu(pkv, name, dtype):
    """Prefill then decode appends on the GPU == the reference's own states."""
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.export import export_unit

    g = _golden()
    cfg, k, v, tp, td = _case(g, name)
    d = k.shape[1]
    tdt = getattr(torch, dtype)
    ec = EngineConfig(**cfg)
    cache = pkv.PatternKVCache(ec, 1, d, dtype=tdt, max_tokens=64, record_decisions=True, stats=True)
    kt = torch.from_numpy(k).to("cuda", tdt)
    vt = torch.from_numpy(v).to("cuda", tdt)
    cache.prefill(kt[None, :tp], vt[None, :tp])
    assert_state(export_unit(cache, 0), g, name + "__pre_", d, ec.bits)
    for t in range(tp, tp + td):
        cache.append(kt[None, t], vt[None, t])
    assert_state(export_unit(cache, 0), g, name + "__fin_", d, ec.bits)
    # exact fp64 reconstruction (engine.py:296-303)
    if name + "__fin_k_hat" in g.files:
        kc, vc = cache.dequant()
        np.testing.assert_array_equal(kc[0].cpu().numpy(), g[name + "__fin_k_hat"])
        np.testing.assert_array_equal(vc[0].cpu().numpy(), g[name + "__fin_v_hat"])


def test_acceptance_instance_gpu(pkv):
    """test_acceptance.py:354-381: MSE at rel 1e-9 and the codes/idx sha256."""
    import hashlib

    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.export import export_unit

    with open(os.path.join(G, "acceptance.json")) as f:
        doc = json.load(f)
    k, v = O.synth_unit(11, 4096, 64, drift=1e-3, clusters=8, spread=10.0, within=0.1, consistency=1.0, vocab=64)
    cache = pkv.PatternKVCache(EngineConfig(bits=2, pattern_count=32, seed=11), 1, 64, dtype=torch.float64,
                               record_decisions=True)
    kt = torch.from_numpy(k).cuda()
    vt = torch.from_numpy(v).cuda()
    cache.prefill(kt[None, :2048], vt[None, :2048])
    for t in range(2048, 4096):
        cache.append(kt[None, t], vt[None, t])
    kc, vc = cache.dequant()
    c = kc.shape[1]
    mse = (((kc[0] - kt[:c]) ** 2).sum() + ((vc[0] - vt[:c]) ** 2).sum()).item() / (2 * c * 64)
    assert math.isclose(mse, doc["mse"], rel_tol=1e-9)
    st = export_unit(cache, 0)
    assert len(st.kpat) == doc["k_patterns"] and len(st.vpat) == doc["v_patterns"]
    h = hashlib.sha256()
    for b in range(len(st.kb_start)):
        s, n = int(st.kb_start[b]), int(st.kb_len[b])
        h.update(st.k_idx[s:s + n].astype(np.int32).tobytes())
        for chunk in st.k_bytes[b]:
            h.update(chunk)
    for t in range(len(st.v_idx)):
        h.update(np.int32(st.v_idx[t]).tobytes())
        h.update(st.v_bytes[t])
    assert h.hexdigest() == doc["sha256"]


def test_multi_unit_encode_injected_patterns(pkv):
    """K1 on U=8 units with reference-mined tables injected: bit-exact vs the
    oracle commit path, fp16 inputs, 4-bit, P=16."""
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.export import export_unit

    U, T, d = 8, 1024, 128
    ec = EngineConfig(bits=4, pattern_count=16)
    ks, vs, kps, vps, heads = [], [], [], [], []
    for u in range(U):
        k, v = O.synth_unit(O.unit_seed(0, 0, u), T, d)
        k = k.astype(np.float16).astype(np.float64)
        v = v.astype(np.float16).astype(np.float64)
        h = O.OracleHead(O.Knobs(bits=4, pattern_count=16), d)
        h.kpat = O.kmeans(k, 16, 0)[0]
        h.vpat = O.kmeans(v, 16, 1)[0]
        ks.append(k); vs.append(v); kps.append(h.kpat); vps.append(h.vpat)
        ncommit = T - 128
        for s in range(0, ncommit, 128):
            h.commit(k[s:s + 128], v[s:s + 128], s)
        heads.append(h)
    cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + 256, stats=True)
    cache.set_patterns(0, torch.from_numpy(np.stack(kps)))
    cache.set_patterns(1, torch.from_numpy(np.stack(vps)))
    cache.commit_prefill(torch.from_numpy(np.stack(ks)).half().cuda(), torch.from_numpy(np.stack(vs)).half().cuda())
    for u in range(U):
        st = export_unit(cache, u, with_bytes=False)
        h = heads[u]
        np.testing.assert_array_equal(st.k_idx, np.concatenate([b[5] for b in h.k_blocks]))
        np.testing.assert_array_equal(st.k_codes, np.concatenate([b[4] for b in h.k_blocks]))
        np.testing.assert_array_equal(st.v_idx, np.array([t[3] for t in h.v_tok]))
        np.testing.assert_array_equal(st.v_codes, np.stack([t[2] for t in h.v_tok]))
    print("refines/exact-div:", cache.info().n_refined, cache.info().n_exact_div)


@pytest.mark.parametrize("bits,gqa", [(2, 4), (4, 4), (4, 8), (2, 7), (8, 1)])
def test_decode_attention_vs_fp64_oracle(pkv, bits, gqa):
    """K3 against fp64 softmax attention over the reconstructed cache + window."""
    from paper_2510_05176_b200.config import EngineConfig

    U, T, d, steps = 4, 1500, 128, 150
    ec = EngineConfig(bits=bits, pattern_count=16)
    ks, vs = [], []
    for u in range(U):
        k, v = O.synth_unit(O.unit_seed(1, 2, u), T + steps, d)
        ks.append(k); vs.append(v)
    kt = torch.from_numpy(np.stack(ks)).half().cuda()
    vt = torch.from_numpy(np.stack(vs)).half().cuda()
    cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + steps + 256)
    cache.prefill(kt[:, :T], vt[:, :T])
    for t in range(T, T + steps):
        cache.append(kt[:, t], vt[:, t])
    rng = np.random.default_rng(5)
    q = rng.normal(size=(U, gqa, d)).astype(np.float32)
    out = cache.decode_attention(torch.from_numpy(q).cuda()).cpu().numpy()
    kc, vc = cache.dequant()
    wk, wv = cache.window()
    for u in range(U):
        kall = np.concatenate([kc[u].cpu().numpy(), wk[u].double().cpu().numpy()])
        vall = np.concatenate([vc[u].cpu().numpy(), wv[u].double().cpu().numpy()])
        ref = O.attention(q[u].astype(np.float64), kall, vall, 1.0 / math.sqrt(d))
        err = np.abs(out[u] - ref).max() / np.abs(ref).max()
        print(f"bits={bits} gqa={gqa} unit={u} max-abs err / max|ref| = {err:.3e}")
        assert err <= 1e-3, (u, err)


def test_errors_map_to_reference_taxonomy(pkv):
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.errors import DataError, UsageError

    with pytest.raises(UsageError):
        EngineConfig(bits=3)
    with pytest.raises(UsageError):
        EngineConfig(group_size=64, residual_window=32)
    cache = pkv.PatternKVCache(EngineConfig(pattern_count=2, group_size=4, residual_window=4), 1, 4,
                               dtype=torch.float64)
    k = torch.zeros((1, 10, 4), dtype=torch.float64)
    v = torch.zeros((1, 10, 4), dtype=torch.float64)
    v[0, 3, 1] = float("inf")
    with pytest.raises(DataError, match="token 3"):
        cache.prefill(k, v, sync_check=True)


@pytest.mark.parametrize("k", [16, 32, 64])
def test_tcgen05_mining_matches_cuda_core_and_oracle(pkv, k, monkeypatch):
    """K2 on tcgen05 (fp16, d=128) == the fp64 CUDA-core miner bit for bit, and
    == the oracle's k-means within 1e-12 (einsum-order ulps only)."""
    from paper_2510_05176_b200.config import EngineConfig

    U, T, d = 3, 2048, 128
    xs = []
    for u in range(U):
        kk, vv = O.synth_unit(O.unit_seed(2, 1, u), T, d)
        xs.append(kk.astype(np.float16).astype(np.float64) if u % 2 == 0 else vv.astype(np.float16).astype(np.float64))
    x = torch.from_numpy(np.stack(xs)).half().cuda()
    ec = EngineConfig(bits=2, pattern_count=k)
    tabs = {}
    for mode in ("tc", "cuda_core"):
        if mode == "cuda_core":
            monkeypatch.setenv("PKV_MINE_CUDA_CORES", "1")
        cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + 256)
        hist, nit = cache.mine(0, x, seed=7)
        nk, _ = cache.pattern_counts()
        tabs[mode] = (cache.patterns(0)[:, :k].cpu().numpy(), hist, nit, nk)
    np.testing.assert_array_equal(tabs["tc"][0], tabs["cuda_core"][0])
    np.testing.assert_array_equal(tabs["tc"][2], tabs["cuda_core"][2])
    for u in range(U):
        cen, lab, hist = O.kmeans(xs[u], k, 7)
        assert tabs["tc"][3][u] == len(cen)
        np.testing.assert_allclose(tabs["tc"][0][u, :len(cen)], cen, rtol=0, atol=1e-12)
        assert int(tabs["tc"][2][u]) == len(hist)
        np.testing.assert_allclose(tabs["tc"][1][u, :len(hist)], hist, rtol=1e-12)


def test_long_decode_pattern_growth_vs_oracle(pkv):
    """Append-and-refresh far past the pruned-matcher range: the tables grow from 8 to
    8 + 75 patterns per side (brute-force matcher above 64, shared-W attention path),
    codes/indices stay bit-exact vs the oracle replay and attention stays within 1e-3."""
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.export import export_unit

    d, tp, G = 64, 256, 64
    steps = 75 * G + 10
    k, v = O.synth_unit(O.unit_seed(5, 5, 5), tp + steps, d)
    k = k.astype(np.float16).astype(np.float64)
    v = v.astype(np.float16).astype(np.float64)
    cfg = dict(bits=2, pattern_count=8, group_size=G, residual_window=G)
    cache = pkv.PatternKVCache(EngineConfig(**cfg), 1, d, dtype=torch.float16, max_tokens=512)
    kt = torch.from_numpy(k).half().cuda()
    vt = torch.from_numpy(v).half().cuda()
    cache.prefill(kt[None, :tp], vt[None, :tp])
    for t in range(tp, tp + steps):
        cache.append(kt[None, t], vt[None, t])
    h = O.replay(k[:tp], v[:tp], k[tp:], v[tp:], O.Knobs(**cfg))
    st = export_unit(cache, 0, with_bytes=False)
    assert len(st.kpat) == len(h.kpat) == 8 + 75
    np.testing.assert_array_equal(st.kpat, h.kpat)
    np.testing.assert_array_equal(st.k_idx, np.concatenate([b[5] for b in h.k_blocks]))
    np.testing.assert_array_equal(st.k_codes, np.concatenate([b[4] for b in h.k_blocks]))
    np.testing.assert_array_equal(st.v_idx, np.array([x[3] for x in h.v_tok]))
    np.testing.assert_array_equal(st.v_codes, np.stack([x[2] for x in h.v_tok]))
    q = np.random.default_rng(9).normal(size=(1, 4, d)).astype(np.float32)
    out = cache.decode_attention(torch.from_numpy(q).cuda()).cpu().numpy()
    ref = O.head_attention(h, q[0].astype(np.float64), 1.0 / math.sqrt(d))
    assert np.abs(out[0] - ref).max() / np.abs(ref).max() <= 1e-3


def test_decode_flush_wide_pruned_matcher_vs_oracle(pkv):
    """Decode flushes past 128 patterns per side on the pruned matcher for wide tables
    (match_pruned_wide: 4 and then 8 pattern chunks per lane, probe table in the staging
    rows): 8 + 125 patterns per side at head_dim 128, codes/indices bit-exact vs the oracle."""
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.export import export_unit

    d, tp, G = 128, 64, 16
    steps = 125 * G + 5
    k, v = O.synth_unit(O.unit_seed(6, 1, 3), tp + steps, d)
    k = k.astype(np.float16).astype(np.float64)
    v = v.astype(np.float16).astype(np.float64)
    cfg = dict(bits=4, pattern_count=8, group_size=G, residual_window=G)
    cache = pkv.PatternKVCache(EngineConfig(**cfg), 1, d, dtype=torch.float16, max_tokens=tp + steps + 64)
    kt = torch.from_numpy(k).half().cuda()
    vt = torch.from_numpy(v).half().cuda()
    cache.prefill(kt[None, :tp], vt[None, :tp])
    for t in range(tp, tp + steps):
        cache.append(kt[None, t], vt[None, t])
    h = O.replay(k[:tp], v[:tp], k[tp:], v[tp:], O.Knobs(**cfg))
    st = export_unit(cache, 0, with_bytes=False)
    assert len(st.kpat) == len(h.kpat) == 8 + 125
    np.testing.assert_array_equal(st.kpat, h.kpat)
    np.testing.assert_array_equal(st.vpat, h.vpat)
    np.testing.assert_array_equal(st.k_idx, np.concatenate([b[5] for b in h.k_blocks]))
    np.testing.assert_array_equal(st.k_codes, np.concatenate([b[4] for b in h.k_blocks]))
    np.testing.assert_array_equal(st.v_idx, np.array([x[3] for x in h.v_tok]))
    np.testing.assert_array_equal(st.v_codes, np.stack([x[2] for x in h.v_tok]))
