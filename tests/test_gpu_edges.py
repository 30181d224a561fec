"""Edge cases of the B200 path against the CPU oracle (bit-exact decisions, codes and
params; attention within 1e-3 of fp64 softmax):

* prefill no longer than the window: nothing committed (engine.py:162-165), attention over
  the exact window alone, then decode appends up to and past the first flush;
* a one-token committed span (T = W + 1) on the K1-TC envelope (fp16, d = G = 128);
* P = 64 patterns, outside K1-TC (P <= 32): the K1 span encoder;
* far more units than CTAs with one span each (work queue: fewer items per CTA than
  subgroups), K1-TC against K1;
* bf16 and fp32 inputs through prefill and decode flushes;
* head_dim 64 / 96 / 40 (the KT = 4 attention kernel, padded channels);
* cfg3's 131072-token context.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import pkv_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def pkv():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_05176_b200 as P
    return P


def _units(n, T, d, seed):
    ks, vs = [], []
    for u in range(n):
        k, v = O.synth_unit(O.unit_seed(seed, 1, u), T, d)
        ks.append(k.astype(np.float16).astype(np.float64))
        vs.append(v.astype(np.float16).astype(np.float64))
    return np.stack(ks), np.stack(vs)


def _assert_matches_oracle(cache, heads):
    from paper_2510_05176_b200.export import export_unit

    for u, h in enumerate(heads):
        st = export_unit(cache, u, with_bytes=False)
        np.testing.assert_array_equal(st.kpat, h.kpat)
        np.testing.assert_array_equal(st.vpat, h.vpat)
        assert len(st.kb_start) == len(h.k_blocks)
        if h.k_blocks:
            np.testing.assert_array_equal(st.k_idx, np.concatenate([b[5] for b in h.k_blocks]))
            np.testing.assert_array_equal(st.k_codes, np.concatenate([b[4] for b in h.k_blocks]))
            np.testing.assert_array_equal(st.k_scale, np.stack([b[2] for b in h.k_blocks]))
            np.testing.assert_array_equal(st.k_zero, np.stack([b[3] for b in h.k_blocks]))
            np.testing.assert_array_equal(st.v_idx, np.array([t[3] for t in h.v_tok]))
            np.testing.assert_array_equal(st.v_codes, np.stack([t[2] for t in h.v_tok]))
            np.testing.assert_array_equal(st.v_scale, np.array([t[0] for t in h.v_tok]))
            np.testing.assert_array_equal(st.v_zero, np.array([t[1] for t in h.v_tok]))
        np.testing.assert_array_equal(st.window_k, np.stack(h.win_k))
        np.testing.assert_array_equal(st.window_v, np.stack(h.win_v))


def _attention_close(pkv, cache, U, d, G=4, seed=3):
    q = np.random.default_rng(seed).normal(size=(U, G, d)).astype(np.float32)
    out = cache.decode_attention(torch.from_numpy(q).cuda()).cpu().numpy()
    kc, vc = cache.dequant()
    wk, wv = cache.window()
    for u in range(U):
        kall = np.concatenate([kc[u].cpu().numpy(), wk[u].double().cpu().numpy()])
        vall = np.concatenate([vc[u].cpu().numpy(), wv[u].double().cpu().numpy()])
        ref = O.attention(q[u].astype(np.float64), kall, vall, 1.0 / math.sqrt(d))
        assert np.abs(out[u] - ref).max() <= 1e-3 * np.abs(ref).max()


@pytest.mark.parametrize("T", [1, 60, 128])
def test_prefill_within_window_then_first_flush(pkv, T):
    from paper_2510_05176_b200.config import EngineConfig

    U, d = 3, 128
    S = 256 - T + 5  # past the first flush at len == W + G (engine.py:186)
    ec = EngineConfig(bits=2, pattern_count=8)
    k, v = _units(U, T + S, d, seed=T)
    heads = [O.replay(k[u, :T], v[u, :T], k[u, T:T + S], v[u, T:T + S], O.Knobs(bits=2, pattern_count=8))
             for u in range(U)]
    cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + S + 256)
    kt, vt = torch.from_numpy(k).half().cuda(), torch.from_numpy(v).half().cuda()
    cache.prefill(kt[:, :T], vt[:, :T])
    assert cache.info().committed_count == 0
    _attention_close(pkv, cache, U, d)
    for t in range(T, T + S):
        cache.append(kt[:, t], vt[:, t])
    assert cache.info().committed_count == heads[0].committed > 0
    _assert_matches_oracle(cache, heads)
    _attention_close(pkv, cache, U, d)


@pytest.mark.parametrize("bits", [2, 4])
def test_one_token_span(pkv, bits):
    """T = W + 1: the prefill commits a single-token span (K groups of one element)."""
    from paper_2510_05176_b200.config import EngineConfig

    U, d, T = 4, 128, 129
    ec = EngineConfig(bits=bits, pattern_count=16)
    k, v = _units(U, T, d, seed=40 + bits)
    heads = [O.replay(k[u], v[u], k[u, :0], v[u, :0], O.Knobs(bits=bits, pattern_count=16)) for u in range(U)]
    cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + 256)
    cache.prefill(torch.from_numpy(k).half().cuda(), torch.from_numpy(v).half().cuda())
    assert cache.info().committed_count == 1
    _assert_matches_oracle(cache, heads)


def test_sixty_four_patterns_span_encoder(pkv):
    """P = 64 (K1-TC serves P <= 32): the K1 span encoder, fp16, against the oracle."""
    from paper_2510_05176_b200.config import EngineConfig

    U, d, T = 2, 128, 1100
    ec = EngineConfig(bits=2, pattern_count=64)
    k, v = _units(U, T, d, seed=64)
    heads = [O.replay(k[u], v[u], k[u, :0], v[u, :0], O.Knobs(bits=2, pattern_count=64)) for u in range(U)]
    cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + 256)
    cache.prefill(torch.from_numpy(k).half().cuda(), torch.from_numpy(v).half().cuda())
    _assert_matches_oracle(cache, heads)


def test_many_units_one_span_each(pkv, monkeypatch):
    """600 units x one 128-token span: fewer queue items per CTA than subgroups; K1-TC == K1
    on the codes and the exact fp64 reconstruction (params, indices, codes)."""
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.synth import synth_kv

    U, T = 600, 256
    ec = EngineConfig(bits=2, pattern_count=16)
    k, v = synth_kv(U, T, 128, seed=5)
    out = []
    for tc in ("1", "0"):
        monkeypatch.setenv("PKV_ENCODE_TC", tc)
        cache = pkv.PatternKVCache(ec, U, 128, dtype=torch.float16, max_tokens=T + 256)
        cache.prefill(k, v)
        kc, vc = cache.codes()
        kd, vd = cache.dequant()
        out.append((kc.cpu(), vc.cpu(), kd.cpu(), vd.cpu()))
        del cache
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("tdt", [torch.bfloat16, torch.float32])
def test_bf16_fp32_inputs_prefill_decode(pkv, tdt):
    """bf16 / fp32 caches (the K1 span encoder; K1-TC is fp16-only): prefill + decode flushes
    bit-exact vs the oracle on the same (rounded) inputs, attention within 1e-3."""
    from paper_2510_05176_b200.config import EngineConfig

    U, d, T, S = 3, 128, 700, 150
    ec = EngineConfig(bits=4, pattern_count=16)
    ks, vs = [], []
    for u in range(U):
        k, v = O.synth_unit(O.unit_seed(77, 2, u), T + S, d)
        ks.append(torch.from_numpy(k).to(tdt))
        vs.append(torch.from_numpy(v).to(tdt))
    kt, vt = torch.stack(ks), torch.stack(vs)
    k64, v64 = kt.double().numpy(), vt.double().numpy()
    heads = [O.replay(k64[u, :T], v64[u, :T], k64[u, T:], v64[u, T:], O.Knobs(bits=4, pattern_count=16))
             for u in range(U)]
    cache = pkv.PatternKVCache(ec, U, d, dtype=tdt, max_tokens=T + S + 256)
    kt, vt = kt.cuda(), vt.cuda()
    cache.prefill(kt[:, :T], vt[:, :T])
    for t in range(T, T + S):
        cache.append(kt[:, t], vt[:, t])
    _assert_matches_oracle(cache, heads)
    _attention_close(pkv, cache, U, d)


@pytest.mark.parametrize("d,bits,gqa", [(64, 2, 4), (96, 4, 8), (40, 2, 2), (42, 4, 3)])
def test_small_head_dims(pkv, d, bits, gqa):
    """head_dim < 128: Dp = 64 (the KT = 4 attention kernel) or padded channels (96 -> 128,
    40 -> 64, 42 -> 64: the window merge's scalar-load path, D % 4 != 0, and a run-time head
    count); fp16 caches off the K1-TC envelope, bit-exact vs the oracle, attention 1e-3."""
    from paper_2510_05176_b200.config import EngineConfig

    U, T, S = 2, 600, 140
    ec = EngineConfig(bits=bits, pattern_count=12)
    k, v = _units(U, T + S, d, seed=d)
    heads = [O.replay(k[u, :T], v[u, :T], k[u, T:], v[u, T:], O.Knobs(bits=bits, pattern_count=12))
             for u in range(U)]
    cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + S + 256)
    kt, vt = torch.from_numpy(k).half().cuda(), torch.from_numpy(v).half().cuda()
    cache.prefill(kt[:, :T], vt[:, :T])
    for t in range(T, T + S):
        cache.append(kt[:, t], vt[:, t])
    _assert_matches_oracle(cache, heads)
    _attention_close(pkv, cache, U, d, G=gqa)


def test_long_context_cfg3_length(pkv, monkeypatch):
    """cfg3's 131072-token context (1023 spans per unit): K1-TC == K1 on codes and the exact fp64
    reconstruction, and attention within 1e-3 of fp64 softmax over it (torch fp64 on the device;
    the numpy oracle is too slow at this length)."""
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.synth import synth_kv

    U, T, d, G = 2, 131072, 128, 4
    ec = EngineConfig(bits=2, pattern_count=32)
    k, v = synth_kv(U, T, d, seed=131)
    res = []
    for tc in ("1", "0"):
        monkeypatch.setenv("PKV_ENCODE_TC", tc)
        cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + 256)
        cache.prefill(k, v)
        kc, vc = cache.codes()
        kd, vd = cache.dequant()
        res.append((kc, vc, kd, vd))
        if tc == "1":
            q = torch.randn((U, G, d), device="cuda", dtype=torch.float32)
            out = cache.decode_attention(q).double()
            wk, wv = cache.window()
            for u in range(U):
                kall = torch.cat([kd[u], wk[u].double()])
                vall = torch.cat([vd[u], wv[u].double()])
                ref = torch.softmax(q[u].double() @ kall.T / math.sqrt(d), dim=-1) @ vall
                assert (out[u] - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()
        del cache
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)


def test_reset_then_decode_only(pkv):
    """pkv_cache_reset after a prefill with a short tail block, then decode appends with no new
    prefill: the first flush starts a fresh block table at token 0 (no stale prefill geometry)
    and equals an oracle head that holds the same pattern tables and only appends."""
    from paper_2510_05176_b200.config import EngineConfig

    d, tp, steps = 128, 700, 300  # 572 committed = 4 full blocks + a 60-token tail
    k, v = _units(2, tp + steps, d, seed=21)
    cfg = dict(bits=2, pattern_count=16)
    cache = pkv.PatternKVCache(EngineConfig(**cfg), 2, d, dtype=torch.float16, max_tokens=1024)
    kt = torch.from_numpy(k).half().cuda()
    vt = torch.from_numpy(v).half().cuda()
    cache.prefill(kt[:, :tp], vt[:, :tp])
    pats = [cache.patterns(s)[:, :16].cpu().numpy() for s in (0, 1)]
    cache.reset(keep_patterns=True)
    for t in range(tp, tp + steps):
        cache.append(kt[:, t], vt[:, t])
    heads = []
    for u in range(2):
        h = O.OracleHead(O.Knobs(**cfg), d)
        h.kpat, h.vpat = pats[0][u].copy(), pats[1][u].copy()
        for t in range(tp, tp + steps):
            h.append(k[u, t], v[u, t])
        heads.append(h)
    assert cache.info().n_blocks == 1 and cache.block_table()[0].tolist() == [0]
    _assert_matches_oracle(cache, heads)


@pytest.mark.parametrize("dtype", ["float16", "float32"])
def test_fused_nonfinite_detection(pkv, dtype):
    """engine.py:136-138 / 180-181 fused into the kernels: K1-TC's tensor-core scores (fp16) /
    K1's staging (fp32) and the window copy flag the first non-finite element -- lowest unit,
    K before V, then token, dim -- and it surfaces as DataError with the reference's message,
    deferred (check(), the next append) or at once (sync_check); reset clears it."""
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.errors import DataError

    tdt = getattr(torch, dtype)
    U, T, d = 3, 1000, 128
    k, v = _units(U, T + 4, d, seed=31)
    cfg = EngineConfig(bits=2, pattern_count=16)
    cache = pkv.PatternKVCache(cfg, U, d, dtype=tdt, max_tokens=2048)
    kt = torch.from_numpy(k).to("cuda", tdt)
    vt = torch.from_numpy(v).to("cuda", tdt)
    # committed-span elements (encoder) and a window element
    kt2, vt2 = kt.clone(), vt.clone()
    vt2[1, 500, 7] = float("nan")
    kt2[2, 100, 3] = float("inf")
    kt2[1, T - 5, 9] = -float("inf")  # window row of unit 1: K before V wins within the unit
    cache.prefill(kt2[:, :T], vt2[:, :T])
    torch.cuda.synchronize()
    with pytest.raises(DataError, match=r"non-finite prefill K element at token 995, dim 9 \(unit 1\)"):
        cache.check()
    with pytest.raises(DataError):
        cache.append(kt[:, T], vt[:, T])  # a flagged cache refuses appends
    # committed-span only
    cache.reset(keep_patterns=False)
    vt3 = vt.clone()
    vt3[0, 300, 127] = float("nan")
    with pytest.raises(DataError, match=r"non-finite prefill V element at token 300, dim 127 \(unit 0\)"):
        cache.prefill(kt[:, :T], vt3[:, :T], sync_check=True)
    # clean prefill, then a non-finite decode vector
    cache.reset(keep_patterns=False)
    cache.prefill(kt[:, :T], vt[:, :T], sync_check=True)
    bad_k = kt[:, T].clone()
    bad_k[2, 5] = float("nan")
    cache.append(bad_k, vt[:, T])
    with pytest.raises(DataError, match=rf"non-finite decode vector at token {T} \(unit 2\)"):
        cache.check()
    # the clean path stays clean
    cache.reset(keep_patterns=False)
    cache.prefill(kt[:, :T], vt[:, :T], sync_check=True)
    for t in range(T, T + 4):
        cache.append(kt[:, t], vt[:, t], sync_check=True)


@pytest.mark.parametrize("d,gqa,dt", [(128, 4, torch.float16), (42, 3, torch.float16), (64, 8, torch.float32)])
def test_long_window_merge_tiles(pkv, d, gqa, dt):
    """A residual window longer than the merge kernel's 1024-row score tile (online softmax across
    window tiles, ring wrap after appends): attention within 1e-3 of fp64 softmax; vector-load
    (d % 4 == 0) and scalar paths, compile-time and run-time head counts, fp16 and fp32 rows."""
    from paper_2510_05176_b200.config import EngineConfig

    U, T, S = 2, 2900, 300
    ec = EngineConfig(bits=2, pattern_count=8, group_size=128, residual_window=1500)
    k, v = _units(U, T + S, d, seed=7 + d)
    cache = pkv.PatternKVCache(ec, U, d, dtype=dt, max_tokens=T + S + 256)
    kt, vt = torch.from_numpy(k).to(dt).cuda(), torch.from_numpy(v).to(dt).cuda()
    cache.prefill(kt[:, :T], vt[:, :T])
    assert cache.info().window_len > 1024
    _attention_close(pkv, cache, U, d, G=gqa)
    for t in range(T, T + S):
        cache.append(kt[:, t], vt[:, t])
    assert cache.info().window_len > 1024 and cache.info().window_slot0 > 0
    _attention_close(pkv, cache, U, d, G=gqa, seed=5)
