"""K3-TC (tcgen05 kind::i8 decode attention, pkv_attn_tc.cu) against fp64 softmax attention
over the exact reconstruction (`committed_matrices` + window, engine.py:255-303), and against
the CUDA-core K3 (PKV_ATTN_TC=0).  Tolerance: max-abs error <= 1e-3 x max|ref| per unit.

Covers 2/4-bit, GQA 1..8 (N = 16 and 32 MMA columns), K groups of 128 and 64 tokens (8 and 4
tiles per block), V pattern tables past one 128-row one-hot tile (decode growth to > 128
patterns), peaked softmax (rescale / V-exponent flush path), raw tokens, and chunked contexts.
"""
import math
import os

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


def _cache(pkv, U, T, steps, d, seed, **kw):
    from paper_2510_05176_b200.config import EngineConfig

    ec = EngineConfig(**kw)
    ks, vs = [], []
    for u in range(U):
        k, v = O.synth_unit(O.unit_seed(seed, 3, u), T + steps, d)
        ks.append(k)
        vs.append(v)
    kt = torch.from_numpy(np.stack(ks)).half().cuda()
    vt = torch.from_numpy(np.stack(vs)).half().cuda()
    cache = pkv.PatternKVCache(ec, U, d, dtype=torch.float16, max_tokens=T + steps + 512)
    cache.prefill(kt[:, :T], vt[:, :T])
    for t in range(T, T + steps):
        cache.append(kt[:, t], vt[:, t])
    return cache


def _ref(cache, q, d):
    kc, vc = cache.dequant()
    wk, wv = cache.window()
    out = []
    for u in range(q.shape[0]):
        kall = np.concatenate([kc[u].cpu().numpy(), wk[u].double().cpu().numpy()])
        vall = np.concatenate([vc[u].cpu().numpy(), wv[u].double().cpu().numpy()])
        out.append(O.attention(q[u].astype(np.float64), kall, vall, 1.0 / math.sqrt(d)))
    return np.stack(out)


def _attend(cache, q, tc: bool):
    old = os.environ.get("PKV_ATTN_TC")
    os.environ["PKV_ATTN_TC"] = "1" if tc else "0"
    try:
        return cache.decode_attention(torch.from_numpy(q).cuda()).cpu().numpy()
    finally:
        if old is None:
            del os.environ["PKV_ATTN_TC"]
        else:
            os.environ["PKV_ATTN_TC"] = old


def _check(out, ref, tag):
    for u in range(ref.shape[0]):
        err = np.abs(out[u] - ref[u]).max() / np.abs(ref[u]).max()
        print(f"{tag} unit={u} max-abs err / max|ref| = {err:.3e}")
        assert err <= 1e-3, (tag, u, err)


@pytest.mark.parametrize("bits", [2, 4])
@pytest.mark.parametrize("gqa", [1, 4, 7, 8])
def test_tc_attention_vs_fp64(pkv, bits, gqa):
    d = 128
    cache = _cache(pkv, 3, 2100, 140, d, 11, bits=bits, pattern_count=16)
    q = np.random.default_rng(gqa).normal(size=(3, gqa, d)).astype(np.float32)
    ref = _ref(cache, q, d)
    _check(_attend(cache, q, True), ref, f"tc bits={bits} gqa={gqa}")
    _check(_attend(cache, q, False), ref, f"legacy bits={bits} gqa={gqa}")


@pytest.mark.parametrize("bits", [2, 4])
def test_tc_group64_peaked(pkv, bits):
    """4-tile blocks (G = 64) and a peaked softmax (q x 8: repeated rescales / flushes)."""
    d = 128
    cache = _cache(pkv, 2, 1700, 100, d, 12, bits=bits, pattern_count=32, group_size=64, residual_window=64)
    q = 8.0 * np.random.default_rng(3).normal(size=(2, 4, d)).astype(np.float32)
    ref = _ref(cache, q, d)
    _check(_attend(cache, q, True), ref, f"tc G=64 peaked bits={bits}")


def test_tc_pattern_growth_past_one_onehot_tile(pkv):
    """generate_new_patterns over a long decode: the V table grows past 128 rows (two
    one-hot M tiles) and the K table past the prefill count."""
    d = 128
    cache = _cache(pkv, 1, 600, 128 * 130, d, 13, bits=2, pattern_count=8)
    q = np.random.default_rng(4).normal(size=(1, 4, d)).astype(np.float32)
    ref = _ref(cache, q, d)
    _check(_attend(cache, q, True), ref, "tc P>128")


@pytest.mark.parametrize("bits", [2, 4])
def test_tc_raw_scheme(pkv, bits):
    """Patterns off on both sides (every index RAW, no one-hot tile)."""
    d = 128
    cache = _cache(pkv, 2, 1500, 60, d, 14, bits=bits, pattern_count=16, use_k_patterns=False,
                   use_v_patterns=False, generate_new_patterns=False)
    q = np.random.default_rng(5).normal(size=(2, 4, d)).astype(np.float32)
    _check(_attend(cache, q, True), _ref(cache, q, d), f"tc raw bits={bits}")


def test_tc_kernel_is_the_one_that_runs(pkv):
    d = 128
    cache = _cache(pkv, 1, 800, 0, d, 15, bits=2, pattern_count=16)
    q = torch.randn(1, 4, d).cuda()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        cache.decode_attention(q)
        torch.cuda.synchronize()
    names = [e.key for e in prof.key_averages()]
    assert any("attn_tc_kernel" in n for n in names), names
