"""K1-TC (persistent tcgen05-assisted fp16 prefill encoder, pkv_encode_tc.cu)
against K1 (encode_span_kernel): every arena the encoder writes must be
bit-identical -- codes, pattern indices, fp32 and fp64 params, gate records --
on mined tables (GPU k-means) over random synthetic KV.  K1 itself is pinned
to the reference by test_gpu_parity.py; the oracle parity tests there run
through K1-TC whenever the input is fp16."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ARENAS = [("kcodes", torch.uint8), ("vcodes", torch.uint8), ("kidx", torch.int16), ("vidx", torch.int16),
          ("kparam64", torch.float64), ("vparam64", torch.float64), ("kparam32", torch.float32),
          ("vparam32", torch.float32), ("vdiag", torch.float64)]


@pytest.fixture(scope="module")
def pkv():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_05176_b200 as P
    return P


def _run(P, monkeypatch, tc, cfg, k, v, diag):
    monkeypatch.setenv("PKV_ENCODE_TC", "1" if tc else "0")
    U, T, d = k.shape
    cache = P.PatternKVCache(cfg, U, d, dtype=torch.float16, max_tokens=T + 256, record_decisions=diag, stats=True)
    cache.prefill(k, v)
    torch.cuda.synchronize()
    out = {}
    for name, dt in ARENAS:
        nb = cache.arena_bytes(name)
        if nb == 0:
            continue
        n = nb // torch.empty((), dtype=dt).element_size()
        out[name] = cache.read(name, dt, (n,)).cpu()
    out["stats"] = cache.read("stats", torch.int32, (4,)).cpu().numpy()
    return out


@pytest.mark.parametrize("bits,P,T,vgate,seed", [
    (2, 32, 4096, True, 0),
    (4, 32, 2048, True, 1),
    (2, 16, 1000, True, 2),     # short last span (872 = 6 x 128 + 104)
    (4, 8, 777, False, 3),      # --no-v-gate, short tail
    (2, 32, 2176, True, 4),
])
def test_encode_tc_matches_k1(pkv, monkeypatch, bits, P, T, vgate, seed):
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.synth import synth_kv

    U = 6
    k, v = synth_kv(U, T, 128, seed=seed)
    cfg = EngineConfig(bits=bits, pattern_count=P, use_v_gate=vgate)
    a = _run(pkv, monkeypatch, True, cfg, k, v, diag=True)
    b = _run(pkv, monkeypatch, False, cfg, k, v, diag=True)
    for name, _ in ARENAS:
        if name in a:
            ta, tb = a[name], b[name]
            if ta.dtype.is_floating_point:
                same = (ta == tb) | (torch.isnan(ta) & torch.isnan(tb))
            else:
                same = ta == tb
            bad = (~same).nonzero()
            assert bad.numel() == 0, f"{name}: {bad.numel()} mismatches, first at {bad[:5].flatten().tolist()}"
    print("tc stats [refine, exact-code, candidates, slow-extrema]:", a["stats"], "k1:", b["stats"])


def test_encode_tc_heavy_ties(pkv, monkeypatch):
    """Low-entropy data (many exact ties in d_mm and in group extrema): the
    slow paths (candidate evaluation, fp64 re-match, multi-candidate extrema)
    must agree with K1 bit for bit."""
    from paper_2510_05176_b200.config import EngineConfig

    U, T = 4, 1536
    g = torch.Generator(device="cuda").manual_seed(11)
    k = torch.randint(-3, 4, (U, T, 128), generator=g, device="cuda").half() * 0.5
    v = torch.randint(-2, 3, (U, T, 128), generator=g, device="cuda").half()
    cfg = EngineConfig(bits=2, pattern_count=32)
    a = _run(pkv, monkeypatch, True, cfg, k, v, diag=True)
    b = _run(pkv, monkeypatch, False, cfg, k, v, diag=True)
    for name, _ in ARENAS:
        if name in a:
            assert torch.equal(a[name], b[name]), name
    print("tc stats:", a["stats"])


@pytest.mark.parametrize("cap,heavy", [(3, False), (3, True), (1000, True)])
def test_encode_tc_fix_list_overflow(pkv, monkeypatch, cap, heavy):
    """Guard-band code fix-ups normally go to kfix_kernel through the cache's fix list; a list
    too small for them (PKV_FIX_CAP) sends the rest down the in-line exact path.  Either way
    every arena equals K1's bit for bit (2 and 4 bits)."""
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.synth import synth_kv

    U, T = 4, 1536
    if heavy:
        g = torch.Generator(device="cuda").manual_seed(12)
        k = torch.randint(-3, 4, (U, T, 128), generator=g, device="cuda").half() * 0.5
        v = torch.randint(-2, 3, (U, T, 128), generator=g, device="cuda").half()
    else:
        k, v = synth_kv(U, T, 128, seed=21)
    for bits in (2, 4):
        cfg = EngineConfig(bits=bits, pattern_count=32)
        monkeypatch.setenv("PKV_FIX_CAP", str(cap))
        a = _run(pkv, monkeypatch, True, cfg, k, v, diag=True)
        monkeypatch.delenv("PKV_FIX_CAP")
        b = _run(pkv, monkeypatch, False, cfg, k, v, diag=True)
        for name, _ in ARENAS:
            if name in a:
                assert torch.equal(a[name], b[name]), (bits, name)
        assert a["stats"][1] > cap, "the data must need more fix-ups than the list holds"
