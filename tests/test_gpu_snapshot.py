"""PKVS images written from the B200 cache equal the reference's save_snapshot
bytes for the same inputs (tests/golden/snapshot.npz): a multi-unit device cache
(prefill + decode appends through the C ABI) and the per-head facade."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pkv_oracle as O  # noqa: E402

G = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["k_gate", "no_vgate4", "short", "raw8"]


@pytest.fixture(scope="module")
def gold():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return np.load(os.path.join(G, "snapshot.npz"))


def _inputs(gold, name):
    p = name + "__"
    kw = json.loads(str(gold[p + "config"]))
    d, tp, td = (int(x) for x in gold[p + "dims"])
    heads = [tuple(int(v) for v in h) for h in gold[p + "heads"]]
    ks, vs = [], []
    for _, _, seed in heads:
        k, v = O.synth_unit(seed, tp + td, d)
        ks.append(k.astype(np.float16).astype(np.float64))
        vs.append(v.astype(np.float16).astype(np.float64))
    return kw, d, tp, td, heads, np.stack(ks), np.stack(vs), gold[p + "blob"].tobytes()


@pytest.mark.parametrize("dtype", [torch.float16, torch.float64])
@pytest.mark.parametrize("name", CASES)
def test_device_cache_snapshot_matches_reference(gold, name, dtype):
    import paper_2510_05176_b200 as P
    from paper_2510_05176_b200 import snapshot
    kw, d, tp, td, heads, k, v, blob = _inputs(gold, name)
    cfg = P.EngineConfig(**kw)
    cache = P.PatternKVCache(cfg, len(heads), d, dtype=dtype, max_tokens=tp + td + 256, record_decisions=True)
    kt = torch.from_numpy(k).to(dtype).cuda()
    vt = torch.from_numpy(v).to(dtype).cuda()
    cache.prefill(kt[:, :tp], vt[:, :tp])
    for t in range(tp, tp + td):
        cache.append(kt[:, t], vt[:, t])
    got = snapshot.cache_snapshot_bytes(cache, [(l, h) for l, h, _ in heads])
    assert len(got) == len(blob)
    assert got == blob


def test_facade_states_snapshot_matches_reference(gold, tmp_path):
    from paper_2510_05176_b200 import engine, snapshot
    kw, d, tp, td, heads, k, v, blob = _inputs(gold, "short")
    cfg = engine.EngineConfig(**kw)
    states = {(l, h): engine.replay_head(k[i, :tp], v[i, :tp], k[i, tp:], v[i, tp:], cfg)
              for i, (l, h, _) in enumerate(heads)}
    path = str(tmp_path / "f.pkvs")
    snapshot.save_snapshot(path, states)
    assert open(path, "rb").read() == blob


@pytest.mark.parametrize("dtype", [torch.float16, torch.float64])
@pytest.mark.parametrize("name", CASES)
def test_restore_roundtrip(gold, name, dtype):
    """load_snapshot -> restore_cache (pkv_cache_import) -> the device cache writes the same image."""
    from paper_2510_05176_b200 import snapshot
    kw, d, tp, td, heads, k, v, blob = _inputs(gold, name)
    _, states = snapshot.parse_snapshot(blob)
    cache, keys = snapshot.restore_cache(states, dtype=dtype)
    assert snapshot.cache_snapshot_bytes(cache, keys) == blob


@pytest.mark.parametrize("name", ["k_gate", "short", "no_vgate4"])
def test_resume_decoding_matches_oracle(gold, name):
    """Restore mid-stream, keep appending (flushes, pattern refresh) and compare with the
    oracle replaying the whole stream from scratch."""
    from paper_2510_05176_b200 import snapshot
    from test_snapshot import _OracleUnit
    kw, d, tp, td, heads, k, v, blob = _inputs(gold, name)
    extra = 300
    ke, ve = [], []
    for _, _, seed in heads:
        a, b = O.synth_unit(seed + 7919, extra, d)
        ke.append(a.astype(np.float16).astype(np.float64))
        ve.append(b.astype(np.float16).astype(np.float64))
    ke, ve = np.stack(ke), np.stack(ve)
    _, states = snapshot.parse_snapshot(blob)
    cache, keys = snapshot.restore_cache(states, dtype=torch.float64)
    kt, vt = torch.from_numpy(ke).cuda(), torch.from_numpy(ve).cuda()
    for t in range(extra):
        cache.append(kt[:, t], vt[:, t])
    got = snapshot.cache_snapshot_bytes(cache, keys)
    from paper_2510_05176_b200.config import EngineConfig
    cfg = EngineConfig(**kw)
    knobs = O.Knobs(**kw)
    parts = [snapshot._header(cfg, d, len(heads))]
    order = sorted(range(len(heads)), key=lambda i: heads[i][:2])
    for i in order:
        h = O.replay(k[i, :tp], v[i, :tp], np.concatenate([k[i, tp:], ke[i]]), np.concatenate([v[i, tp:], ve[i]]), knobs)
        parts.append(snapshot._unit_bytes(heads[i][0], heads[i][1], _OracleUnit(h, cfg.bits), cfg.bits, d))
    assert got == b"".join(parts)


def test_mixed_prefill_pattern_counts():
    """Units that mine different numbers of patterns (one has only 5 distinct rows, so
    patterns.py:95-101 returns 5 centroids) keep per-unit origin tags: the decode-appended
    patterns of the short unit are tagged "decode" from index 5 on, the image equals the
    oracle-built one, and it restores and round-trips."""
    import paper_2510_05176_b200 as P
    from paper_2510_05176_b200 import snapshot
    from test_snapshot import _OracleUnit

    d, tp, td = 64, 512, 300
    kw = dict(bits=2, pattern_count=16, group_size=128, residual_window=128)
    k0, v0 = O.synth_unit(O.unit_seed(1, 2, 3), tp + td, d)
    k1, v1 = O.synth_unit(O.unit_seed(4, 5, 6), tp + td, d)
    rows = np.random.default_rng(3).integers(0, 5, size=tp)
    k1[:tp] = k1[rows]
    v1[:tp] = v1[rows]
    k = np.stack([k0, k1]).astype(np.float16).astype(np.float64)
    v = np.stack([v0, v1]).astype(np.float16).astype(np.float64)
    cfg = P.EngineConfig(**kw)
    cache = P.PatternKVCache(cfg, 2, d, dtype=torch.float64, max_tokens=tp + td + 256, record_decisions=True)
    kt, vt = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    cache.prefill(kt[:, :tp], vt[:, :tp])
    for t in range(tp, tp + td):
        cache.append(kt[:, t], vt[:, t])
    npk, npv = cache.prefill_pattern_counts
    assert list(npk) == [16, 5] and list(npv) == [16, 5]
    keys = [(0, 0), (0, 1)]
    got = snapshot.cache_snapshot_bytes(cache, keys)
    knobs = O.Knobs(**kw)
    parts = [snapshot._header(cfg, d, 2)]
    for i in range(2):
        h = O.replay(k[i, :tp], v[i, :tp], k[i, tp:], v[i, tp:], knobs)
        parts.append(snapshot._unit_bytes(0, i, _OracleUnit(h, cfg.bits), cfg.bits, d))
    assert got == b"".join(parts)
    _, states = snapshot.parse_snapshot(got)
    cache2, keys2 = snapshot.restore_cache(states, dtype=torch.float64)
    assert snapshot.cache_snapshot_bytes(cache2, keys2) == got
