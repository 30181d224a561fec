"""KVTR ingestion on the GPU: the device-resident layout equals the reference reader's
arrays (unit u = layer * heads + head), non-finite payloads are reported like
read_trace, and an ingested trace encodes exactly like the oracle replay of the
reference-read stream."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pkv_oracle as O  # noqa: E402

G = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return np.load(os.path.join(G, "trace.npz"))


@pytest.mark.parametrize("name", ["f16", "f32"])
def test_device_layout(gold, tmp_path, name):
    from paper_2510_05176_b200 import trace
    p = str(tmp_path / "t.kvtr")
    open(p, "wb").write(gold[name + "_blob"].tobytes())
    ref = trace.read_trace(p)
    dt = trace.load_trace_device(p)
    L, H, T, d = ref.prefill_k.shape
    np.testing.assert_array_equal(dt.prefill_k.double().cpu().numpy(), ref.prefill_k.reshape(L * H, T, d))
    np.testing.assert_array_equal(dt.prefill_v.double().cpu().numpy(), ref.prefill_v.reshape(L * H, T, d))
    S = ref.decode_steps
    np.testing.assert_array_equal(dt.decode_k.double().cpu().numpy(),
                                  np.transpose(ref.decode_k.reshape(L * H, S, d), (1, 0, 2)))
    np.testing.assert_array_equal(dt.decode_v.double().cpu().numpy(),
                                  np.transpose(ref.decode_v.reshape(L * H, S, d), (1, 0, 2)))


def test_device_nonfinite_report(gold, tmp_path):
    from paper_2510_05176_b200 import trace
    from paper_2510_05176_b200.errors import DataError
    blob = gold["f32_blob"].tobytes()
    body = np.frombuffer(blob[29:], "<f4").copy()
    npre = 2 * 2 * 3 * 40 * 16
    body[npre + (5 * 2 + 1) * 2 * 3 * 16 + 3 * 16 + 16 + 7] = np.nan  # step 5, layer 1, V, head 1, dim 7
    p = str(tmp_path / "nan.kvtr")
    open(p, "wb").write(blob[:29] + body.tobytes())
    with pytest.raises(DataError, match="non-finite decode V element at layer 1, head 1, token 5, dim 7"):
        trace.read_trace(p)
    with pytest.raises(DataError, match="non-finite decode V element at layer 1, head 1, token 5, dim 7"):
        trace.load_trace_device(p)


def test_ingest_trace_matches_oracle(gold, tmp_path):
    from paper_2510_05176_b200 import trace
    from paper_2510_05176_b200.config import EngineConfig
    p = str(tmp_path / "t.kvtr")
    open(p, "wb").write(gold["f16_blob"].tobytes())
    cfg = EngineConfig(bits=2, pattern_count=4, group_size=16, residual_window=16)
    cache, tr = trace.ingest_trace(p, cfg)
    ref = trace.read_trace(p)
    kc, vc = cache.codes()
    knobs = O.Knobs(bits=2, pattern_count=4, group_size=16, residual_window=16)
    for u in range(tr.n_units):
        kp, vp, kd, vd = ref.head_slices(u // ref.num_heads, u % ref.num_heads)
        h = O.replay(kp, vp, kd, vd, knobs)
        np.testing.assert_array_equal(kc[u].cpu().numpy(), np.concatenate([b[4] for b in h.k_blocks]))
        np.testing.assert_array_equal(vc[u].cpu().numpy(), np.stack([x[2] for x in h.v_tok]))
