"""KVTR traces (reference stream.py) on the host: writer and reader pinned to images
written by the reference itself (tests/golden/trace.npz), malformed-input errors."""

import os
import struct

import numpy as np
import pytest

G = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(G, "trace.npz"))


@pytest.fixture(scope="module")
def tr():
    from paper_2510_05176_b200 import trace
    return trace


def _stream(gold):
    from paper_2510_05176_b200.analysis import KvStream
    return KvStream(gold["prefill_k"], gold["prefill_v"], gold["decode_k"], gold["decode_v"])


@pytest.mark.parametrize("code,name", [(1, "f16"), (2, "f32")])
def test_writer_matches_reference_bytes(gold, tr, tmp_path, code, name):
    p = str(tmp_path / "t.kvtr")
    tr.write_trace(p, _stream(gold), dtype_code=code)
    assert open(p, "rb").read() == gold[name + "_blob"].tobytes()


@pytest.mark.parametrize("name", ["f16", "f32"])
def test_reader_matches_reference(gold, tr, tmp_path, name):
    p = str(tmp_path / "t.kvtr")
    open(p, "wb").write(gold[name + "_blob"].tobytes())
    s = tr.read_trace(p)
    np.testing.assert_array_equal(s.prefill_k, gold[name + "_read_prefill_k"])
    np.testing.assert_array_equal(s.decode_v, gold[name + "_read_decode_v"])
    h = tr.read_trace_header(p)
    assert (h.num_layers, h.num_heads, h.head_dim, h.prefill_len, h.decode_steps) == (2, 3, 16, 40, 12)
    assert h.dtype_name == ("float16" if name == "f16" else "float32")


def test_malformed_traces(gold, tr, tmp_path):
    from paper_2510_05176_b200.errors import DataError, UsageError
    blob = gold["f32_blob"].tobytes()
    p = str(tmp_path / "bad.kvtr")

    def check(b, msg):
        open(p, "wb").write(b)
        with pytest.raises(DataError, match=msg):
            tr.read_trace(p)

    check(blob[:10], "trace truncated inside the header: file ends at byte offset 10, header needs 29")
    check(b"KVTX" + blob[4:], "bad magic")
    check(blob[:4] + struct.pack("<I", 3) + blob[8:], "unsupported trace version 3 at byte offset 4, expected 1")
    check(blob[:8] + struct.pack("<I", 0) + blob[12:], "num_layers is 0 at byte offset 8")
    check(blob[:20] + bytes([9]) + blob[21:], "unknown dtype code 9 at byte offset 20")
    check(blob[:-4], r"trace body is \d+ bytes, expected \d+; file diverges from the format at byte offset")
    body = np.frombuffer(blob[29:], "<f4").copy()
    body[3 * 40 * 16 + 5] = np.inf  # layer 0: K [3][40][16] then V -> prefill V, head 0, token 0, dim 5
    check(blob[:29] + body.tobytes(), "non-finite prefill V element at layer 0, head 0, token 0, dim 5")
    with pytest.raises(UsageError, match="unknown trace dtype code 5"):
        tr.write_trace(p, _stream(gold), dtype_code=5)
