"""PKVS snapshots (reference snapshot.py) on the host: the writer and reader are
pinned to images produced by the reference's own save_snapshot
(tests/golden/snapshot.npz, make_golden.gen_snapshot):

* parse -> re-serialize reproduces every golden image byte for byte;
* the oracle's replay of the same inputs, serialized by this package's bulk writer,
  reproduces the image (the GPU test does the same from the device cache);
* malformed images raise DataError with the reference's messages, bad calls UsageError.
"""

import json
import os
import struct

import numpy as np
import pytest

from oracle import pkv_oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["k_gate", "no_vgate4", "short", "raw8"]


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(G, "snapshot.npz"))


@pytest.fixture(scope="module")
def snap():
    from paper_2510_05176_b200 import snapshot
    return snapshot


def _case(gold, name):
    p = name + "__"
    kw = json.loads(str(gold[p + "config"]))
    d, tp, td = (int(x) for x in gold[p + "dims"])
    heads = [tuple(int(v) for v in h) for h in gold[p + "heads"]]
    return kw, d, tp, td, heads, gold[p + "blob"].tobytes()


class _OracleUnit:
    """An oracle head in export.UnitState shape (what the bulk writer consumes)."""

    def __init__(self, h, bits):
        d = h.d
        self.kpat, self.vpat = h.kpat.reshape(-1, d), h.vpat.reshape(-1, d)
        self.n_prefill_k = sum(o == "prefill" for o in h.kpat_origin)
        self.n_prefill_v = sum(o == "prefill" for o in h.vpat_origin)
        self.kb_start = np.array([b[0] for b in h.k_blocks], np.int64)
        self.kb_len = np.array([b[1] for b in h.k_blocks], np.int64)
        self.k_scale = np.array([b[2] for b in h.k_blocks]).reshape(-1, d)
        self.k_zero = np.array([b[3] for b in h.k_blocks]).reshape(-1, d)
        self.k_idx = np.concatenate([b[5] for b in h.k_blocks]) if h.k_blocks else np.zeros(0, np.int32)
        self.k_bytes = [[O.pack(b[4][:, c], bits) for c in range(d)] for b in h.k_blocks]
        self.v_idx = np.array([t[3] for t in h.v_tok], np.int64)
        self.v_scale = np.array([t[0] for t in h.v_tok])
        self.v_zero = np.array([t[1] for t in h.v_tok])
        self.v_bytes = [O.pack(t[2], bits) for t in h.v_tok]
        self.window_k = np.array(h.win_k).reshape(-1, d)
        self.window_v = np.array(h.win_v).reshape(-1, d)
        self.vdec = np.array(h.vdec, np.float64).reshape(-1, 3)
        self.kdec = np.array(h.kdec, np.float64).reshape(-1, 3)
        self.token_count = h.tokens


@pytest.mark.parametrize("name", CASES)
def test_roundtrip_is_byte_exact(gold, snap, name):
    kw, d, tp, td, heads, blob = _case(gold, name)
    cfg, states = snap.parse_snapshot(blob)
    assert cfg.bits == kw["bits"] and sorted(states) == sorted((l, h) for l, h, _ in heads)
    st = next(iter(states.values()))
    assert st.head_dim == d and st.token_count == tp + td
    assert snap.snapshot_bytes(states) == blob


@pytest.mark.parametrize("name", CASES)
def test_oracle_replay_serializes_to_reference_image(gold, snap, name):
    from paper_2510_05176_b200.config import EngineConfig
    kw, d, tp, td, heads, blob = _case(gold, name)
    cfg = EngineConfig(**kw)
    knobs = O.Knobs(**kw)
    parts = [snap._header(cfg, d, len(heads))]
    for layer, head, seed in sorted(heads):
        k, v = O.synth_unit(seed, tp + td, d)
        k = k.astype(np.float16).astype(np.float64)
        v = v.astype(np.float16).astype(np.float64)
        h = O.replay(k[:tp], v[:tp], k[tp:], v[tp:], knobs)
        parts.append(snap._unit_bytes(layer, head, _OracleUnit(h, cfg.bits), cfg.bits, d))
    assert b"".join(parts) == blob


def test_malformed_images_raise_data_error(gold, snap):
    from paper_2510_05176_b200.errors import DataError
    blob = _case(gold, "short")[-1]
    with pytest.raises(DataError, match="bad magic"):
        snap.parse_snapshot(b"XKVS" + blob[4:])
    with pytest.raises(DataError, match="unsupported snapshot version 2 at byte offset 4"):
        snap.parse_snapshot(blob[:4] + struct.pack("<I", 2) + blob[8:])
    with pytest.raises(DataError, match="snapshot truncated at byte offset"):
        snap.parse_snapshot(blob[:-3])
    with pytest.raises(DataError, match="unexpected 2 trailing bytes"):
        snap.parse_snapshot(blob + b"\x00\x00")
    # first K pattern origin byte: header 4+4+30+8, state header 16, count 4
    off = 4 + 4 + (1 + 4 + 4 + 4 + 8 + 1 + 8) + 8 + 16 + 4
    bad = bytearray(blob)
    bad[off] = 7
    with pytest.raises(DataError, match=f"unknown pattern origin code 7 at byte offset {off}"):
        snap.parse_snapshot(bytes(bad))


def test_usage_errors(gold, snap, tmp_path):
    from paper_2510_05176_b200.errors import UsageError
    with pytest.raises(UsageError, match="empty cache"):
        snap.save_snapshot(str(tmp_path / "x.pkvs"), {})
    _, a = snap.parse_snapshot(_case(gold, "short")[-1])
    _, b = snap.parse_snapshot(_case(gold, "raw8")[-1])
    mixed = {(0, 0): a[(0, 0)], (9, 9): b[(0, 0)]}
    with pytest.raises(UsageError, match="share one config"):
        snap.save_snapshot(str(tmp_path / "x.pkvs"), mixed)


def test_save_load_file(gold, snap, tmp_path):
    blob = _case(gold, "k_gate")[-1]
    cfg, states = snap.parse_snapshot(blob)
    path = str(tmp_path / "s.pkvs")
    snap.save_snapshot(path, states)
    assert open(path, "rb").read() == blob
    cfg2, states2 = snap.load_snapshot(path)
    assert cfg2 == cfg and sorted(states2) == sorted(states)
