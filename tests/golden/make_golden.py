"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Every fixture is produced by the reference package itself (imported
read-only), so the oracle (oracle/pkv_oracle.py) and the GPU path are
both pinned against the reference's own outputs.  The files are small
(.npz, compressed) and committed; the GPU box never needs the reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from patternkv import analysis, engine, gate, patterns, quant  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)


def gen_quant():
    rng = np.random.default_rng(1234)
    out = {}
    for bits in (2, 4, 8):
        vals, offs, scales, zeros, codes, packed, plen = [], [0], [], [], [], [], [0]
        for trial in range(300):
            n = int(rng.integers(1, 300))
            x = rng.normal(0.0, 10.0 ** rng.uniform(-4, 4), n) + rng.uniform(-5, 5)
            if trial % 25 == 0:
                x[:] = x[0]
            elif trial % 25 == 1:
                x = np.round(x)
            g = quant.quantize_group(x, bits)
            vals.append(x)
            offs.append(offs[-1] + n)
            scales.append(g.params.scale)
            zeros.append(g.params.zero_point)
            codes.append(quant.unpack_codes(g.codes, n, bits))
            packed.append(np.frombuffer(g.codes, np.uint8))
            plen.append(plen[-1] + len(g.codes))
        out[f"b{bits}_values"] = np.concatenate(vals)
        out[f"b{bits}_offsets"] = np.array(offs, np.int64)
        out[f"b{bits}_scale"] = np.array(scales)
        out[f"b{bits}_zero"] = np.array(zeros)
        out[f"b{bits}_codes"] = np.concatenate(codes)
        out[f"b{bits}_packed"] = np.concatenate(packed)
        out[f"b{bits}_packed_offsets"] = np.array(plen, np.int64)
    save("quant.npz", **out)


def gen_match():
    rng = np.random.default_rng(99)
    out = {}
    for case, (n, p, d) in enumerate([(200, 16, 128), (150, 37, 64), (64, 5, 8), (40, 3, 3)]):
        x = rng.normal(size=(n, d)) * rng.uniform(0.1, 10.0, size=d)
        m = x[rng.integers(0, n, p)] + rng.normal(0, 0.3, size=(p, d))
        if case == 2:
            m[1] = m[0] + 2.5  # shift-invariant exact tie: lowest index must win
            x[:8] = m[0] + 1.0
        ps = patterns.PatternSet(d)
        for row in m:
            ps.append(row, patterns.ORIGIN_PREFILL)
        idx, res, dist = patterns.match_many(x, ps)
        out[f"c{case}_x"] = x
        out[f"c{case}_m"] = m
        out[f"c{case}_idx"] = idx.astype(np.int64)
        out[f"c{case}_dist"] = dist
        out[f"c{case}_res"] = res
    save("match.npz", **out)


def gen_kmeans():
    rng = np.random.default_rng(7)
    out = {}
    cases = [(300, 8, 4, 0), (1000, 64, 16, 3), (512, 128, 32, 11), (6, 4, 8, 5), (2048, 128, 16, 1)]
    for i, (n, d, k, seed) in enumerate(cases):
        if i == 3:
            x = np.repeat(rng.normal(size=(3, d)), 2, axis=0)  # 3 distinct rows <= k
        else:
            cen = rng.normal(0, 5, size=(k + 3, d))
            x = cen[rng.integers(0, k + 3, n)] + rng.normal(0, 0.5, size=(n, d))
            x = x.astype(np.float16).astype(np.float64)
        c, lab, hist = patterns.lloyd_kmeans(x, k, seed)
        out[f"c{i}_x"] = x
        out[f"c{i}_k"] = np.int64(k)
        out[f"c{i}_seed"] = np.int64(seed)
        out[f"c{i}_first"] = np.int64(np.random.default_rng(seed).integers(n))
        out[f"c{i}_centers"] = c
        out[f"c{i}_labels"] = lab.astype(np.int64)
        out[f"c{i}_hist"] = np.array(hist)
    save("kmeans.npz", **out)


def gen_gate():
    dims = np.array([4, 8, 16, 32, 64, 128, 256])
    alphas = np.array([0.01, 0.025, 0.05, 0.1, 0.25, 0.5])
    thr = np.full((len(dims), len(alphas)), np.nan)
    for i, d in enumerate(dims):
        for j, a in enumerate(alphas):
            try:
                thr[i, j] = gate.contraction_threshold(int(d), float(a))
            except ValueError:
                pass
    z = np.array([gate.z_quantile(float(a)) for a in alphas])
    save("gate.npz", dims=dims, alphas=alphas, thr=thr, z=z)


def synth_spec(seed, tokens, d, drift=None, clusters=32, spread=5.0, within=0.2, consistency=0.9, vocab=1024):
    return analysis.SyntheticStreamSpec(
        layers=1, heads=1, head_dim=d, prefill_len=tokens, decode_len=0,
        k_model=analysis.KeyModel(outlier_channels=(3,), outlier_multipliers=(32.0,),
                                  drift_rate=(1.0 / tokens if drift is None else drift), noise_std=0.05),
        v_model=analysis.ValueModel(cluster_count=clusters, center_spread=spread, within_std=within,
                                    consistency=consistency, vocab_size=vocab),
        seed=seed,
    )


def gen_synth():
    out = {}
    for i, (seed, t, d) in enumerate([(0, 300, 128), (1_000_003 * 3 + 1_009 * 5 + 2, 257, 64)]):
        s = analysis.generate_synthetic_stream(synth_spec(seed, t, d))
        out[f"c{i}_seed"] = np.int64(seed)
        out[f"c{i}_k"] = s.prefill_k[0, 0]
        out[f"c{i}_v"] = s.prefill_v[0, 0]
    save("synth.npz", **out)


def state_arrays(st, prefix, out):
    cfg = st.config
    d = st.head_dim
    out[prefix + "kpat"] = st.k_patterns.matrix
    out[prefix + "vpat"] = st.v_patterns.matrix
    out[prefix + "kpat_decode"] = np.array([st.k_patterns.origin(i) == "decode" for i in range(len(st.k_patterns))])
    out[prefix + "vpat_decode"] = np.array([st.v_patterns.origin(i) == "decode" for i in range(len(st.v_patterns))])
    out[prefix + "kb_start"] = np.array([b.start_token for b in st.k_blocks], np.int64)
    out[prefix + "kb_len"] = np.array([b.length for b in st.k_blocks], np.int64)
    if st.k_blocks:
        out[prefix + "k_scale"] = np.concatenate([[g.params.scale for g in b.channel_groups] for b in st.k_blocks])
        out[prefix + "k_zero"] = np.concatenate([[g.params.zero_point for g in b.channel_groups] for b in st.k_blocks])
        out[prefix + "k_codes"] = np.concatenate(
            [np.stack([quant.unpack_codes(g.codes, b.length, cfg.bits) for g in b.channel_groups], axis=1)
             for b in st.k_blocks])
        out[prefix + "k_bytes"] = np.frombuffer(b"".join(g.codes for b in st.k_blocks for g in b.channel_groups), np.uint8)
        out[prefix + "k_idx"] = np.concatenate([b.pattern_indices for b in st.k_blocks]).astype(np.int64)
        out[prefix + "v_scale"] = np.array([t.group.params.scale for t in st.v_tokens])
        out[prefix + "v_zero"] = np.array([t.group.params.zero_point for t in st.v_tokens])
        out[prefix + "v_codes"] = np.stack([quant.unpack_codes(t.group.codes, d, cfg.bits) for t in st.v_tokens])
        out[prefix + "v_bytes"] = np.frombuffer(b"".join(t.group.codes for t in st.v_tokens), np.uint8)
        out[prefix + "v_idx"] = np.array([t.pattern_index for t in st.v_tokens], np.int64)
        kc, vc = engine.committed_matrices(st)
        out[prefix + "k_hat"] = kc
        out[prefix + "v_hat"] = vc
    out[prefix + "vdec"] = np.array([[x.raw_range, x.flat_range, float(x.flatten), x.ratio] for x in st.v_decisions]).reshape(-1, 4)
    out[prefix + "kdec"] = np.array([[x.raw_range, x.flat_range, float(x.flatten), x.ratio] for x in st.k_decisions]).reshape(-1, 4)
    out[prefix + "window_k"] = np.array(st.window_k).reshape(-1, d)
    out[prefix + "window_v"] = np.array(st.window_v).reshape(-1, d)
    out[prefix + "token_count"] = np.int64(st.token_count)


ENGINE_CASES = {
    # name: (seed, d, prefill, decode, EngineConfig kwargs)
    "default2": (5, 128, 700, 300, dict(bits=2, pattern_count=16)),
    "four_bit": (6, 128, 520, 260, dict(bits=4, pattern_count=16)),
    "g64": (7, 64, 300, 200, dict(bits=2, pattern_count=8, group_size=64, residual_window=96)),
    "k_gate": (8, 64, 400, 140, dict(bits=2, pattern_count=8, use_k_gate=True)),
    "no_vgate": (9, 64, 400, 140, dict(bits=4, pattern_count=8, use_v_gate=False)),
    "raw": (10, 64, 400, 140, dict(bits=2, pattern_count=8, use_k_patterns=False, use_v_patterns=False,
                                   generate_new_patterns=False)),
    "no_new": (11, 128, 400, 300, dict(bits=2, pattern_count=8, generate_new_patterns=False)),
    "eight_bit": (12, 32, 300, 140, dict(bits=8, pattern_count=4, group_size=32, residual_window=32)),
    "short": (13, 16, 100, 60, dict(bits=2, pattern_count=4)),
}


def gen_engine():
    out = {}
    for name, (seed, d, tp, td, kw) in ENGINE_CASES.items():
        s = analysis.generate_synthetic_stream(synth_spec(seed, tp + td, d))
        k = s.prefill_k[0, 0].astype(np.float16).astype(np.float64)
        v = s.prefill_v[0, 0].astype(np.float16).astype(np.float64)
        cfg = engine.EngineConfig(**kw)
        st = engine.replay_head(k[:tp], v[:tp], k[tp:], v[tp:], cfg)
        p = name + "__"
        out[p + "seed"] = np.int64(seed)
        out[p + "d"] = np.int64(d)
        out[p + "prefill"] = np.int64(tp)
        out[p + "decode"] = np.int64(td)
        out[p + "config"] = np.array(json.dumps(kw))
        # prefill-only state too (no decode), for the prefill parity test
        st0 = engine.prefill(k[:tp], v[:tp], cfg)
        state_arrays(st0, p + "pre_", out)
        state_arrays(st, p + "fin_", out)
    save("engine.npz", **out)


def gen_acceptance():
    """test_acceptance.py:186-196 clustered_spec(2048, 2048) instance."""
    spec = analysis.SyntheticStreamSpec(
        layers=1, heads=1, head_dim=64, prefill_len=2048, decode_len=2048,
        k_model=analysis.KeyModel(outlier_channels=(3,), outlier_multipliers=(32.0,), drift_rate=1e-3, noise_std=0.05),
        v_model=analysis.ValueModel(cluster_count=8, center_spread=10.0, within_std=0.1, consistency=1.0),
        seed=11,
    )
    stream = analysis.generate_synthetic_stream(spec)
    cfg = engine.EngineConfig(bits=2, pattern_count=32, group_size=128, residual_window=128, seed=11)
    raw, pkv = engine.run_scheme_comparison(stream, [("patternkv", cfg)])
    kp, vp, kd, vd = stream.head_slices(0, 0)
    st = engine.replay_head(kp, vp, kd, vd, cfg)
    h = hashlib.sha256()
    for b in st.k_blocks:
        h.update(b.pattern_indices.astype(np.int32).tobytes())
        for g in b.channel_groups:
            h.update(g.codes)
    for t in st.v_tokens:
        h.update(np.int32(t.pattern_index).tobytes())
        h.update(t.group.codes)
    doc = {
        "raw_mse": raw.mse, "mse": pkv.mse, "k_mse": pkv.k_mse, "v_mse": pkv.v_mse,
        "raw_k_mse": raw.k_mse, "raw_v_mse": raw.v_mse,
        "gate_acceptance": pkv.v_gate_acceptance_rate, "committed": pkv.committed_tokens,
        "bits_per_token": pkv.bits_per_token, "raw_bits_per_token": raw.bits_per_token,
        "k_patterns": len(st.k_patterns), "v_patterns": len(st.v_patterns),
        "sha256": h.hexdigest(),
        "k_seed_first": int(np.random.default_rng(11).integers(2048)),
        "v_seed_first": int(np.random.default_rng(12).integers(2048)),
    }
    # the generator output is pinned separately; keep the first rows as a spot check
    doc["kp_head"] = kp[:2, :4].tolist()
    doc["vd_tail"] = vd[-2:, -4:].tolist()
    with open(os.path.join(HERE, "acceptance.json"), "w") as f:
        json.dump(doc, f, indent=1)


SNAPSHOT_CASES = {
    # name: (EngineConfig kwargs, head_dim, prefill, decode, [(layer, head, seed), ...])
    "k_gate": (dict(bits=2, pattern_count=8, use_k_gate=True), 64, 400, 140, [(0, 0, 21), (0, 1, 22), (1, 0, 23)]),
    "no_vgate4": (dict(bits=4, pattern_count=8, use_v_gate=False), 32, 300, 150, [(0, 0, 31), (2, 3, 32)]),
    "short": (dict(bits=2, pattern_count=4), 16, 100, 60, [(0, 0, 41), (0, 1, 42), (0, 2, 43), (5, 7, 44)]),
    "raw8": (dict(bits=8, pattern_count=4, group_size=32, residual_window=32, use_k_patterns=False,
                  use_v_patterns=False, generate_new_patterns=False), 32, 100, 40, [(0, 0, 51), (0, 1, 52)]),
}


def gen_snapshot():
    """Reference PKVS images (snapshot.py:57-99) of multi-head replays; the inputs are the
    synthetic generator's, cast to fp16 (so the GPU replays exactly the same values)."""
    import tempfile
    from patternkv import snapshot

    out = {}
    for name, (kw, d, tp, td, heads) in SNAPSHOT_CASES.items():
        cfg = engine.EngineConfig(**kw)
        states = {}
        for layer, head, seed in heads:
            s = analysis.generate_synthetic_stream(synth_spec(seed, tp + td, d))
            k = s.prefill_k[0, 0].astype(np.float16).astype(np.float64)
            v = s.prefill_v[0, 0].astype(np.float16).astype(np.float64)
            states[(layer, head)] = engine.replay_head(k[:tp], v[:tp], k[tp:], v[tp:], cfg)
        with tempfile.NamedTemporaryFile(suffix=".pkvs") as f:
            snapshot.save_snapshot(f.name, states)
            blob = open(f.name, "rb").read()
        p = name + "__"
        out[p + "config"] = np.array(json.dumps(kw))
        out[p + "dims"] = np.array([d, tp, td], np.int64)
        out[p + "heads"] = np.array(heads, np.int64)
        out[p + "blob"] = np.frombuffer(blob, np.uint8)
    save("snapshot.npz", **out)


def gen_trace():
    """KVTR images written by the reference (stream.py:126-150) for a small generated stream,
    fp16 and fp32, and the reference reader's fp64 arrays."""
    import tempfile
    from patternkv import stream as rstream

    spec = analysis.SyntheticStreamSpec(
        layers=2, heads=3, head_dim=16, prefill_len=40, decode_len=12,
        k_model=analysis.KeyModel(outlier_channels=(3,), outlier_multipliers=(32.0,), drift_rate=1.0 / 52,
                                  noise_std=0.05),
        v_model=analysis.ValueModel(cluster_count=8, center_spread=5.0, within_std=0.2, consistency=0.9,
                                    vocab_size=64),
        seed=77,
    )
    st = analysis.generate_synthetic_stream(spec)
    out = {"prefill_k": st.prefill_k, "prefill_v": st.prefill_v, "decode_k": st.decode_k, "decode_v": st.decode_v}
    for code, name in ((1, "f16"), (2, "f32")):
        with tempfile.NamedTemporaryFile(suffix=".kvtr") as f:
            rstream.write_trace(f.name, st, dtype_code=code)
            blob = open(f.name, "rb").read()
            back = rstream.read_trace(f.name)
        out[name + "_blob"] = np.frombuffer(blob, np.uint8)
        out[name + "_read_prefill_k"] = back.prefill_k
        out[name + "_read_decode_v"] = back.decode_v
    save("trace.npz", **out)


def gen_analysis():
    """variance_decomposition / covering_bound_check instances (the verify suites' host checks)."""
    import dataclasses

    rng = np.random.default_rng(2024)
    out = {}
    n = 40
    for i in range(n):
        t = int(rng.integers(2, 120))
        d = int(rng.integers(1, 6))
        k = int(rng.integers(1, 8))
        pts = rng.normal(0.0, 10.0 ** rng.uniform(-2, 2), size=(t, d)) + rng.uniform(-50, 50)
        if i == n - 1:  # the diagonal set: zero width radius
            pts = np.outer(np.linspace(-3, 3, 17), np.ones(3)) + 0.5
        lab = rng.integers(0, k, size=pts.shape[0])
        rho = float(rng.uniform(0.2, 0.9))
        rep = analysis.variance_decomposition(pts, lab, group_count=k)
        cov = analysis.covering_bound_check(pts, rho, bits=2)
        out.update({f"pts{i}": pts, f"lab{i}": lab, f"k{i}": k, f"rho{i}": rho, f"total{i}": rep.total,
                    f"intra{i}": rep.intra, f"inter{i}": rep.inter,
                    f"cov{i}": np.array(dataclasses.astuple(cov), dtype=np.float64)})
    save("analysis.npz", n=n, **out)


if __name__ == "__main__":
    gen_quant()
    gen_match()
    gen_kmeans()
    gen_gate()
    gen_synth()
    gen_engine()
    gen_acceptance()
    gen_snapshot()
    gen_trace()
    gen_analysis()
    print("golden fixtures written to", HERE)
