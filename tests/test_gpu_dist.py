"""Multi-rank execution of the codec on the GPU: two processes share one
B200 and exchange through gloo (device -> host staging), standing in for NCCL ranks.

* sequence split (cfg3 at 8 GPUs): every rank attends its committed-block range with
  pkv_decode_attn_partial (the last rank adds the exact window), the ranks exchange
  (o, m, l) and LSE-merge == the single-rank pkv_decode_attn over the whole cache;
* head sharding (cfg5): rank r holds KV heads [4r, 4r+4) of every (batch, layer), runs
  decode attention on its units and all-gathers the outputs == one cache with all heads;
* unit fork (parallel samples, cfg4): forked units equal their source and keep decoding
  bit-exactly like the oracle.
"""

import math
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pkv_oracle as O  # noqa: E402

B, L, H, G, D, T = 2, 2, 8, 4, 128, 1200


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    ks, vs = [], []
    for b in range(B):
        for l in range(L):
            for h in range(H):
                k, v = O.synth_unit(O.unit_seed(b, l, h), T + 40, D)
                ks.append(k)
                vs.append(v)
    q = np.random.default_rng(5).normal(size=(B * L * H, G, D)).astype(np.float32)
    return np.stack(ks).astype(np.float16), np.stack(vs).astype(np.float16), q


def _cache(P, k, v, steps=40):
    cache = P.PatternKVCache(P.EngineConfig(bits=2, pattern_count=16), k.shape[0], D, dtype=torch.float16,
                             max_tokens=T + 512)
    kt, vt = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    cache.prefill(kt[:, :T], vt[:, :T])
    for t in range(T, T + steps):
        cache.append(kt[:, t], vt[:, t])
    return cache


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2510_05176_b200 as P
    from paper_2510_05176_b200 import dist as Dd

    k, v, qq = _data()
    out = {}
    # sequence split over the committed blocks of every unit
    cache = _cache(P, k, v)
    qt = torch.from_numpy(qq).cuda()
    full = cache.decode_attention(qt).cpu().numpy()
    merged = Dd.sequence_split_attention(cache, qt).cpu().numpy()
    out["seq_err"] = float(np.abs(merged - full).max() / np.abs(full).max())
    b0, b1, win = Dd.sequence_block_range(cache.info().n_blocks, world, rank)
    out["range"] = (b0, b1, win)
    # head sharding: this rank's units are kv heads [4r, 4r+4) of every (batch, layer)
    mine = Dd.shard_units(B, L, H, world, rank, by="head")
    hc = _cache(P, k[mine], v[mine])
    local = hc.decode_attention(qt[mine]).view(B, L, H // world, G, D)
    gathered = Dd.gather_head_outputs(local).reshape(B * L * H, G, D).cpu().numpy()
    out["head_err"] = float(np.abs(gathered - full).max() / np.abs(full).max())
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_sequence_split_and_head_gather():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the two ranks' block ranges tile the committed blocks; only the last takes the window
    r0, r1 = res[0]["range"], res[1]["range"]
    assert r0[0] == 0 and r0[1] == r1[0] and not r0[2] and r1[2]
    for r in (0, 1):
        assert res[r]["seq_err"] <= 1e-5, res[r]
        assert res[r]["head_err"] <= 1e-5, res[r]


def test_partial_attention_matches_fp64_pieces():
    """pkv_decode_attn_partial over disjoint block ranges (+ window) LSE-merges to the fp64
    softmax over the oracle's reconstruction; an empty range gives (0, -inf, 0)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_05176_b200 as P
    from paper_2510_05176_b200 import dist as Dd

    k, v, qq = _data()
    k, v, qq = k[:3], v[:3], qq[:3]
    cache = _cache(P, k, v)
    nb = cache.info().n_blocks
    qt = torch.from_numpy(qq).cuda()
    parts = [cache.decode_attention_partial(qt, 0, 3, with_window=False),
             cache.decode_attention_partial(qt, 3, nb, with_window=False),
             cache.decode_attention_partial(qt, nb, nb, with_window=True)]
    o = torch.stack([p[0] for p in parts]).double()
    m = torch.stack([p[1] for p in parts]).double()
    l = torch.stack([p[2] for p in parts]).double()
    got = Dd.lse_merge(o, m, l).cpu().numpy()
    e = cache.decode_attention_partial(qt, 2, 2, with_window=False)
    assert float(e[0].abs().max()) == 0.0 and bool(torch.isinf(e[1]).all()) and float(e[2].abs().max()) == 0.0
    kk = k.astype(np.float64)
    vv = v.astype(np.float64)
    for u in range(3):
        h = O.replay(kk[u, :T], vv[u, :T], kk[u, T:T + 40], vv[u, T:T + 40], O.Knobs(bits=2, pattern_count=16))
        ref = O.head_attention(h, qq[u].astype(np.float64), 1.0 / math.sqrt(D))
        assert np.abs(got[u] - ref).max() / np.abs(ref).max() <= 1e-3


def test_fork_units_then_decode_matches_oracle():
    """Fork one prompt's unit into parallel samples (cfg4): every copy equals the source, then
    each sample decodes its own tokens bit-exactly like an oracle head with the same history."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_05176_b200 as P
    from paper_2510_05176_b200.export import export_unit

    tp, steps, S = 512, 300, 4
    k, v = O.synth_unit(O.unit_seed(9, 9, 9), tp, D)
    k = k.astype(np.float16).astype(np.float64)
    v = v.astype(np.float16).astype(np.float64)
    cfg = dict(bits=2, pattern_count=32)
    cache = P.PatternKVCache(P.EngineConfig(**cfg), S, D, dtype=torch.float16, max_tokens=tp + steps + 256,
                             record_decisions=True)
    kt = torch.from_numpy(np.repeat(k[None], S, 0)).half().cuda()
    vt = torch.from_numpy(np.repeat(v[None], S, 0)).half().cuda()
    kt[1:] = 0  # only unit 0 holds the prompt; the others are overwritten by the fork
    vt[1:] = 0
    cache.prefill(kt, vt)
    cache.fork([0] * (S - 1), list(range(1, S)))
    s0 = export_unit(cache, 0, with_bytes=False)
    for s in range(1, S):
        st = export_unit(cache, s, with_bytes=False)
        for f in ("kpat", "vpat", "k_codes", "v_codes", "k_idx", "v_idx", "k_scale", "v_scale", "window_k", "vdec"):
            np.testing.assert_array_equal(getattr(st, f), getattr(s0, f))
    dk, dv = [], []
    for s in range(S):
        a, b = O.synth_unit(O.unit_seed(10 + s, 0, 0), steps, D)
        dk.append(a.astype(np.float16).astype(np.float64))
        dv.append(b.astype(np.float16).astype(np.float64))
    dkt = torch.from_numpy(np.stack(dk)).half().cuda()
    dvt = torch.from_numpy(np.stack(dv)).half().cuda()
    for t in range(steps):
        cache.append(dkt[:, t], dvt[:, t])
    for s in range(S):
        h = O.replay(k, v, dk[s], dv[s], O.Knobs(**cfg))
        st = export_unit(cache, s, with_bytes=False)
        np.testing.assert_array_equal(st.kpat, h.kpat)
        np.testing.assert_array_equal(st.vpat, h.vpat)
        np.testing.assert_array_equal(st.k_codes, np.concatenate([b[4] for b in h.k_blocks]))
        np.testing.assert_array_equal(st.v_codes, np.stack([x[2] for x in h.v_tok]))
        np.testing.assert_array_equal(st.k_idx, np.concatenate([b[5] for b in h.k_blocks]))


def test_fork_from_prompt_cache_into_samples():
    """pkv_cache_fork_from: a 2-unit prompt cache (prefill + a few appends, so the window and a
    flush are part of the state) becomes 3 samples x 2 units in a second cache with larger
    capacities; each sample then decodes its own tokens == the oracle replay of its history."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_05176_b200 as P
    from paper_2510_05176_b200.export import export_unit

    tp, pre, steps, S = 600, 150, 200, 3
    cfg = dict(bits=4, pattern_count=16)
    ks, vs = [], []
    for u in range(2):
        a, b = O.synth_unit(O.unit_seed(2, u, 7), tp + pre, D)
        ks.append(a.astype(np.float16).astype(np.float64))
        vs.append(b.astype(np.float16).astype(np.float64))
    k, v = np.stack(ks), np.stack(vs)
    prompt = P.PatternKVCache(P.EngineConfig(**cfg), 2, D, dtype=torch.float16, max_tokens=1024)
    kt, vt = torch.from_numpy(k).half().cuda(), torch.from_numpy(v).half().cuda()
    prompt.prefill(kt[:, :tp], vt[:, :tp])
    for t in range(tp, tp + pre):
        prompt.append(kt[:, t], vt[:, t])
    big = P.PatternKVCache(P.EngineConfig(**cfg), 2 * S, D, dtype=torch.float16, max_tokens=4096, max_patterns=200)
    big.fork_from(prompt, [i % 2 for i in range(2 * S)])
    del prompt
    dk, dv = [], []
    for i in range(2 * S):
        a, b = O.synth_unit(O.unit_seed(20 + i, 1, 1), steps, D)
        dk.append(a.astype(np.float16).astype(np.float64))
        dv.append(b.astype(np.float16).astype(np.float64))
    dkt = torch.from_numpy(np.stack(dk)).half().cuda()
    dvt = torch.from_numpy(np.stack(dv)).half().cuda()
    for t in range(steps):
        big.append(dkt[:, t], dvt[:, t])
    q = np.random.default_rng(3).normal(size=(2 * S, 4, D)).astype(np.float32)
    out = big.decode_attention(torch.from_numpy(q).cuda()).cpu().numpy()
    for i in range(2 * S):
        u = i % 2
        h = O.replay(k[u, :tp], v[u, :tp], np.concatenate([k[u, tp:], dk[i]]), np.concatenate([v[u, tp:], dv[i]]),
                     O.Knobs(**cfg))
        st = export_unit(big, i, with_bytes=False)
        assert st.n_prefill_k == 16
        np.testing.assert_array_equal(st.kpat, h.kpat)
        np.testing.assert_array_equal(st.vpat, h.vpat)
        np.testing.assert_array_equal(st.k_codes, np.concatenate([b[4] for b in h.k_blocks]))
        np.testing.assert_array_equal(st.v_codes, np.stack([x[2] for x in h.v_tok]))
        np.testing.assert_array_equal(st.v_idx, np.array([x[3] for x in h.v_tok]))
        np.testing.assert_array_equal(st.window_k, np.stack(h.win_k))
        ref = O.head_attention(h, q[i].astype(np.float64), 1.0 / math.sqrt(D))
        assert np.abs(out[i] - ref).max() / np.abs(ref).max() <= 1e-3
