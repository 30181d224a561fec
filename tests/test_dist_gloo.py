"""Multi-process (gloo, world_size 2, CPU) tests of the unit sharding and the
only exchange steps (head-output all-gather, sequence-split LSE merge)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_05176_b200 import dist as D

    out = {}
    # unit sharding: batch split covers each unit exactly once
    out["batch_units"] = D.shard_units(3, 4, 8, world, rank, by="batch")
    out["head_units"] = D.shard_units(2, 3, 8, world, rank, by="head")
    # head-sharded outputs: rank r holds heads [4r, 4r+4) of a [B=2, L=3, H=8, G=4, d=16] tensor
    g = torch.Generator().manual_seed(0)
    full = torch.randn((2, 3, 8, 4, 16), generator=g)
    local = full[:, :, 4 * rank:4 * rank + 4].clone()
    out["gather_ok"] = bool(torch.equal(D.gather_head_outputs(local), full))
    # sequence split: each rank owns half the tokens of every head
    T, G, d = 50, 4, 16
    qv = torch.randn((G, d), generator=g, dtype=torch.float64)
    k = torch.randn((T, d), generator=g, dtype=torch.float64)
    v = torch.randn((T, d), generator=g, dtype=torch.float64)
    s0, s1 = D.shard_range(T, world, rank)
    sc = qv @ k[s0:s1].T
    m = sc.max(dim=1).values
    p = torch.exp(sc - m[:, None])
    o = p @ v[s0:s1]
    merged = D.gather_and_merge_partials(o, m, p.sum(dim=1))
    ref = torch.softmax(qv @ k.T, dim=1) @ v
    out["merge_err"] = float((merged - ref).abs().max())
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_and_exchanges_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_b = sorted(res[0]["batch_units"] + res[1]["batch_units"])
    assert all_b == list(range(3 * 4 * 8))
    all_h = sorted(res[0]["head_units"] + res[1]["head_units"])
    assert all_h == list(range(2 * 3 * 8))
    assert res[0]["gather_ok"] and res[1]["gather_ok"]
    assert res[0]["merge_err"] < 1e-12 and res[1]["merge_err"] < 1e-12


def test_shard_range_balanced():
    from paper_2510_05176_b200.dist import shard_range

    for n in (0, 1, 7, 2048, 2049):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
