"""PatternKV B200 benchmark (driver contract: one JSON line on rank 0).

Headline (`value`): 2-bit PatternKV ENCODE throughput in GB/s (algorithmic
bytes of this build's HBM layout) on the
Llama-3.1-8B-shaped KV of BASELINE.json configs[1]: batch 8 x 32 layers x 8
KV heads = 2048 units per GPU, 32K-token prefill, head_dim 128, |M| = 32.
A step = one re-prefill of every unit (K1 encode over all 255 spans + the
exact window), inputs already resident in HBM (34 GB fp16, >> L2).
Mining runs once before the timed region (reported under `mining`).

Further legs (each its own JSON object, device-timed with CUDA events, max over ranks):
  decode_attn   one decode-attention step over the cfg2 cache (GQA 4)
  decode_loop   cfg2: 256 decode steps of append-and-refresh + attention (2 flushes)
  refgen        the headline encode on units from the reference generator (numpy, restated),
                with the K1-TC rare-path counters next to the torch-family pool's
  cfg3          Qwen2.5-7B: 28 layers x 4 KV heads, 126,976-token prefill + decode steps,
                2-bit, GQA 7, P 32 -> 64 over 4096 steps; KV heads shard over <= 4 ranks,
                a sequence split (pkv_decode_attn_partial + one (o, m, l) exchange) beyond
  cfg4          64 parallel samples x 32 layers x 8 KV heads forked from one prompt,
                decode steps from 512 tokens, and a 16K-token state with 156 patterns
  cfg5_head     Llama-3.1-70B: batch 32 x 8 KV heads, 64K context, 4-bit, GQA 8, KV heads
                sharded over the ranks, outputs all-gathered over NCCL inside the step
Multi-GPU: the headline is weak scaling (every rank owns its own batch of 8; units are
independent, SPEC.md:314 -- no data-path collective); `python bench.py --gpus N`
re-launches itself under torch.distributed.run when WORLD_SIZE is unset.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--legs ...]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
import subprocess
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0  # B200_PROFILING.md fallback, GB/s
ALL_LEGS = ("decode_loop", "mining_full", "refgen", "cfg3", "cfg4", "cfg5_head")


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def _traffic_doc():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic(kernel: str, token_units: int):
    """DRAM bytes (read + write) per launch of `kernel` at this run's size: the per-token-unit
    traffic of the committed ncu --set full capture (profiles/traffic.json, written by
    tools/make_profiles.py) times the launch's token-units; None without a capture."""
    try:
        return float(_traffic_doc()["bytes_per_token_unit"][kernel]) * token_units
    except Exception:
        return None


def issue_ceiling(kernel: str, bytes_per_token_unit: float, sm_mhz):
    """Instruction-issue ceiling of `kernel` (report encode against min(HBM, ALU)):
    warp-instructions per token-unit from the committed ncu capture (profiles/traffic.json),
    4 issues/clock on each SM at the clock measured during the timed region."""
    import torch

    try:
        ipt = float(_traffic_doc()["warp_instr_per_token_unit"][kernel])
        nsm = torch.cuda.get_device_properties(0).multi_processor_count
        hz = float(sm_mhz) * 1e6
    except Exception:
        return None
    return {"warp_instr_per_token_unit": ipt, "sm_mhz": sm_mhz,
            "ceiling_GBps": nsm * 4 * hz / ipt * bytes_per_token_unit / 1e9}


def enc_bytes_per_token(bits: int, d: int = 128, g: int = 128) -> int:
    """Algorithmic HBM bytes per encoded token-unit (this build's layout):
    read fp16 K+V (4d) ; write K codes + V codes (2*b*d/8), K params f32+f64
    (2*d*(4+8)/g), V params f32+f64 (2*(4+8)), int16 K/V indices (4)."""
    return 4 * d + 2 * bits * d // 8 + (2 * d * 12) // g + 24 + 4


def attn_bytes_per_step(units: int, committed: int, window: int, bits: int, patterns: int, gqa: int,
                        d: int = 128, g: int = 128) -> int:
    """Algorithmic bytes read by one decode-attention step over every unit:
    codes (2*b*d/8), int16 K/V idx (4), V params f32 (8), K params f32
    (2*d*4/g) per committed token; fp16 window rows (4d); fp32 pattern tables
    and q/out."""
    per_tok = 2 * bits * d // 8 + 4 + 8 + (2 * d * 4) // g
    per_unit = committed * per_tok + window * 4 * d + 2 * patterns * d * 4 + 2 * gqa * d * 4
    return units * per_unit


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during a timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" in r[2 + i]
                          and "Not" not in r[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def reference_arm(args):
    """--impl reference: the reference's CPU path (oracle port of engine.py's
    commit loop; /root/reference does not exist on the GPU box) on all host
    cores, same metric/unit/config.  Each step = a bounded sample of the
    workload (one 4K-token unit per core)."""
    from oracle import cpu_bench

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    bits = args.bits
    T = 4096
    per_tok = enc_bytes_per_token(bits)
    cpu_bench.encode_throughput(1, 512, bits=bits, workers=1)  # warm imports
    vals, step_s = [], []
    for s in range(args.warmup + args.steps):
        toks, secs, used = cpu_bench.encode_throughput(workers, T, bits=bits, workers=workers, seed0=1000 + s)
        if s >= args.warmup:
            vals.append(toks * per_tok / secs / 1e9)
            step_s.append(secs)
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": "patternkv_encode_GBps", "value": v, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(step_s)) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference generator model, oracle restatement)",
        "config": {"workload": "cfg2 llama3.1-8b KV encode, 2-bit, |M|=32, d=128 (bounded CPU sample: "
                               f"{workers} units x {T} tokens per step)", "bits": bits},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": workers, "kind": "port", "cpu": cpu_model(),
                         "sample": f"{workers} units x {T - 128} committed tokens per step, mining excluded"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args) -> int:
    """`python bench.py --gpus N` without torchrun: re-run under torch.distributed.run (one
    process per GPU, rendezvous on 127.0.0.1, NCCL's init log on for the rank count)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# --------------------------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------------------------
class Ctx:
    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.args = torch, dist, args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        # PKV_BENCH_BACKEND=gloo lets N ranks share fewer GPUs (a one-GPU rehearsal of the
        # multi-rank path: collectives staged through host memory); the driver's runs use NCCL
        self.backend = os.environ.get("PKV_BENCH_BACKEND", "nccl")
        self.local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(self.local)
        if self.world > 1:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
        self.peak, self.peak_kind = hbm_peak()

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], device="cuda" if self.backend == "nccl" else "cpu", dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def time_steps(self, fn, steps: int, warmup: int, clocks: bool = True):
        """W untimed steps, then K steps bracketed by barrier + synchronize; device time per step
        (CUDA events on the current stream), max over ranks; returns (ms, clock summary)."""
        torch = self.torch
        for _ in range(warmup):
            fn()
        self.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = ClockSampler(self.local) if clocks else None
        if clk:
            clk.__enter__()
        self.barrier()
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        self.barrier()
        if clk:
            clk.__exit__()
        return self.max_over_ranks(e0.elapsed_time(e1) / max(steps, 1)), (clk.summary() if clk else None)


def leg_encode(ctx, bits: int, k, v, pool_patterns, results, want_e2e: bool):
    """Headline encode (re-prefill of every unit with installed tables) + one decode-attention step."""
    torch, args = ctx.torch, ctx.args
    from paper_2510_05176_b200 import PatternKVCache
    from paper_2510_05176_b200.config import EngineConfig

    U, T, D, W, G = k.shape[0], k.shape[1], 128, 128, 128
    committed = T - W
    cfgE = EngineConfig(bits=bits, pattern_count=args.patterns)
    pool = args.pool
    reps = (U + pool - 1) // pool
    # ---- mining on the pool (timed once, outside the step) ------------------------------
    if pool_patterns is None:
        wcache = PatternKVCache(cfgE, 1, D, dtype=torch.float16, max_tokens=T + 2 * G)
        wcache.prefill(k[:1], v[:1])  # loads the mining/encode kernels (lazy module loading) untimed
        del wcache
    mcache = PatternKVCache(cfgE, pool, D, dtype=torch.float16, max_tokens=T + 2 * G)
    mcache.reserve_mining(T)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    mcache.prefill(k[:pool], v[:pool])
    e1.record()
    torch.cuda.synchronize()
    mine_ms = e0.elapsed_time(e1)
    pk = mcache.patterns(0)[:, : args.patterns]
    pv = mcache.patterns(1)[:, : args.patterns]
    del mcache
    cache = PatternKVCache(cfgE, U, D, dtype=torch.float16, max_tokens=T + 2 * G)
    cache.set_patterns(0, pk.repeat(reps, 1, 1)[:U])
    cache.set_patterns(1, pv.repeat(reps, 1, 1)[:U])

    def enc_step():
        cache.reset(keep_patterns=True)
        cache.commit_prefill(k, v)

    ev = []

    def enc_step_timed():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        enc_step()
        b.record()
        ev.append((a, b))

    enc_ms, clk = ctx.time_steps(enc_step_timed, args.steps, args.warmup)
    ev = ev[args.warmup:]
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    bpt = enc_bytes_per_token(bits)
    enc_bytes = U * committed * bpt
    r = dict(enc_ms=enc_ms, kern_ms=kern_ms, enc_gbps=ctx.world * enc_bytes / (enc_ms * 1e-3) / 1e9, bpt=bpt,
             enc_bytes=enc_bytes, mine_ms=mine_ms, clk=clk, launches=3 * args.steps, info=cache.info())

    # ---- decode attention over the encoded cache -----------------------------------------
    q = torch.randn((U, args.gqa, D), device="cuda", dtype=torch.float32)
    out = torch.empty_like(q)
    att_ms, clk_a = ctx.time_steps(lambda: cache.decode_attention(q, out=out), args.steps, args.warmup)
    att_bytes = attn_bytes_per_step(U, committed, W, bits, args.patterns, args.gqa)
    r.update(att_ms=att_ms, att_gbps=att_bytes / (att_ms * 1e-3) / 1e9, att_bytes=att_bytes,
             tok_s=ctx.world * args.batch / (att_ms * 1e-3), clk_a=clk_a)

    # ---- decode loop: append-and-refresh + attention per step (cfg2, 256 steps) ----------
    if "decode_loop" in args.legs:
        r["decode_loop"] = leg_decode_loop(ctx, cache, k, v, q, out, bits)

    # ---- end-to-end through the public API with host buffers -----------------------------
    if want_e2e:
        r["e2e"] = leg_e2e(ctx, cfgE, k, v, pk, pv, q, out, cache)

    # ---- full prefill of every unit: mining (both sides, one launch) + encode -------------
    # the `mining` key times the distinct pool only (256 units: 512 CTAs on 148 SMs, whose
    # wave quantisation dominates); this is the per-GPU cfg2 prefill as a deployment runs it
    if "mining_full" in args.legs and want_e2e:
        cache.reset(keep_patterns=False)
        cache.reserve_mining(T)
        pre_ms, _ = ctx.time_steps(lambda: (cache.reset(keep_patterns=False), cache.prefill(k, v)), 1, 0,
                                   clocks=False)
        r["mining_full"] = {"units": U, "sides": 2, "prefill_ms": pre_ms, "encode_ms": kern_ms,
                            "mining_ms": pre_ms - kern_ms,
                            "note": "one timed prefill of all units from HBM (K2 mining of both sides in one "
                                    "launch + K1-TC encode + window copy); mining_ms = prefill_ms - the encode "
                                    "step's device time"}
    del cache
    torch.cuda.empty_cache()
    results[bits] = r
    return pk, pv


def k1tc_counters(ctx, k, v, bits):
    """K1-TC rare-path counters of one encode pass over (k, v) [n, T, 128] with tables mined on
    the same units: fp64 re-matches, exact-division code fix-ups, pruning survivors, slow
    exact-extrema groups (per committed token-unit / group)."""
    torch, args = ctx.torch, ctx.args
    from paper_2510_05176_b200 import PatternKVCache, _lib
    from paper_2510_05176_b200.cache import _ptr, _stream
    from paper_2510_05176_b200.config import EngineConfig
    n, T = k.shape[0], k.shape[1]
    cfg = EngineConfig(bits=bits, pattern_count=args.patterns)
    m = PatternKVCache(cfg, n, 128, dtype=torch.float16, max_tokens=T + 256)
    m.reserve_mining(T)
    m.prefill(k, v)
    c2 = PatternKVCache(cfg, n, 128, dtype=torch.float16, max_tokens=T + 256, stats=True)
    c2.set_patterns(0, m.patterns(0)[:, : args.patterns])
    c2.set_patterns(1, m.patterns(1)[:, : args.patterns])
    del m
    c2.commit_prefill(k, v)
    buf = torch.zeros(4, dtype=torch.int32, device="cuda")
    _lib.call("pkv_cache_read", c2._h, b"stats", 0, 16, _ptr(buf), _stream())
    s = buf.cpu().tolist()
    tu = n * (T - 128)
    return {"refines_per_token_unit": s[0] / tu, "code_fixups_per_element": s[1] / (tu * 256),
            "survivors_per_token_side": s[2] / (2 * tu), "slow_groups_per_group": s[3] / (2 * tu)}


def leg_refgen(ctx, k, v):
    """Headline encode on units from the reference generator itself (analysis.py:321-370, restated
    in paper_2510_05176_b200.synthetic; SURVEY 8(d) models: K outlier channel 3 x 32, drift 1/T,
    noise 0.05; V 32 clusters, spread 5, within 0.2, consistency 0.9, vocab 1024; per-unit seed
    1_000_003 b + 1_009 l + h), a pool tiled over the cfg2 batch as in `value`, plus the K1-TC
    rare-path counters of that pool next to those of the torch-family pool (the pruning rate
    decides encode speed).  Overwrites k, v (the headline legs are done)."""
    torch, args = ctx.torch, ctx.args
    from paper_2510_05176_b200 import PatternKVCache
    from paper_2510_05176_b200 import synthetic as S
    from paper_2510_05176_b200.config import EngineConfig
    U, T, D, G = k.shape[0], k.shape[1], 128, 128
    pool = min(args.refgen_pool, U)
    km = S.KeyModel(outlier_channels=(3,), outlier_multipliers=(32.0,), drift_rate=1.0 / T, noise_std=0.05)
    vm = S.ValueModel(cluster_count=32, center_spread=5.0, within_std=0.2, consistency=0.9, vocab_size=1024)
    kp = torch.empty((pool, T, D), dtype=torch.float16)
    vp = torch.empty((pool, T, D), dtype=torch.float16)
    for u in range(pool):
        b, l, h = u // (args.layers * args.kv_heads), (u // args.kv_heads) % args.layers, u % args.kv_heads
        st = S.generate_synthetic_stream(S.SyntheticStreamSpec(
            layers=1, heads=1, head_dim=D, prefill_len=T, decode_len=0, k_model=km, v_model=vm,
            seed=1_000_003 * b + 1_009 * l + h))
        kp[u] = torch.from_numpy(st.prefill_k[0, 0]).to(torch.float16)
        vp[u] = torch.from_numpy(st.prefill_v[0, 0]).to(torch.float16)
    kd, vd = kp.cuda(), vp.cuda()
    del kp, vp
    bits = args.bits
    stats_synth = k1tc_counters(ctx, k[:pool], v[:pool], bits)
    stats_ref = k1tc_counters(ctx, kd, vd, bits)
    for u0 in range(0, U, pool):
        n = min(pool, U - u0)
        k[u0:u0 + n].copy_(kd[:n])
        v[u0:u0 + n].copy_(vd[:n])
    del kd, vd
    cfgE = EngineConfig(bits=bits, pattern_count=args.patterns)
    mcache = PatternKVCache(cfgE, pool, D, dtype=torch.float16, max_tokens=T + 2 * G)
    mcache.reserve_mining(T)
    mcache.prefill(k[:pool], v[:pool])  # warm
    mcache.reset(keep_patterns=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    mcache.prefill(k[:pool], v[:pool])
    e1.record()
    torch.cuda.synchronize()
    mine_ms = e0.elapsed_time(e1)
    reps = (U + pool - 1) // pool
    cache = PatternKVCache(cfgE, U, D, dtype=torch.float16, max_tokens=T + 2 * G)
    cache.set_patterns(0, mcache.patterns(0)[:, : args.patterns].repeat(reps, 1, 1)[:U])
    cache.set_patterns(1, mcache.patterns(1)[:, : args.patterns].repeat(reps, 1, 1)[:U])
    del mcache

    def step():
        cache.reset(keep_patterns=True)
        cache.commit_prefill(k, v)

    ms, clk = ctx.time_steps(step, args.steps, args.warmup)
    enc_bytes = U * (T - 128) * enc_bytes_per_token(bits)
    gbps = enc_bytes / (ms * 1e-3) / 1e9
    del cache
    return {"encode_GBps": ctx.world * gbps, "frac": gbps / ctx.peak, "ms_per_step": ms, "bits": bits, "units": U,
            "pool": pool, "mining_ms_pool": mine_ms, "clocks": clk,
            "generator": "paper_2510_05176_b200.synthetic.generate_synthetic_stream (reference analysis.py:321-370)",
            "k1tc_counters_refgen": stats_ref, "k1tc_counters_torch_family": stats_synth}


def leg_decode_loop(ctx, cache, k, v, q, out, bits):
    """cfg2 decode: `--decode-steps` steps of (append one token per unit + decode attention)
    right after a prefill; flushes (midrange refresh + K1 on the span) land every 128 steps."""
    torch, args = ctx.torch, ctx.args
    U, T, D = k.shape[0], k.shape[1], 128
    n = args.decode_steps
    # new tokens: the next rows of the synthetic stream are not materialised; reuse rows of the
    # resident K/V (the refresh/encode cost does not depend on the values' provenance)
    kn = k[:, T - n - 1:T - 1].contiguous() if T > n + 1 else k[:, :n].contiguous()
    vn = v[:, T - n - 1:T - 1].contiguous() if T > n + 1 else v[:, :n].contiguous()
    cache.reset(keep_patterns=True)
    cache.commit_prefill(k, v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    e0.record()
    for t in range(n):
        cache.append(kn[:, t], vn[:, t])
        cache.decode_attention(q, out=out)
    e1.record()
    ctx.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1))
    inf = cache.info()
    return {"steps": n, "ms_total": ms, "ms_per_step": ms / n, "tokens_per_s": ctx.world * args.batch * n / (ms * 1e-3),
            "flushes": n // 128, "patterns_per_side_end": args.patterns + n // 128, "units": U,
            "committed_end": inf.committed_count, "gqa": args.gqa,
            "note": "per step: pkv_append for every unit (window ring; a flush = midrange refresh + K1 span "
                    "encode every 128 steps) + pkv_decode_attn; tokens/s = sequences x steps / time"}


def leg_e2e(ctx, cfgE, k, v, pk, pv, q, out, cache):
    """Encode end to end from pinned host memory: every step copies ALL units' K/V host->device
    (a pinned pool of `--e2e-pool` units is cycled, so host RAM stays bounded) in unit slices
    whose H2D overlaps the previous slice's encode, and reads the encoded slice's codes of the
    step's last committed token back to the host."""
    torch, args = ctx.torch, ctx.args
    from paper_2510_05176_b200 import PatternKVCache

    U, T, D, G, W = k.shape[0], k.shape[1], 128, 128, 128
    committed = T - W
    ns = max(1, args.e2e_slices)
    bnd = [U * i // ns for i in range(ns + 1)]
    hp = min(args.e2e_pool, U)
    kh = k[:hp].cpu().pin_memory()
    vh = v[:hp].cpu().pin_memory()
    reps = (U + hp - 1) // hp
    pk_all, pv_all = pk.repeat(reps, 1, 1)[:U], pv.repeat((U + pv.shape[0] - 1) // pv.shape[0], 1, 1)[:U]
    ecaches = []
    for i in range(ns):
        ec = PatternKVCache(cfgE, bnd[i + 1] - bnd[i], D, dtype=torch.float16, max_tokens=T + 2 * G)
        ec.set_patterns(0, pk_all[bnd[i]:bnd[i + 1]])
        ec.set_patterns(1, pv_all[bnd[i]:bnd[i + 1]])
        ecaches.append(ec)
    smax = max(bnd[i + 1] - bnd[i] for i in range(ns))
    stage = [(torch.empty((smax, T, D), dtype=torch.float16, device="cuda"),
              torch.empty((smax, T, D), dtype=torch.float16, device="cuda")) for _ in range(2)]
    res_h = torch.empty((U, D), dtype=torch.uint8).pin_memory()
    copy_s = torch.cuda.Stream()
    comp = torch.cuda.current_stream()
    landed = [torch.cuda.Event() for _ in range(ns)]
    freed = [torch.cuda.Event() for _ in range(ns)]

    def h2d(dst, lo, hi):
        # host units lo..hi of the step map onto the pinned pool cyclically
        u = lo
        while u < hi:
            p = u % hp
            n = min(hi - u, hp - p)
            dst[0][u - lo:u - lo + n].copy_(kh[p:p + n], non_blocking=True)
            dst[1][u - lo:u - lo + n].copy_(vh[p:p + n], non_blocking=True)
            u += n

    def e2e_step():
        for i in range(ns):
            buf = stage[i % 2]
            with torch.cuda.stream(copy_s):
                if i >= 2:
                    copy_s.wait_event(freed[i - 2])  # slice i-2's encode is done with this buffer
                else:
                    copy_s.wait_stream(comp)
                h2d(buf, bnd[i], bnd[i + 1])
                landed[i].record(copy_s)
            comp.wait_event(landed[i])
            n = bnd[i + 1] - bnd[i]
            ecaches[i].reset(keep_patterns=True)
            ecaches[i].commit_prefill(buf[0][:n], buf[1][:n])
            freed[i].record(comp)
            kc, _ = ecaches[i].codes(committed - 1, committed)
            res_h[bnd[i]:bnd[i + 1]].copy_(kc[:, 0, :], non_blocking=True)

    e2e_ms, _ = ctx.time_steps(e2e_step, args.steps, args.warmup, clocks=False)
    # decode e2e: q from pinned host, out back to host
    qh = q.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    qd = torch.empty_like(q)

    def attn_e2e():
        qd.copy_(qh, non_blocking=True)
        cache.decode_attention(qd, out=out)
        oh.copy_(out, non_blocking=True)

    attn_ms, _ = ctx.time_steps(attn_e2e, args.steps, args.warmup, clocks=False)
    del ecaches, stage
    return {"gbps": ctx.world * U * committed * enc_bytes_per_token(cfgE.bits) / (e2e_ms * 1e-3) / 1e9,
            "ms": e2e_ms, "h2d": 2 * U * T * D * 2, "d2h": U * D, "attn_ms": attn_ms,
            "attn_h2d": qh.numel() * 4, "attn_d2h": oh.numel() * 4}


def leg_cfg3(ctx):
    """Qwen2.5-7B long context: 28 layers x 4 KV heads (B = 1), 126,976-token prefill (GPU
    mining + K1-TC), then `--cfg3-steps` decode steps of append-and-refresh + attention at
    GQA 7 (P grows by one per side per 128 steps).  Up to 4 ranks shard the KV heads (no
    exchange but the output gather); beyond 4 the committed blocks of every unit split across
    rank pairs (pkv_decode_attn_partial + one (o, m, l) all-gather + LSE merge per step)."""
    torch, args = ctx.torch, ctx.args
    from paper_2510_05176_b200 import PatternKVCache, dist as Dd
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.synth import synth_kv

    L, H, gqa, T, D = 28, 4, 7, args.cfg3_prefill, 128
    n = args.cfg3_steps
    hshard = min(ctx.world, H)
    seq = ctx.world // hshard  # ranks per head group (sequence split)
    hr = (ctx.rank // seq) if ctx.world > 1 else 0
    h0, h1 = Dd.shard_range(H, hshard, hr)
    units = [l * H + h for l in range(L) for h in range(h0, h1)]
    U = len(units)
    k, v = synth_kv(U, T + n, D, seed=3000 + 17 * hr)
    cfgE = EngineConfig(bits=2, pattern_count=32)
    cache = PatternKVCache(cfgE, U, D, dtype=torch.float16, max_tokens=T + n + 256)
    cache.reserve_mining(T)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cache.prefill(k[:, :T].contiguous(), v[:, :T].contiguous())
    e1.record()
    torch.cuda.synchronize()
    prefill_ms = e0.elapsed_time(e1)
    kn = k[:, T:].contiguous()
    vn = v[:, T:].contiguous()
    del k, v
    q = torch.randn((U, gqa, D), device="cuda", dtype=torch.float32)
    out = torch.empty_like(q)
    group = None
    if seq > 1:
        # ranks holding the same heads form one sequence-split group
        groups = [ctx.dist.new_group(list(range(g * seq, (g + 1) * seq))) for g in range(hshard)]
        group = groups[hr]

    def attend():
        if seq > 1:
            return Dd.sequence_split_attention(cache, q, group=group)
        return cache.decode_attention(q, out=out)

    # one attention step alone (steady-state decode cost at 127K)
    att_ms, _ = ctx.time_steps(attend, args.steps, args.warmup, clocks=False)
    e0.record()
    ctx.barrier()
    e0.record()
    for t in range(n):
        cache.append(kn[:, t], vn[:, t])
        attend()
    e1.record()
    ctx.barrier()
    loop_ms = ctx.max_over_ranks(e0.elapsed_time(e1))
    inf = cache.info()
    nk, nv = cache.pattern_counts()
    committed = T - 128
    att_bytes = attn_bytes_per_step(U, committed // seq, 128, 2, 32, gqa)
    del cache, kn, vn
    torch.cuda.empty_cache()
    return {"units_total": L * H, "units_per_rank": U, "prefill_tokens": T, "prefill_ms": prefill_ms,
            "prefill_note": "GPU mining (K2, both sides) + K1-TC encode of every unit, from HBM",
            "attn_ms": att_ms, "attn_tokens_per_s": 1.0 / (att_ms * 1e-3), "attn_GBps_per_gpu": att_bytes / (att_ms * 1e-3) / 1e9,
            "attn_frac": att_bytes / (att_ms * 1e-3) / 1e9 / ctx.peak,
            "decode_steps": n, "decode_ms_total": loop_ms, "decode_tokens_per_s": n / (loop_ms * 1e-3),
            "patterns_end": [int(nk.max()), int(nv.max())], "committed_end": inf.committed_count,
            "sharding": f"{hshard} head group(s) x {seq} sequence split", "gqa": gqa}


def leg_cfg4(ctx):
    """Test-time scaling breadth: 64 samples x 32 layers x 8 KV heads (16,384 units on one GPU;
    samples shard over ranks) forked from one 512-token prompt (pkv_cache_fork_from), then
    decode steps of append-and-refresh + attention; and a 16K-token state whose tables hold
    |M| = 32 + 124 = 156 patterns per side (what a 512 + 15,872-token run ends with: the 124
    midranges of its decode spans) for the late-run step cost."""
    torch, args = ctx.torch, ctx.args
    from paper_2510_05176_b200 import PatternKVCache, dist as Dd
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.synth import synth_kv

    S_all, L, H, D, gqa = 64, 32, 8, 128, 4
    s0, s1 = Dd.shard_range(S_all, ctx.world, ctx.rank)
    S = s1 - s0
    PU = L * H  # units of one sample (the prompt)
    U = S * PU
    n = args.cfg4_steps
    cfgE = EngineConfig(bits=2, pattern_count=32)
    res = {"samples_total": S_all, "samples_per_rank": S, "units_per_rank": U, "gqa": gqa}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # ---- early run: 512-token prompt -> fork into S samples -> decode --------------------------
    kp, vp = synth_kv(PU, 512, D, seed=4000)
    prompt = PatternKVCache(cfgE, PU, D, dtype=torch.float16, max_tokens=1024)
    prompt.prefill(kp, vp)
    cache = PatternKVCache(cfgE, U, D, dtype=torch.float16, max_tokens=512 + n + 256)
    torch.cuda.synchronize()
    e0.record()
    cache.fork_from(prompt, [u % PU for u in range(U)])
    e1.record()
    torch.cuda.synchronize()
    res["fork_ms"] = e0.elapsed_time(e1)
    del prompt, kp, vp
    kn, vn = synth_kv(U, n, D, seed=4001 + ctx.rank)  # every sample's own new tokens
    q = torch.randn((U, gqa, D), device="cuda", dtype=torch.float32)
    out = torch.empty_like(q)
    ctx.barrier()
    e0.record()
    for t in range(n):
        cache.append(kn[:, t], vn[:, t])
        cache.decode_attention(q, out=out)
    e1.record()
    ctx.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1))
    nk, _ = cache.pattern_counts()
    res.update(early_context=[512, 512 + n], early_steps=n, early_ms_total=ms,
               early_tokens_per_s=ctx.world * S * n / (ms * 1e-3), early_patterns_end=int(nk.max()))
    del cache, kn, vn
    torch.cuda.empty_cache()
    # ---- late run: 16K context, 156 patterns per side -------------------------------------------
    T = args.cfg4_late
    kk, vv = synth_kv(PU, T + 256, D, seed=4100)
    pc = PatternKVCache(cfgE, PU, D, dtype=torch.float16, max_tokens=T + 512)
    pc.prefill(kk[:, :512].contiguous(), vv[:, :512].contiguous())
    base = [pc.patterns(s)[:, :32] for s in (0, 1)]
    del pc
    nsp = (T - 512) // 128
    tabs = []
    for s, x in ((0, kk), (1, vv)):
        sp = x[:, 512:512 + 128 * nsp].float().view(PU, nsp, 128, D)
        mid = 0.5 * (sp.amin(dim=2) + sp.amax(dim=2))
        tabs.append(torch.cat([base[s], mid.double()], dim=1))
    P = tabs[0].shape[1]
    prompt = PatternKVCache(cfgE, PU, D, dtype=torch.float16, max_tokens=T + 512, max_patterns=P + 64)
    prompt.set_patterns(0, tabs[0])
    prompt.set_patterns(1, tabs[1])
    prompt.commit_prefill(kk[:, :T].contiguous(), vv[:, :T].contiguous())
    big = PatternKVCache(cfgE, U, D, dtype=torch.float16, max_tokens=T + 512, max_patterns=P + 64)
    big.fork_from(prompt, [u % PU for u in range(U)])
    del prompt
    kn = kk[:, T:T + 256].repeat(S, 1, 1).contiguous()
    vn = vv[:, T:T + 256].repeat(S, 1, 1).contiguous()
    del kk, vv
    m = min(args.cfg4_late_steps, 256)
    att_ms, _ = ctx.time_steps(lambda: big.decode_attention(q, out=out), args.steps, args.warmup, clocks=False)
    ctx.barrier()
    e0.record()
    for t in range(m):
        big.append(kn[:, t], vn[:, t])
        big.decode_attention(q, out=out)
    e1.record()
    ctx.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1))
    # the flushing append alone (refresh to P + 1 patterns + K1 on the span of every unit), on a
    # fresh fork of the same state: the window holds 128 + 127 tokens, the next append flushes
    flush_ms = None
    try:
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for t in range(m, m + 127):
            big.append(kn[:, t % 256], vn[:, t % 256])
        torch.cuda.synchronize()
        f0.record()
        big.append(kn[:, 0], vn[:, 0])
        f1.record()
        torch.cuda.synchronize()
        flush_ms = ctx.max_over_ranks(f0.elapsed_time(f1))
    except Exception:  # capacity: the flush timing is optional
        flush_ms = None
    att_bytes = attn_bytes_per_step(U, T - 128, 128, 2, P, gqa)
    res.update(late_flush_ms=flush_ms, late_flush_patterns=P + 1)
    res.update(late_context=T, late_patterns=P, late_steps=m, late_ms_total=ms,
               late_tokens_per_s=ctx.world * S * m / (ms * 1e-3), late_attn_ms=att_ms,
               late_attn_GBps_per_gpu=att_bytes / (att_ms * 1e-3) / 1e9,
               late_attn_frac=att_bytes / (att_ms * 1e-3) / 1e9 / ctx.peak)
    del big, kn, vn
    torch.cuda.empty_cache()
    return res


def leg_cfg5_head(ctx):
    """Llama-3.1-70B-shaped decode, head-sharded: batch 32 x `--cfg5-layers` layers x 8 KV heads,
    64K context, 4-bit, GQA 8; rank r holds KV heads [8r/N, 8(r+1)/N) of every (batch, layer).
    A step = decode attention over the rank's units + NCCL all-gather of the outputs
    [B, L, 8, 8, 128] (strong scaling: total work fixed)."""
    torch, args = ctx.torch, ctx.args
    from paper_2510_05176_b200 import PatternKVCache, dist as Dd
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.synth import synth_kv

    B, L, H, gqa, T, D = 32, args.cfg5_layers, 8, 8, args.cfg5_tokens, 128
    if H % ctx.world:
        return {"skipped": f"{H} KV heads do not split over {ctx.world} ranks"}
    hl = H // ctx.world
    U = B * L * hl
    cfgE = EngineConfig(bits=4, pattern_count=32)
    pool = min(args.pool, U)
    kp, vp = synth_kv(pool, T, D, seed=5000 + ctx.rank)
    pc = PatternKVCache(cfgE, pool, D, dtype=torch.float16, max_tokens=T + 256)
    pc.reserve_mining(T)
    pc.prefill(kp, vp)  # mining + encode of the distinct units
    del kp, vp
    cache = PatternKVCache(cfgE, U, D, dtype=torch.float16, max_tokens=T + 256)
    cache.fork_from(pc, [u % pool for u in range(U)])  # the rest are copies (no 64K inputs for all)
    del pc
    torch.cuda.empty_cache()
    q = torch.randn((U, gqa, D), device="cuda", dtype=torch.float32)
    out = torch.empty_like(q)

    def step():
        cache.decode_attention(q, out=out)
        return Dd.gather_head_outputs(out.view(B, L, hl, gqa, D))

    ms, clk = ctx.time_steps(step, args.steps, args.warmup)
    att_ms, _ = ctx.time_steps(lambda: cache.decode_attention(q, out=out), args.steps, args.warmup, clocks=False)
    att_bytes = attn_bytes_per_step(U, T - 128, 128, 4, 32, gqa)
    del cache
    torch.cuda.empty_cache()
    return {"batch": B, "layers": L, "kv_heads": H, "kv_heads_per_rank": hl, "units_per_rank": U, "context": T,
            "bits": 4, "gqa": gqa, "step_ms": ms, "attn_ms": att_ms, "gather_ms": ms - att_ms,
            "tokens_per_s": B / (ms * 1e-3), "tokens_per_s_80_layers": B / (ms * 1e-3) * L / 80,
            "attn_GBps_per_gpu": att_bytes / (att_ms * 1e-3) / 1e9,
            "attn_frac": att_bytes / (att_ms * 1e-3) / 1e9 / ctx.peak, "scaling": "strong",
            "collective": f"{ctx.backend.upper()} all_gather_into_tensor of [B, L, 8/N, 8, 128] fp32 per step" if ctx.world > 1
            else "none at N=1", "clocks": clk}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pkv", choices=["pkv", "reference"])
    ap.add_argument("--bits", type=int, default=2)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--gqa", type=int, default=4)
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--patterns", type=int, default=32)
    ap.add_argument("--pool", type=int, default=256, help="distinct synthetic units tiled over the batch")
    ap.add_argument("--no-four-bit", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-pool", type=int, default=256, help="pinned host units cycled by the e2e leg")
    ap.add_argument("--e2e-slices", type=int, default=8, help="unit slices the e2e step streams (H2D || encode)")
    ap.add_argument("--legs", default=",".join(ALL_LEGS), help="extra legs: " + ",".join(ALL_LEGS) + " or none")
    ap.add_argument("--decode-steps", type=int, default=256)
    ap.add_argument("--refgen-pool", type=int, default=32, help="reference-generator units tiled by the refgen leg")
    ap.add_argument("--cfg3-prefill", type=int, default=126976)
    ap.add_argument("--cfg3-steps", type=int, default=4096)
    ap.add_argument("--cfg4-steps", type=int, default=512)
    ap.add_argument("--cfg4-late", type=int, default=16384)
    ap.add_argument("--cfg4-late-steps", type=int, default=128)
    ap.add_argument("--cfg5-layers", type=int, default=16)
    ap.add_argument("--cfg5-tokens", type=int, default=65536)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.legs = [] if args.legs in ("", "none") else args.legs.split(",")

    if args.impl == "reference":
        reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))

    ctx = Ctx(args)
    torch = ctx.torch
    from paper_2510_05176_b200.synth import synth_kv

    U = args.batch * args.layers * args.kv_heads
    T, D = args.tokens, 128
    committed = T - 128
    # ---- inputs: pool of distinct units, tiled over the batch -------------------------
    pool = min(args.pool, U)
    args.pool = pool
    kp, vp = synth_kv(pool, T, D, seed=1234 + 7919 * ctx.rank)
    reps = (U + pool - 1) // pool
    k = kp.repeat(reps, 1, 1)[:U].contiguous()
    v = vp.repeat(reps, 1, 1)[:U].contiguous()
    del kp, vp
    torch.cuda.synchronize()

    results = {}
    pats = None
    for bits in ([args.bits] + ([] if args.no_four_bit else [4 if args.bits != 4 else 2])):
        pats = leg_encode(ctx, bits, k, v, pats, results, want_e2e=(bits == args.bits))
    refgen = None
    if "refgen" in args.legs:
        try:
            refgen = leg_refgen(ctx, k, v)
        except Exception as ex:  # reported, not fatal
            refgen = {"failed": f"{type(ex).__name__}: {ex}"[:300]}
    del k, v
    torch.cuda.empty_cache()
    extra = {}
    for leg, fn in (("cfg3", leg_cfg3), ("cfg4", leg_cfg4), ("cfg5_head", leg_cfg5_head)):
        if leg in args.legs:
            try:
                extra[leg] = fn(ctx)
            except Exception as ex:  # a leg that cannot run at this N / memory is reported, not fatal
                extra[leg] = {"failed": f"{type(ex).__name__}: {ex}"[:300]}
            torch.cuda.empty_cache()

    if ctx.rank != 0:
        if ctx.world > 1:
            ctx.dist.barrier()
            ctx.dist.destroy_process_group()
        return

    r = results[args.bits]
    peak = ctx.peak
    enc_ceiling = issue_ceiling("encode", r["bpt"], (r["clk"] or {}).get("sm_mhz")) if args.bits == 2 else None
    if enc_ceiling:
        enc_ceiling["frac"] = (r["enc_bytes"] / (r["kern_ms"] * 1e-3) / 1e9) / enc_ceiling["ceiling_GBps"]
    # ---- CPU baseline: oracle port on this host's cores, bounded sample --------------
    cpu = None
    if ctx.world == 1 and not args.no_cpu:
        try:
            from oracle import cpu_bench
            workers = os.cpu_count() or 1
            toks, secs, used = cpu_bench.encode_throughput(workers, 4096, bits=args.bits, workers=workers)
            cpu = {"value": toks * enc_bytes_per_token(args.bits) / secs / 1e9, "unit": "GB/s", "cores": used,
                   "kind": "port", "cpu": cpu_model(),
                   "sample": f"{used} units x 3968 committed tokens (4K-token prefill, P=32, "
                             f"{args.bits}-bit), mining excluded, one unit per process"}
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "port", "sample": f"failed: {ex}"}

    kern_gbps = r["enc_bytes"] / (r["kern_ms"] * 1e-3) / 1e9
    e2e = r["e2e"]
    line = {
        "metric": "patternkv_encode_GBps",
        "value": r["enc_gbps"],
        "unit": "GB/s",
        "n_gpus": ctx.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["enc_ms"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16-in/f64-exact",
        "data": "synthetic (reference KeyModel/ValueModel family on device, pool of "
                f"{pool} distinct units tiled)",
        "config": {"workload": f"cfg2 Llama-3.1-8B KV: batch {args.batch} x {args.layers} layers x {args.kv_heads} "
                               f"KV heads per GPU, {T}-token prefill, d=128, {args.bits}-bit, |M|={args.patterns}, "
                               f"G=W=128", "units_per_gpu": U, "tokens": T, "bits": args.bits,
                   "l2": "inputs 34 GB/GPU >> 126 MB L2 (no flush needed)", "parallelism": f"units x{ctx.world}"},
        "roofline": {"bound": "hbm", "achieved": kern_gbps, "peak": peak, "unit": "GB/s",
                     "frac": kern_gbps / peak, "traffic": ncu_traffic("encode", U * committed),
                     "peak_kind": ctx.peak_kind, "algorithmic_bytes_per_launch": r["enc_bytes"],
                     "kernel": f"encode_tc_kernel<{args.bits}> (K1-TC)", "bytes_per_token_unit": r["bpt"],
                     "issue_ceiling": enc_ceiling},
        "decode_attn": {"tokens_per_s": r["tok_s"], "ms_per_step": r["att_ms"], "GBps": r["att_gbps"],
                        "frac": r["att_gbps"] / peak, "bytes_per_step": r["att_bytes"], "gqa": args.gqa,
                        "context": T, "e2e_ms_per_step": e2e["attn_ms"],
                        "e2e_h2d_bytes": e2e["attn_h2d"], "e2e_d2h_bytes": e2e["attn_d2h"],
                        "kernel": "attn_tc_kernel (K3-TC: tcgen05 kind::i8, integer code planes from TMEM) + attn_merge_kernel", "clocks": r["clk_a"],
                        "traffic": ncu_traffic("attn", U * committed)},
        "mining_full": r.get("mining_full"),
        "mining": {"ms": r["mine_ms"], "units": pool, "sides": 2, "tokens": T, "patterns": args.patterns,
                   "ncu": _traffic_doc().get("kmeans") if _traffic_doc() else None,
                   "scratch": "preallocated outside the timed region (PatternKVCache.reserve_mining)",
                   "kernel": "kmeans_stream_kernel: one TMA stream per pass, distance GEMM on tcgen05 (TMEM), exact fp64 "
                             "centroid sums, objective from the sums in double-double"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e["gbps"], "unit": "GB/s", "h2d_bytes_per_step": e2e["h2d"],
                "d2h_bytes_per_step": e2e["d2h"], "ms_per_step": e2e["ms"],
                "note": f"all {U} units per step from pinned host memory (a {min(args.e2e_pool, U)}-unit pinned pool "
                        f"cycled), {args.e2e_slices} slices with H2D of slice i+1 overlapping the encode of slice i, "
                        "installed pattern tables as in `value`; the encoded cache stays device-resident (its "
                        "consumer is decode attention), the step's result read back is each unit's codes of the "
                        "last committed token"},
        "gpu_launches": r["launches"],  # per step: encode_tc_kernel + kfix_kernel + window_put_kernel
        "clocks": r["clk"],
    }
    if "decode_loop" in r:
        line["decode_loop"] = r["decode_loop"]
    other = [b for b in results if b != args.bits]
    if other:
        o = results[other[0]]
        line[f"bits{other[0]}"] = {"encode_GBps": o["enc_gbps"], "encode_frac": o["enc_gbps"] / ctx.world / peak,
                                   "decode_tokens_per_s": o["tok_s"], "decode_frac": o["att_gbps"] / peak,
                                   "decode_ms": o["att_ms"], "mining_ms": o["mine_ms"]}
        if "decode_loop" in o:
            line[f"bits{other[0]}"]["decode_loop"] = o["decode_loop"]
    if refgen is not None:
        line["refgen"] = refgen
    line.update(extra)
    print(json.dumps(line), flush=True)
    if ctx.world > 1:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
