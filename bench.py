"""PatternKV B200 benchmark (driver contract: one JSON line on rank 0).

Headline (`value`): 2-bit PatternKV ENCODE throughput in GB/s (algorithmic
bytes of this build's HBM layout) on the
Llama-3.1-8B-shaped KV of BASELINE.json configs[1]: batch 8 x 32 layers x 8
KV heads = 2048 units per GPU, 32K-token prefill, head_dim 128, |M| = 32.
A step = one re-prefill of every unit (K1 encode over all 255 spans + the
exact window), inputs already resident in HBM (34 GB fp16, >> L2).
Mining runs once before the timed region (reported under `mining`).
`decode_attn` reports the same cache's decode attention (GQA 4, one query
token per (batch, layer) head group) in tokens/s; `four_bit` repeats both at
4 bits.  Multi-GPU: weak scaling, every rank owns its own batch of 8 (units
are independent) -- no data-path collective.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0  # B200_PROFILING.md fallback, GB/s


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def ncu_traffic(kernel: str, token_units: int):
    """DRAM bytes (read + write) per launch of `kernel` at this run's size: the per-token-unit
    traffic of the committed ncu --set full capture (profiles/traffic.json, written by
    tools/make_profiles.py) times the launch's token-units; None without a capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return float(json.load(f)["bytes_per_token_unit"][kernel]) * token_units
    except Exception:
        return None


def issue_ceiling(kernel: str, bytes_per_token_unit: float, sm_mhz):
    """Instruction-issue ceiling of `kernel` (report encode against min(HBM, ALU)):
    warp-instructions per token-unit from the committed ncu capture (profiles/traffic.json),
    4 issues/clock on each SM at the clock measured during the timed region."""
    import torch

    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            ipt = float(json.load(f)["warp_instr_per_token_unit"][kernel])
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
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": workers, "kind": "port",
                         "sample": f"{workers} units x {T - 128} committed tokens per step, mining excluded"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    ap.add_argument("--e2e-units", type=int, default=256)
    ap.add_argument("--e2e-slices", type=int, default=8, help="unit slices the e2e step streams (H2D || encode)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2510_05176_b200 import PatternKVCache
    from paper_2510_05176_b200.config import EngineConfig
    from paper_2510_05176_b200.synth import synth_kv

    U = args.batch * args.layers * args.kv_heads
    T, D, W, G = args.tokens, 128, 128, 128
    committed = T - W
    peak, peak_kind = hbm_peak()
    launches = 0

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- inputs: pool of distinct units, tiled over the batch -------------------------
    pool = min(args.pool, U)
    kp, vp = synth_kv(pool, T, D, seed=1234 + 7919 * rank)
    reps = (U + pool - 1) // pool
    k = kp.repeat(reps, 1, 1)[:U].contiguous()
    v = vp.repeat(reps, 1, 1)[:U].contiguous()
    del kp, vp
    torch.cuda.synchronize()

    results = {}
    for bits in ([args.bits] + ([] if args.no_four_bit else [4 if args.bits != 4 else 2])):
        cfgE = EngineConfig(bits=bits, pattern_count=args.patterns)
        # ---- mining on the pool (timed once, outside the step) ---------------------------
        mcache = PatternKVCache(cfgE, pool, D, dtype=torch.float16, max_tokens=T + 2 * G)
        wcache = PatternKVCache(cfgE, 1, D, dtype=torch.float16, max_tokens=T + 2 * G)
        wcache.prefill(k[:1], v[:1])  # loads the mining/encode kernels (lazy module loading) untimed
        del wcache
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

        for _ in range(args.warmup):
            enc_step()
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        with ClockSampler(local) as clk:
            t_start = torch.cuda.Event(enable_timing=True)
            t_end = torch.cuda.Event(enable_timing=True)
            barrier()
            t_start.record()
            for i in range(args.steps):
                ev[i][0].record()
                enc_step()
                ev[i][1].record()
            t_end.record()
            barrier()
        enc_ms = max_over_ranks(t_start.elapsed_time(t_end) / args.steps)
        kern_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
        launches_enc = 2 * args.steps  # K1 encode + window copy per step
        bpt = enc_bytes_per_token(bits)
        enc_bytes = U * committed * bpt
        enc_gbps = world * enc_bytes / (enc_ms * 1e-3) / 1e9

        # ---- decode attention over the encoded cache ------------------------------------
        q = torch.randn((U, args.gqa, D), device="cuda", dtype=torch.float32)
        out = torch.empty_like(q)
        for _ in range(args.warmup):
            cache.decode_attention(q, out=out)
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk_a:
            barrier()
            a0.record()
            for _ in range(args.steps):
                cache.decode_attention(q, out=out)
            a1.record()
            barrier()
        att_ms = max_over_ranks(a0.elapsed_time(a1) / args.steps)
        att_bytes = attn_bytes_per_step(U, committed, W, bits, args.patterns, args.gqa)
        att_gbps = att_bytes / (att_ms * 1e-3) / 1e9
        tok_s = world * args.batch / (att_ms * 1e-3)  # one new token per sequence per step
        results[bits] = dict(enc_ms=enc_ms, kern_ms=kern_ms, enc_gbps=enc_gbps, bpt=bpt, enc_bytes=enc_bytes,
                             mine_ms=mine_ms, att_ms=att_ms, att_gbps=att_gbps, tok_s=tok_s, att_bytes=att_bytes,
                             clk=clk.summary(), clk_a=clk_a.summary(), launches=launches_enc + 2 * args.steps,
                             info=cache.info())

        # ---- end-to-end through the public API with host buffers (headline bits only) ----
        if bits == args.bits:
            ue = min(args.e2e_units, U)
            kh = k[:ue].cpu().pin_memory()
            vh = v[:ue].cpu().pin_memory()
            # the host K/V stream in unit slices (one cache per slice, as a streaming caller would
            # hold them): slice i's H2D on a copy stream overlaps slice i-1's encode
            ns = max(1, min(args.e2e_slices, ue))
            bnd = [ue * i // ns for i in range(ns + 1)]
            ecaches, kds, vds = [], [], []
            for i in range(ns):
                sl = slice(bnd[i], bnd[i + 1])
                ec = PatternKVCache(cfgE, bnd[i + 1] - bnd[i], D, dtype=torch.float16, max_tokens=T + 2 * G)
                ec.set_patterns(0, pk.repeat(reps, 1, 1)[:ue][sl])
                ec.set_patterns(1, pv.repeat(reps, 1, 1)[:ue][sl])
                ecaches.append(ec)
                kds.append(torch.empty_like(k[sl]))
                vds.append(torch.empty_like(v[sl]))
            res_h = torch.empty((ue, 128), dtype=torch.uint8).pin_memory()
            copy_s = torch.cuda.Stream()
            comp = torch.cuda.current_stream()
            landed = [torch.cuda.Event() for _ in range(ns)]

            def e2e_step():
                copy_s.wait_stream(comp)  # the previous step is done with the device buffers
                with torch.cuda.stream(copy_s):
                    for i in range(ns):
                        kds[i].copy_(kh[bnd[i]:bnd[i + 1]], non_blocking=True)
                        vds[i].copy_(vh[bnd[i]:bnd[i + 1]], non_blocking=True)
                        landed[i].record(copy_s)
                for i in range(ns):
                    comp.wait_event(landed[i])
                    ecaches[i].reset(keep_patterns=True)
                    ecaches[i].commit_prefill(kds[i], vds[i])
                    kc, _ = ecaches[i].codes(0, 1)  # the step's result: first token's codes per unit
                    res_h[bnd[i]:bnd[i + 1]].copy_(kc[:, 0, :], non_blocking=True)

            for _ in range(args.warmup):
                e2e_step()
            barrier()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record()
            for _ in range(args.steps):
                e2e_step()
            b1.record()
            barrier()
            e2e_ms = max_over_ranks(b0.elapsed_time(b1) / args.steps)
            results["e2e"] = dict(gbps=world * ue * committed * enc_bytes_per_token(bits) / (e2e_ms * 1e-3) / 1e9,
                                  h2d=2 * kh.numel() * 2, d2h=res_h.numel())
            # decode e2e: q from pinned host, out back to host
            qh = q.cpu().pin_memory()
            oh = torch.empty_like(qh).pin_memory()
            qd = torch.empty_like(q)
            b0.record()
            for _ in range(args.steps):
                qd.copy_(qh, non_blocking=True)
                cache.decode_attention(qd, out=out)
                oh.copy_(out, non_blocking=True)
            b1.record()
            barrier()
            results["e2e_attn_ms"] = max_over_ranks(b0.elapsed_time(b1) / args.steps)
            del ecaches, kds, vds
        del cache
        torch.cuda.empty_cache()

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    r = results[args.bits]
    # instruction-issue ceiling of the encode kernel (the committed capture is the 2-bit kernel)
    enc_ceiling = issue_ceiling("encode", r["bpt"], (r["clk"] or {}).get("sm_mhz")) if args.bits == 2 else None
    if enc_ceiling:
        enc_ceiling["frac"] = (r["enc_bytes"] / (r["kern_ms"] * 1e-3) / 1e9) / enc_ceiling["ceiling_GBps"]
    # ---- CPU baseline: oracle port on this host's cores, bounded sample --------------
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            from oracle import cpu_bench
            workers = os.cpu_count() or 1
            toks, secs, used = cpu_bench.encode_throughput(workers, 4096, bits=args.bits, workers=workers)
            cpu = {"value": toks * enc_bytes_per_token(args.bits) / secs / 1e9, "unit": "GB/s", "cores": used,
                   "kind": "port", "sample": f"{used} units x 3968 committed tokens (4K-token prefill, P=32, "
                                             f"{args.bits}-bit), mining excluded, one unit per process"}
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "port", "sample": f"failed: {ex}"}

    kern_gbps = r["enc_bytes"] / (r["kern_ms"] * 1e-3) / 1e9
    line = {
        "metric": "patternkv_encode_GBps",
        "value": r["enc_gbps"],
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["enc_ms"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16-in/f64-exact",
        "data": "synthetic (reference KeyModel/ValueModel family on device, pool of "
                f"{min(args.pool, U)} distinct units tiled)",
        "config": {"workload": f"cfg2 Llama-3.1-8B KV: batch {args.batch} x {args.layers} layers x {args.kv_heads} "
                               f"KV heads per GPU, {T}-token prefill, d=128, {args.bits}-bit, |M|={args.patterns}, "
                               f"G=W=128", "units_per_gpu": U, "tokens": T, "bits": args.bits,
                   "l2": "inputs 34 GB/GPU >> 126 MB L2 (no flush needed)", "parallelism": f"units x{world}"},
        "roofline": {"bound": "hbm", "achieved": kern_gbps, "peak": peak, "unit": "GB/s",
                     "frac": kern_gbps / peak, "traffic": ncu_traffic("encode", U * committed), "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": r["enc_bytes"],
                     "kernel": f"encode_tc_kernel<{args.bits}> (K1-TC)", "bytes_per_token_unit": r["bpt"],
                     "issue_ceiling": enc_ceiling},
        "decode_attn": {"tokens_per_s": r["tok_s"], "ms_per_step": r["att_ms"], "GBps": r["att_gbps"],
                        "frac": r["att_gbps"] / peak, "bytes_per_step": r["att_bytes"], "gqa": args.gqa,
                        "context": T, "e2e_ms_per_step": results.get("e2e_attn_ms"),
                        "kernel": "attn_chunk_kernel + attn_merge_kernel", "clocks": r["clk_a"],
                        "traffic": ncu_traffic("attn", U * committed)},
        "mining": {"ms": r["mine_ms"], "units": min(args.pool, U), "sides": 2, "tokens": T,
                   "patterns": args.patterns,
                   "kernel": "kmeans_kernel<__half, TC>: distance GEMM on tcgen05 (TMA + TMEM), fp64 means/objective"},
        "cpu_baseline": cpu,
        "e2e": {"value": results["e2e"]["gbps"], "unit": "GB/s", "h2d_bytes_per_step": results["e2e"]["h2d"],
                "d2h_bytes_per_step": results["e2e"]["d2h"],
                "note": f"{min(args.e2e_units, U)} units per step from pinned host memory, streamed in "
                        f"{args.e2e_slices} slices (H2D of slice i+1 overlaps the encode of slice i)"},
        "gpu_launches": r["launches"],
        "clocks": r["clk"],
    }
    other = [b for b in results if isinstance(b, int) and b != args.bits]
    if other:
        o = results[other[0]]
        line[f"bits{other[0]}"] = {"encode_GBps": o["enc_gbps"], "encode_frac": o["enc_gbps"] / world / peak,
                                   "decode_tokens_per_s": o["tok_s"], "decode_frac": o["att_gbps"] / peak,
                                   "decode_ms": o["att_ms"], "mining_ms": o["mine_ms"]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
