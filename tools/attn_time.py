"""Decode-attention timing for A/B builds (same box, one process per library):

    for lib in a.so b.so; do PKV_LIB=$lib python tools/attn_time.py --units 512; done

Builds a cfg2-shaped cache (32K-token prefill, d = 128, |M| = 32, GQA 4) of --units units at
2 and 4 bits through the public API and prints the mean decode_attention time (CUDA events,
20 timed calls after 5 warm-ups) and the algorithmic HBM fraction (bench.py's byte model).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_05176_b200 as P  # noqa: E402
from paper_2510_05176_b200.synth import synth_kv  # noqa: E402
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=512)
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--gqa", type=int, default=4)
    ap.add_argument("--bits", default="2,4")
    args = ap.parse_args()
    U, T, D = args.units, args.tokens, 128
    k, v = synth_kv(min(U, 64), T, D, seed=0)
    reps = (U + k.shape[0] - 1) // k.shape[0]
    k = k.repeat(reps, 1, 1)[:U].contiguous()
    v = v.repeat(reps, 1, 1)[:U].contiguous()
    peak = bench.hbm_peak()[0] if hasattr(bench, "hbm_peak") else 6535.1
    for bits in [int(b) for b in args.bits.split(",")]:
        cfg = P.EngineConfig(bits=bits, pattern_count=32)
        cache = P.PatternKVCache(cfg, U, D, dtype=torch.float16, max_tokens=T + 256)
        cache.reserve_mining(T)
        cache.prefill(k, v)
        q = torch.randn((U, args.gqa, D), device="cuda")
        out = torch.empty_like(q)
        for _ in range(5):
            cache.decode_attention(q, out=out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            cache.decode_attention(q, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        committed = T - 128
        nbytes = bench.attn_bytes_per_step(U, committed, 128, bits, 32, args.gqa)
        gbps = nbytes / (ms * 1e-3) / 1e9
        print(f"{os.path.basename(os.environ.get('PKV_LIB', 'default'))} bits={bits} U={U} {ms:.3f} ms "
              f"{gbps:.0f} GB/s frac={gbps / peak:.3f}", flush=True)
        del cache


if __name__ == "__main__":
    main()
