"""Wider encode fuzzing on the GPU: verify.run_suite('encode', seed) over many seeds (whole
caches through K1-TC / K1 / K2 / decode-flush refresh, checked per group against the
exhaustive GPU matcher and the gate), plus K1-TC == K1 arena equality on random and
heavy-tie data with the deferred fix-up list full and empty.  Prints one JSON line.
    python tools/fuzz_encode.py [n_seeds]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_05176_b200 import verify  # noqa: E402
import paper_2510_05176_b200 as P  # noqa: E402
from paper_2510_05176_b200.config import EngineConfig  # noqa: E402

ARENAS = [("kcodes", torch.uint8), ("vcodes", torch.uint8), ("kidx", torch.int16), ("vidx", torch.int16),
          ("kparam64", torch.float64), ("vparam64", torch.float64), ("kparam32", torch.float32),
          ("vparam32", torch.float32), ("vdiag", torch.float64)]


def arenas(tc, cfg, k, v):
    os.environ["PKV_ENCODE_TC"] = "1" if tc else "0"
    U, T, d = k.shape
    c = P.PatternKVCache(cfg, U, d, dtype=torch.float16, max_tokens=T + 256, record_decisions=True)
    c.prefill(k, v)
    out = {}
    for name, dt in ARENAS:
        nb = c.arena_bytes(name)
        if nb:
            out[name] = c.read(name, dt, (nb // torch.empty((), dtype=dt).element_size(),)).cpu()
    return out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    t0 = time.time()
    suite_fail = []
    for seed in range(100, 100 + n):
        for r in verify.run_suite("encode", seed):
            if not r.passed:
                suite_fail.append((seed, r.name, r.detail[:200]))
    tc_fail, cases = [], 0
    for seed in range(n):
        g = torch.Generator(device="cuda").manual_seed(seed)
        U, T = 4, 1024 + 128 * (seed % 5)
        heavy = seed % 2 == 1
        if heavy:
            k = torch.randint(-3, 4, (U, T, 128), generator=g, device="cuda").half() * 0.5
            v = torch.randint(-2, 3, (U, T, 128), generator=g, device="cuda").half()
        else:
            k = (torch.randn((U, T, 128), generator=g, device="cuda") * (1 + seed % 3)).half()
            v = torch.randn((U, T, 128), generator=g, device="cuda").half()
        for bits in (2, 4):
            for cap in (None, "7"):
                if cap:
                    os.environ["PKV_FIX_CAP"] = cap
                else:
                    os.environ.pop("PKV_FIX_CAP", None)
                cfg = EngineConfig(bits=bits, pattern_count=8 + 8 * (seed % 4))
                a, b = arenas(True, cfg, k, v), arenas(False, cfg, k, v)
                cases += 1
                for name, _ in ARENAS:
                    if name in a and not torch.equal(a[name], b[name]):
                        tc_fail.append((seed, bits, cap, name))
    os.environ.pop("PKV_FIX_CAP", None)
    print(json.dumps({"encode_suite_seeds": n, "encode_suite_failures": suite_fail, "k1tc_vs_k1_cases": cases,
                      "k1tc_vs_k1_failures": tc_fail, "seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
