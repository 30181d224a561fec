"""K1-TC rare-path counters on bench-shaped data (cfg2: 32K tokens, d = 128, P = 32):
stats[0] fp64 re-matches, [1] exact-division code fix-ups, [2] pruning survivors,
[3] slow exact-extrema groups (K k_slow channels + V tokens).  One GPU process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_05176_b200 as P  # noqa: E402
from paper_2510_05176_b200.synth import synth_kv  # noqa: E402

U, T = int(sys.argv[1]) if len(sys.argv) > 1 else 32, 32768
k, v = synth_kv(U, T, 128, seed=0)
for bits in (2, 4):
    cache = P.PatternKVCache(P.EngineConfig(bits=bits, pattern_count=32), U, 128, dtype=torch.float16,
                             max_tokens=T + 256, stats=True)
    cache.reserve_mining(T)
    cache.prefill(k, v)
    pk, pv = cache.patterns(0)[:, :32], cache.patterns(1)[:, :32]
    c2 = P.PatternKVCache(P.EngineConfig(bits=bits, pattern_count=32), U, 128, dtype=torch.float16,
                          max_tokens=T + 256, stats=True)
    c2.set_patterns(0, pk)
    c2.set_patterns(1, pv)
    c2.commit_prefill(k, v)  # encode only (no mining): the counters of one K1-TC pass
    import ctypes as C
    from paper_2510_05176_b200 import _lib
    from paper_2510_05176_b200.cache import _ptr, _stream
    buf = torch.zeros(4, dtype=torch.int32, device="cuda")
    _lib.call("pkv_cache_read", c2._h, b"stats", 0, 16, _ptr(buf), _stream())
    s = buf.cpu().tolist()
    tu = U * (T - 128)
    nb = U * (T - 128) // 128
    print(f"bits={bits}: refines {s[0]} ({s[0] / tu:.2e}/token), exact-div {s[1]} ({s[1] / tu / 128:.2e}/element), "
          f"survivors {s[2]} ({s[2] / tu:.3f}/token-side), slow groups {s[3]} "
          f"(K channels: {s[3] / (nb * 128):.3f} of groups if all K)")
