"""Mining timing: K and V sides timed separately (CUDA events), U units x T tokens."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_05176_b200 as P
from paper_2510_05176_b200.synth import synth_kv

U = int(os.environ.get("U", "256")); T = int(os.environ.get("T", "32768"))
k, v = synth_kv(U, T, 128, seed=1234)
cfg = P.EngineConfig(bits=2, pattern_count=int(os.environ.get("P", "32")))
c = P.PatternKVCache(cfg, U, 128, dtype=torch.float16, max_tokens=T + 256)
c.reserve_mining(T)
ev = lambda: torch.cuda.Event(enable_timing=True)
for i in range(int(os.environ.get("REPS", "3"))):
    c.reset(keep_patterns=False)
    torch.cuda.synchronize()
    a, b, d, e, f, g = ev(), ev(), ev(), ev(), ev(), ev()
    a.record(); hk, nk = c.mine(0, k, seed=0); b.record()
    d.record(); hv, nv = c.mine(1, v, seed=1); e.record()
    c.reset(keep_patterns=False)
    f.record(); c.prefill(k, v); g.record()
    torch.cuda.synchronize()
    print(f"K {a.elapsed_time(b):.1f} ms ({int(nk.max())} rounds)  V {d.elapsed_time(e):.1f} ms ({int(nv.max())} rounds)"
          f"  prefill(both sides + encode) {f.elapsed_time(g):.1f} ms", flush=True)
