import sys, time, torch, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2510_05176_b200 as P
from paper_2510_05176_b200.synth import synth_kv
U, T = 256, 32768
k, v = synth_kv(U, T, 128, seed=1234)
for bits in (2,):
    cfg = P.EngineConfig(bits=bits, pattern_count=32)
    c = P.PatternKVCache(cfg, U, 128, dtype=torch.float16, max_tokens=T + 256)
    c.reserve_mining(T)
    for i in range(3):
        c.reset(keep_patterns=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hk, nk = c.mine(0, k, seed=0)
        hv, nv = c.mine(1, v, seed=1)
        e1.record(); torch.cuda.synchronize()
        print("mine ms", e0.elapsed_time(e1), "rounds K", np.bincount(nk).nonzero()[0], "V", np.bincount(nv).nonzero()[0], flush=True)
    pk = c.patterns(0)[:, :32].clone(); pv = c.patterns(1)[:, :32].clone()
    print("hist0", hk[0, :3], hv[0, :3])
