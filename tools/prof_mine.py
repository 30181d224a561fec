"""Mining-only workload for ncu captures: U units x T tokens; SIDE=k|v|both."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_05176_b200 as P
from paper_2510_05176_b200.synth import synth_kv

U = int(os.environ.get("U", "16")); T = int(os.environ.get("T", "32768")); side = os.environ.get("SIDE", "both")
k, v = synth_kv(U, T, 128, seed=1234)
c = P.PatternKVCache(P.EngineConfig(bits=2, pattern_count=32), U, 128, dtype=torch.float16, max_tokens=T + 256)
c.reserve_mining(T)
for i in range(int(os.environ.get("REPS", "2"))):
    c.reset(keep_patterns=False)
    if side == "both":
        c.prefill(k, v)
    else:
        c.mine(0 if side == "k" else 1, k if side == "k" else v, seed=0)
torch.cuda.synchronize()
print("ok")
