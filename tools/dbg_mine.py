import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_05176_b200 as P
from oracle import pkv_oracle as O
T = int(os.environ.get("T", "1024"))
k, v = O.synth_unit(5, T, 128)
x = torch.from_numpy(k.astype(np.float16)[None]).cuda()
c = P.PatternKVCache(P.EngineConfig(bits=2, pattern_count=16), 1, 128, dtype=torch.float16, max_tokens=T + 256)
h, n, lab = c.mine(0, x, seed=0, labels=True)
print("niter", n, "hist", h[0, :4], "nk", c.pattern_counts())
cen, l, hh = O.kmeans(k.astype(np.float16).astype(np.float64), 16, 0)
print("oracle", len(hh), hh[:4])
print("pat0", c.patterns(0)[0, 0, :4].cpu().numpy(), cen[0, :4])
