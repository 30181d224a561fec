import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2510_05176_b200 import verify
from paper_2510_05176_b200.cache import PatternKVCache
from paper_2510_05176_b200.export import export_unit
from oracle import pkv_oracle as O
seed = 151
rng = np.random.default_rng(seed)
for i in range(6):
    repro, cfg, k, v, T, S, dtype = verify._encode_instance(rng, i, seed)
print(repro)
U, _, d = k.shape
cache = PatternKVCache(cfg, U, d, dtype=dtype, max_tokens=T + S + 2 * cfg.group_size)
cache.prefill(k[:, :T], v[:, :T])
for s in range(T, T + S):
    cache.append(k[:, s], v[:, s])
kx = k.double().cpu().numpy(); vx = v.double().cpu().numpy()
knobs = O.Knobs(bits=cfg.bits, pattern_count=cfg.pattern_count, group_size=cfg.group_size, residual_window=cfg.residual_window,
                use_v_gate=cfg.use_v_gate, generate_new_patterns=cfg.generate_new_patterns, seed=cfg.seed)
u = 0
h = O.replay(kx[u, :T], vx[u, :T], kx[u, T:], vx[u, T:], knobs)
st = export_unit(cache, u, with_bytes=False)
print("kpat equal", np.array_equal(st.kpat, h.kpat), "kidx", np.array_equal(st.k_idx, np.concatenate([b[5] for b in h.k_blocks])),
      "kcodes", np.array_equal(st.k_codes, np.concatenate([b[4] for b in h.k_blocks])))
b = 4
s0, ln = int(st.kb_start[b]), int(st.kb_len[b])
r = kx[u, s0:s0+ln] - st.kpat[st.k_idx[s0:s0+ln]]
c = 3
vals = r[:, c]; sc = st.k_scale[b, c]; z = st.k_zero[b, c]; codes = st.k_codes[s0:s0+ln, c]
deq = sc * codes + z
print("scale", sc, "zero", z, "spread", vals.max()-vals.min(), "max|v|", np.abs(vals).max(), "maxerr-scale/2", np.abs(deq-vals).max()-sc/2, "4eps spread", 4*np.finfo(float).eps*(vals.max()-vals.min()))
