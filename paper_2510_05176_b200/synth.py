"""On-device synthetic KV of the reference generator's model family
(analysis.py:248-370: KeyModel = drifting channel profile with outlier
channels + noise, ValueModel = clustered values with token-consistent home
clusters).  torch RNG, so values differ from the numpy generator; used only
for throughput runs (parity tests regenerate exact reference inputs with the
oracle's restatement)."""

from __future__ import annotations

import torch


@torch.no_grad()
def synth_kv(n_units: int, tokens: int, head_dim: int, seed: int = 0, dtype=torch.float16, device="cuda",
             outlier=((3, 32.0),), drift=None, noise=0.05, clusters=32, spread=5.0, within=0.2,
             consistency=0.9, vocab=1024, chunk: int = 32):
    """K, V tensors [n_units, tokens, head_dim] in `dtype` on `device`."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if drift is None:
        drift = 1.0 / tokens
    k = torch.empty((n_units, tokens, head_dim), dtype=dtype, device=device)
    v = torch.empty_like(k)
    tok = torch.randint(0, vocab, (tokens,), generator=g, device=device)
    a = (torch.arange(tokens, device=device, dtype=torch.float32) * drift).clamp(0.0, 1.0)[None, :, None]
    for u0 in range(0, n_units, chunk):
        n = min(chunk, n_units - u0)

        def profile():
            mag = torch.rand((n, head_dim), generator=g, device=device) + 0.5
            sign = torch.randint(0, 2, (n, head_dim), generator=g, device=device).float() * 2 - 1
            p = mag * sign
            for ch, mul in outlier:
                p[:, ch] *= mul
            return p

        p0, p1 = profile(), profile()
        kk = (1.0 - a) * p0[:, None, :] + a * p1[:, None, :]
        if noise > 0:
            kk += noise * torch.randn((n, tokens, head_dim), generator=g, device=device)
        k[u0:u0 + n] = kk.to(dtype)
        del kk
        cen = spread * torch.randn((n, clusters, head_dim), generator=g, device=device)
        home = torch.randint(0, clusters, (n, vocab), generator=g, device=device)
        stray = torch.randint(0, clusters, (n, tokens), generator=g, device=device)
        keep = torch.rand((n, tokens), generator=g, device=device) <= consistency
        cl = torch.where(keep, home[:, tok], stray)
        vv = torch.gather(cen, 1, cl[:, :, None].expand(n, tokens, head_dim))
        if within > 0:
            vv += within * torch.randn((n, tokens, head_dim), generator=g, device=device)
        v[u0:u0 + n] = vv.to(dtype)
        del vv
    return k, v
