"""Multi-GPU placement of PatternKV units.

The codec's units (batch, layer, kv-head) are independent, so
mining, encode and append-and-refresh shard with NO data-path collective: each
rank owns a contiguous slice of units (weak scaling).  The only exchange step
is in decode attention when the KV heads of one (batch, layer) are split
across ranks (Llama-70B cfg5): every rank produces the outputs of its heads
and the model's next layer needs all of them -> one all-gather of
[B, L, Hkv_local, G, d] per step.  For a sequence split of one head (cfg3 at 8
GPUs) ranks exchange partial (o, m, l) and LSE-merge.

Process model: one process per GPU, torch.distributed (NCCL on GPU, gloo in
the CPU tests), launched by torchrun.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of n items: [start, stop) of `rank`."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_units(batch: int, layers: int, kv_heads: int, world: int, rank: int, by: str = "batch"):
    """Unit ids (flattened b*L*H + l*H + h) owned by `rank`.

    by="batch": whole sequences per rank (cfg2/cfg4, no collective at all);
    by="head":  every rank holds kv_heads/world heads of every (batch, layer)
                (cfg5: the attention outputs are all-gathered along heads)."""
    if by == "batch":
        s, e = shard_range(batch, world, rank)
        return [b * layers * kv_heads + l * kv_heads + h for b in range(s, e) for l in range(layers)
                for h in range(kv_heads)]
    if by == "head":
        if kv_heads % world:
            raise ValueError(f"{kv_heads} KV heads do not split over {world} ranks")
        s, e = shard_range(kv_heads, world, rank)
        return [b * layers * kv_heads + l * kv_heads + h for b in range(batch) for l in range(layers)
                for h in range(s, e)]
    raise ValueError(f"unknown sharding {by!r}")


def _host_staged(t: torch.Tensor, group) -> bool:
    """gloo moves only host tensors: device tensors are staged through host memory."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def gather_head_outputs(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather head-sharded attention outputs.

    local: [B, L, Hkv_local, G, d] on this rank -> [B, L, Hkv, G, d] with rank r's
    heads at [r*Hkv_local, (r+1)*Hkv_local)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    dev = local.device
    local = local.contiguous()
    if _host_staged(local, group):
        local = local.cpu()
    parts = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(parts, local, group=group)
    else:
        dist.all_gather(list(parts.unbind(0)), local, group=group)
    parts = parts.to(dev)
    # [world, B, L, h, G, d] -> [B, L, world*h, G, d]
    return parts.permute(1, 2, 0, 3, 4, 5).reshape(local.shape[0], local.shape[1], -1, *local.shape[3:])


def lse_merge(o: torch.Tensor, m: torch.Tensor, l: torch.Tensor) -> torch.Tensor:
    """Merge n partial softmax-attention results over disjoint token sets.

    o [n, ..., d] unnormalised sums sum_t e^(s_t - m) v_t, m [n, ...] partial
    maxima, l [n, ...] partial sums sum_t e^(s_t - m).  Returns the normalised
    output over the union."""
    M = m.max(dim=0).values
    w = torch.exp(m - M)
    w = torch.where(torch.isfinite(m), w, torch.zeros_like(w))
    num = (o * w[..., None]).sum(dim=0)
    den = (l * w).sum(dim=0)
    return num / den[..., None]


def gather_and_merge_partials(o: torch.Tensor, m: torch.Tensor, l: torch.Tensor, group=None) -> torch.Tensor:
    """Sequence-split decode attention: every rank holds a token range of the
    same heads; exchange (o, m, l) once and LSE-merge locally."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return lse_merge(o[None], m[None], l[None])
    packed = torch.cat([o.reshape(-1), m.reshape(-1), l.reshape(-1)])
    dev = packed.device
    if _host_staged(packed, group):
        packed = packed.cpu()
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    parts = [p.to(dev) for p in parts]
    no, nm = o.numel(), m.numel()
    os_ = torch.stack([p[:no].view_as(o) for p in parts])
    ms = torch.stack([p[no:no + nm].view_as(m) for p in parts])
    ls = torch.stack([p[no + nm:].view_as(l) for p in parts])
    return lse_merge(os_, ms, ls)


def sequence_block_range(n_blocks: int, world: int, rank: int) -> tuple[int, int, bool]:
    """Committed-block range [b0, b1) a rank attends in a sequence split, and whether it also
    takes the exact window (the last rank: it holds the newest tokens)."""
    b0, b1 = shard_range(n_blocks, world, rank)
    return b0, b1, rank == world - 1


def sequence_split_attention(cache, q: torch.Tensor, group=None, sm_scale: float | None = None) -> torch.Tensor:
    """Decode attention with the committed tokens of every unit split across the ranks of
    `group` (cfg3 at 8 GPUs: 4 KV heads cannot occupy 8 GPUs by head sharding alone).  Each
    rank runs pkv_decode_attn_partial over its block range, the ranks exchange (o, m, l) once
    and LSE-merge locally.  Returns the normalised [U, G, D] output on every rank."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b0, b1, win = sequence_block_range(cache.info().n_blocks, world, rank)
    o, m, l = cache.decode_attention_partial(q, b0, b1, with_window=win, sm_scale=sm_scale)
    if world == 1:
        return lse_merge(o[None], m[None], l[None])
    return gather_and_merge_partials(o, m, l, group=group)
