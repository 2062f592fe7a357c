"""KV-head sharding of decode units across the GPUs of one node.

Decode units (layer, batch, KV head) are independent: per-unit codebook, mu, alpha,
selection and attention.  Rank r of N owns KV heads [r*H/N, (r+1)*H/N) for every layer
and batch element, so the decode step needs no collective on the data path; the only
exchange is one all-gather of the step's attention outputs (bf16 [layers, batch, H_q, D]).
"""

from __future__ import annotations

import torch


def heads_of(rank: int, world: int, kv_heads: int) -> range:
    if kv_heads % world:
        raise ValueError(f"{kv_heads} KV heads do not shard over {world} ranks")
    per = kv_heads // world
    return range(rank * per, (rank + 1) * per)


def local_units(layers: int, batch: int, kv_heads: int, rank: int, world: int) -> torch.Tensor:
    """Global unit ids ((layer * batch + b) * kv_heads + h) owned by `rank`, in the
    (layer, b, local head) order the rank stores them in."""
    hs = torch.tensor(list(heads_of(rank, world, kv_heads)))
    lb = torch.arange(layers * batch)
    return (lb[:, None] * kv_heads + hs[None, :]).reshape(-1)


def gather_outputs(local_out: torch.Tensor, layers: int, batch: int, kv_heads: int, world: int,
                   group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather per-rank outputs [layers*batch*H_local, Gq, D] into the model layout
    [layers, batch, kv_heads * Gq, D] (q head = kv_head * Gq + g)."""
    import torch.distributed as dist
    ul, gq, d = local_out.shape
    hl = kv_heads // world
    if world == 1:
        flat = local_out
    else:
        flat = torch.empty(world * ul, gq, d, dtype=local_out.dtype, device=local_out.device)
        dist.all_gather_into_tensor(flat, local_out.contiguous(), group=group)
    # flat: [world, layers*batch, hl, gq, d] -> [layers*batch, world*hl, gq, d]
    x = flat.view(world, layers * batch, hl, gq, d).permute(1, 0, 2, 3, 4).reshape(layers, batch, kv_heads * gq, d)
    if out is not None:
        out.copy_(x)
        return out
    return x
