"""Sharding of decode units across the GPUs of one node.

Decode units (layer, batch element, KV head) are independent: each has its own codebook,
mu, alpha, selection and attention, so the decode step needs no collective on the data
path.  The only exchange is one all-gather of the step's attention outputs into the model
layout [layers, batch, H_q, D].

The partition is 2-D, KV head x batch:

* ``head_parts = gcd(kv_heads, world)`` groups of KV heads;
* ``batch_parts = world / head_parts`` slices of the batch (must divide the batch).

Rank r owns head group ``r // batch_parts`` and batch slice ``r % batch_parts`` for every
layer.  C2 (8 KV heads) on 8 GPUs is a pure head split (1 KV head, 512 units per GPU);
C4 (Qwen2.5-7B, 4 KV heads, batch 64) on 8 GPUs is 4 head groups x 2 batch halves
(896 units per GPU); C3 (batch 1) on 2/4/8 GPUs splits the 8 KV heads.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class ShardPlan:
    layers: int
    batch: int
    kv_heads: int
    world: int

    def __post_init__(self):
        if self.world < 1:
            raise ValueError(f"world size must be >= 1, got {self.world}")
        if self.batch % self.batch_parts:
            raise ValueError(f"{self.kv_heads} KV heads x batch {self.batch} do not shard over {self.world} "
                             f"ranks (batch must split into {self.batch_parts} parts)")

    @property
    def head_parts(self) -> int:
        return math.gcd(self.kv_heads, self.world)

    @property
    def batch_parts(self) -> int:
        return self.world // self.head_parts

    @property
    def heads_per_rank(self) -> int:
        return self.kv_heads // self.head_parts

    @property
    def batch_per_rank(self) -> int:
        return self.batch // self.batch_parts

    @property
    def units_per_rank(self) -> int:
        return self.layers * self.batch_per_rank * self.heads_per_rank

    def heads(self, rank: int) -> range:
        hp = rank // self.batch_parts
        return range(hp * self.heads_per_rank, (hp + 1) * self.heads_per_rank)

    def batches(self, rank: int) -> range:
        bp = rank % self.batch_parts
        return range(bp * self.batch_per_rank, (bp + 1) * self.batch_per_rank)

    def local_units(self, rank: int) -> torch.Tensor:
        """Global unit ids ((layer * batch + b) * kv_heads + h) owned by `rank`, in the
        (layer, local b, local head) order the rank stores them in."""
        if not 0 <= rank < self.world:
            raise ValueError(f"rank {rank} outside world {self.world}")
        hs = torch.tensor(list(self.heads(rank)))
        bs = torch.tensor(list(self.batches(rank)))
        ls = torch.arange(self.layers)
        ids = (ls[:, None, None] * self.batch + bs[None, :, None]) * self.kv_heads + hs[None, None, :]
        return ids.reshape(-1)


def heads_of(rank: int, world: int, kv_heads: int) -> range:
    """KV heads of `rank` under a pure head split (kv_heads divisible by world)."""
    if kv_heads % world:
        raise ValueError(f"{kv_heads} KV heads do not shard over {world} ranks")
    per = kv_heads // world
    return range(rank * per, (rank + 1) * per)


def local_units(layers: int, batch: int, kv_heads: int, rank: int, world: int) -> torch.Tensor:
    return ShardPlan(layers, batch, kv_heads, world).local_units(rank)


def assemble(flat: torch.Tensor, plan: ShardPlan) -> torch.Tensor:
    """[world * units_per_rank, Gq, D] rank-major outputs -> [layers, batch, kv_heads * Gq, D]
    (q head = kv_head * Gq + g)."""
    _, gq, d = flat.shape
    x = flat.view(plan.head_parts, plan.batch_parts, plan.layers, plan.batch_per_rank, plan.heads_per_rank, gq, d)
    # -> layers, batch_parts, batch_per_rank, head_parts, heads_per_rank, gq, d
    return x.permute(2, 1, 3, 0, 4, 5, 6).reshape(plan.layers, plan.batch, plan.kv_heads * gq, d)


def gather_outputs(local_out: torch.Tensor, layers: int, batch: int, kv_heads: int, world: int,
                   group=None, out: torch.Tensor | None = None, flat: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather per-rank outputs [units_per_rank, Gq, D] (NCCL all_gather_into_tensor) into
    the model layout [layers, batch, kv_heads * Gq, D]."""
    import torch.distributed as dist
    plan = ShardPlan(layers, batch, kv_heads, world)
    ul, gq, d = local_out.shape
    if ul != plan.units_per_rank:
        raise ValueError(f"expected {plan.units_per_rank} local units, got {ul}")
    if world == 1:
        g = local_out
    else:
        g = flat if flat is not None else torch.empty(world * ul, gq, d, dtype=local_out.dtype,
                                                     device=local_out.device)
        dist.all_gather_into_tensor(g, local_out.contiguous(), group=group)
    x = assemble(g, plan)
    if out is not None:
        out.copy_(x)
        return out
    return x
