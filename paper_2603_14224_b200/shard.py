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


class OutputExchange:
    """The output all-gather fused into the decode step over NVLink peer memory.

    Replaces ``gather_outputs``' NCCL all-gather + reassembly. Every rank owns a bf16 buffer
    [units_total, Gq, 128], which is the model layout [layers, batch, kv_heads * Gq, 128], since
    the row of a unit is its global id. It also owns a u64 arrival counter. CUDA IPC hands
    every rank the other ranks' buffers and counters. ``batch.decode_step(...,
    exchange=self)`` makes the attention epilogue store each finished unit's rows into every
    rank's buffer and release one arrival on every counter (``sikv_decode_step_x``).
    ``wait()`` then orders a stream after the current step of all ranks.

    ``ranks`` simulates a world inside one process, one exchange per rank, sharing
    buffers without IPC. Tests use it to run every rank's shard on a single GPU.

    The buffer holds the latest step. The next step's stores overwrite it, so whatever reads
    it must be ordered before any rank enqueues its next exchange step. In a model forward the
    layers' other collectives give that order; a standalone loop needs a barrier.
    """

    def __init__(self, plan: ShardPlan, gq: int, rank: int, device, group=None, ranks: list | None = None):
        import ctypes as C

        from . import _lib as L_
        self.plan, self.gq, self.rank = plan, gq, rank
        self.total = plan.layers * plan.batch * plan.kv_heads
        if plan.world > L_.MAX_PEERS:
            raise ValueError(f"the fused exchange supports at most {L_.MAX_PEERS} ranks, got {plan.world}")
        dev = torch.device(device)
        self.buffer = torch.zeros(self.total, gq, 128, dtype=torch.bfloat16, device=dev)
        self.counter = torch.zeros(1, dtype=torch.int64, device=dev)      # u64 arrivals
        gid = plan.local_units(rank).to(torch.int32)
        self.gid = gid.to(dev)
        self.gid_heads = (gid[:, None] * gq + torch.arange(gq, dtype=torch.int32)[None, :]).reshape(-1).to(dev)
        self.epoch = 0
        self._opened = []
        if ranks is not None:                       # in-process world (tests)
            peers = [(r.buffer.data_ptr(), r.counter.data_ptr()) for r in ranks] + \
                    [(self.buffer.data_ptr(), self.counter.data_ptr())]
            if rank != len(ranks) or rank >= plan.world:
                raise ValueError("ranks must hold the exchanges of ranks 0 .. rank-1, in order")
            for i, r in enumerate(ranks):           # earlier ranks learn about this one
                r._peers[rank] = peers[rank]
                r._build()
            self._peers = dict(enumerate(peers))
        elif plan.world == 1:
            self._peers = {0: (self.buffer.data_ptr(), self.counter.data_ptr())}
        else:
            import torch.distributed as dist
            mine = (self._handle(self.buffer), self._handle(self.counter))
            allh = [None] * plan.world
            dist.all_gather_object(allh, mine, group=group)
            self._peers = {}
            for r, (hb, hc) in enumerate(allh):
                if r == rank:
                    self._peers[r] = (self.buffer.data_ptr(), self.counter.data_ptr())
                else:
                    self._peers[r] = (self._open(*hb), self._open(*hc))
        self._C, self._L = C, L_
        self._build()

    # ---- CUDA IPC (the offset: the caching allocator hands out interior pointers)
    def _handle(self, t: torch.Tensor):
        import ctypes as C

        from . import _lib as L_
        h = (C.c_char * 64)()
        off = C.c_size_t(0)
        L_.call("sikv_ipc_handle", L_.ptr(t), h, C.byref(off))
        return bytes(h), int(off.value)

    def _open(self, handle: bytes, offset: int) -> int:
        import ctypes as C

        from . import _lib as L_
        h = (C.c_char * 64).from_buffer_copy(handle)
        p = C.c_void_p(0)
        L_.call("sikv_ipc_open", h, C.byref(p))
        self._opened.append(p.value)
        return p.value + offset

    def _build(self) -> None:
        from . import _lib as L_
        self._structs = {}
        n = len(self._peers)
        for per_head, gid in ((False, self.gid), (True, self.gid_heads)):
            x = L_.Exchange()
            x.npeers = n
            for r in range(n):
                x.out[r], x.flag[r] = self._peers[r]
            x.unit_gid = gid.data_ptr()
            self._structs[per_head] = x

    def cstruct(self, units: int, gq: int):
        """The C struct for a decode over `units` query units of `gq` heads (the group-sum
        policy: the local units; the per-q-head policy: one query unit per head)."""
        if units == self.gid.numel() and gq == self.gq:
            return self._structs[False]
        if units == self.gid_heads.numel() and gq == 1:
            return self._structs[True]
        raise ValueError(f"exchange built for {self.gid.numel()} units x {self.gq} heads, "
                         f"got {units} x {gq}")

    def wait(self, stream=None) -> torch.Tensor:
        """Enqueue (on `stream`, default the current one) the wait for this step of every rank;
        returns the model-layout view [layers, batch, kv_heads * Gq, 128] of the buffer."""
        from . import _lib as L_
        self.epoch += 1
        st = L_.P((stream or torch.cuda.current_stream()).cuda_stream)
        L_.call("sikv_exchange_wait", L_.ptr(self.counter), self.epoch * self.total * self.gq, st)
        p = self.plan
        return self.buffer.view(p.layers, p.batch, p.kv_heads * self.gq, 128)

    def close(self) -> None:
        from . import _lib as L_
        for ptr in self._opened:
            L_.call("sikv_ipc_close", ptr)
        self._opened = []
