"""Head-sharded decode bookkeeping on CPU: world_size 2 over gloo reassembles exactly the
single-process output layout (no GPU needed)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_14224_b200.shard import gather_outputs, heads_of, local_units

LAYERS, BATCH, KVH, GQ, D = 3, 2, 4, 2, 8


def fake_out(units: torch.Tensor) -> torch.Tensor:
    # the "attention output" of unit u, head g, channel d is a unique number
    g = torch.arange(GQ)[None, :, None]
    d = torch.arange(D)[None, None, :]
    return (units[:, None, None] * 1000 + g * 100 + d).to(torch.float32)


def reference_layout() -> torch.Tensor:
    all_units = torch.arange(LAYERS * BATCH * KVH)
    o = fake_out(all_units).view(LAYERS, BATCH, KVH, GQ, D)
    return o.reshape(LAYERS, BATCH, KVH * GQ, D)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        units = local_units(LAYERS, BATCH, KVH, rank, world)
        got = gather_outputs(fake_out(units), LAYERS, BATCH, KVH, world)
        q.put((rank, bool(torch.equal(got, reference_layout()))))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_heads_partition():
    assert [list(heads_of(r, 2, 8)) for r in range(2)] == [[0, 1, 2, 3], [4, 5, 6, 7]]
    allu = torch.cat([local_units(2, 3, 8, r, 4) for r in range(4)])
    assert sorted(allu.tolist()) == list(range(2 * 3 * 8))
    with pytest.raises(ValueError):
        heads_of(0, 3, 8)


def test_single_rank_layout():
    assert torch.equal(gather_outputs(fake_out(local_units(LAYERS, BATCH, KVH, 0, 1)), LAYERS, BATCH, KVH, 1),
                       reference_layout())


def test_gloo_world2_allgather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
