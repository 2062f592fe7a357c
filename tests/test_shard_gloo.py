"""Sharded decode across ranks with torch.distributed world sizes 2 and 4.

* CPU (gloo): the ShardPlan partition (KV head x batch) covers every unit exactly once and
  the all-gather + assemble reproduces the single-process output layout.
* GPU (gloo, every rank on cuda:0): each rank builds and decodes only its own shard with
  the real kernels, the CPU copies are all-gathered, and the assembled model output equals
  the single-process decode of the whole batch.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_14224_b200.shard import ShardPlan, assemble, gather_outputs, heads_of, local_units

LAYERS, BATCH, KVH, GQ, D = 3, 2, 4, 2, 8


def fake_out(units: torch.Tensor, gq: int = GQ, d: int = D) -> torch.Tensor:
    # the "attention output" of unit u, head g, channel d is a unique number
    g = torch.arange(gq)[None, :, None]
    dd = torch.arange(d)[None, None, :]
    return (units[:, None, None] * 1000 + g * 100 + dd).to(torch.float32)


def reference_layout(layers=LAYERS, batch=BATCH, kvh=KVH) -> torch.Tensor:
    all_units = torch.arange(layers * batch * kvh)
    o = fake_out(all_units).view(layers, batch, kvh, GQ, D)
    return o.reshape(layers, batch, kvh * GQ, D)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


def _fake_worker(rank, world, port, q, layers, batch, kvh):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        units = local_units(layers, batch, kvh, rank, world)
        got = gather_outputs(fake_out(units), layers, batch, kvh, world)
        q.put((rank, bool(torch.equal(got, reference_layout(layers, batch, kvh)))))
    finally:
        dist.destroy_process_group()


def test_plan_partition():
    assert [list(heads_of(r, 2, 8)) for r in range(2)] == [[0, 1, 2, 3], [4, 5, 6, 7]]
    for (layers, batch, kvh, world) in [(2, 3, 8, 4), (28, 64, 4, 8), (32, 1, 8, 8), (2, 4, 2, 4), (3, 6, 1, 3)]:
        plan = ShardPlan(layers, batch, kvh, world)
        allu = torch.cat([plan.local_units(r) for r in range(world)])
        assert sorted(allu.tolist()) == list(range(layers * batch * kvh))
        assert all(len(plan.local_units(r)) == plan.units_per_rank for r in range(world))
    c4 = ShardPlan(28, 64, 4, 8)   # Qwen2.5-7B at 8 GPUs: 4 head groups x 2 batch halves
    assert (c4.head_parts, c4.batch_parts, c4.units_per_rank) == (4, 2, 896)
    with pytest.raises(ValueError):
        heads_of(0, 3, 8)
    with pytest.raises(ValueError):
        ShardPlan(32, 1, 8, 16)    # batch 1 cannot be split


def test_weak_scaling_keeps_units_per_gpu():
    """bench.py's default weak scaling: at N GPUs the batch is N x the config's and every rank
    keeps the N = 1 unit count (KV-head x batch shard); strong scaling splits the N = 1 model."""
    import bench
    for name in ("c2", "c3", "c4"):
        base = bench.CONFIGS[name]
        n1 = base[0] * base[1] * base[2]
        for n in (1, 2, 4, 8):
            cfg, rep = bench.scaled_config(name, n, "weak")
            layers, batch, kvh = cfg[:3]
            assert rep == n and batch == base[1] * n
            plan = ShardPlan(layers, batch, kvh, n)
            assert plan.units_per_rank == n1
            allu = torch.cat([plan.local_units(r) for r in range(n)])
            assert sorted(allu.tolist()) == list(range(n * n1))
            d = bench.decode_config(name, n, cfg, rep)
            assert d["units_per_gpu"] == n1 and d["global_batch"] == base[1] * n
            cfg_s, rep_s = bench.scaled_config(name, n, "strong")
            assert rep_s == 1 and cfg_s == base


def test_assemble_is_the_model_layout():
    for (layers, batch, kvh, world) in [(3, 2, 4, 1), (3, 2, 4, 2), (3, 4, 2, 4), (2, 6, 1, 3)]:
        plan = ShardPlan(layers, batch, kvh, world)
        flat = torch.cat([fake_out(plan.local_units(r)) for r in range(world)])
        assert torch.equal(assemble(flat, plan), reference_layout(layers, batch, kvh))


def test_single_rank_layout():
    assert torch.equal(gather_outputs(fake_out(local_units(LAYERS, BATCH, KVH, 0, 1)), LAYERS, BATCH, KVH, 1),
                       reference_layout())


@pytest.mark.parametrize("world,batch,kvh", [(2, 2, 4), (4, 4, 2)])
def test_gloo_allgather(world, batch, kvh):
    assert _run(_fake_worker, world, LAYERS, batch, kvh) == {r: True for r in range(world)}


# ---------------------------------------------------------------- real decode (GPU)
G_LAYERS, G_BATCH, G_KVH, G_GQ, G_L, G_K, G_SEED = 2, 4, 2, 4, 4096, 256, 55


def _gpu_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2603_14224_b200 import batch as B
        torch.cuda.set_device(0)
        plan = ShardPlan(G_LAYERS, G_BATCH, G_KVH, world)
        cb, qq = bench.build_cache(plan.local_units(rank).tolist(), G_L, G_GQ, G_SEED, torch.device("cuda", 0))
        res = B.decode_step(cb, qq, G_K)
        model = gather_outputs(res.out.cpu(), G_LAYERS, G_BATCH, G_KVH, world)
        q.put((rank, model if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_gloo_sharded_decode_matches_single_process(world):
    import bench
    from paper_2603_14224_b200 import batch as B
    units = G_LAYERS * G_BATCH * G_KVH
    cb, qq = bench.build_cache(range(units), G_L, G_GQ, G_SEED, torch.device("cuda", 0))
    full = B.decode_step(cb, qq, G_K).out.cpu().view(G_LAYERS, G_BATCH, G_KVH * G_GQ, 128)
    got = _run(_gpu_worker, world)[0]
    # same kernel (one CTA per unit) on every shard size here: bit-identical
    assert torch.equal(got, full)
