"""The multi-GPU output all-gather fused into the decode step (shard.OutputExchange,
sikv_decode_step_x): every rank's attention epilogue stores its units' rows as bf16 into every
rank's model-layout buffer and releases them on every rank's arrival counter.

On one GPU:
  * an in-process world of 2 / 4 / 8 ranks (each rank's exchange shares the others'
    buffers), every decode path (two-kernel epilogue; one-CTA and cluster-split paths via the
    push kernel), both GQA policies, two consecutive steps: every rank's buffer equals the
    bf16 model-layout output of the single-process run, and every counter holds exactly the
    arrivals of the steps;
  * two processes on cuda:0 with CUDA IPC peer mappings (the real multi-GPU code path; gloo
    exchanges the handles).
"""
import os
import socket

import pytest
import torch

import bench
from paper_2603_14224_b200 import _lib
from paper_2603_14224_b200 import batch as B
from paper_2603_14224_b200.shard import OutputExchange, ShardPlan

pytestmark = pytest.mark.gpu

LAYERS, BATCH, KVH, GQ, L, K, SEED = 2, 4, 2, 4, 4096, 256, 77


def _full(per_head=False, kernel=0):
    dev = torch.device("cuda", 0)
    cb, q = bench.build_cache(range(LAYERS * BATCH * KVH), L, GQ, SEED, dev)
    dec = B.decode_step_per_head if per_head else B.decode_step
    return cb, q, dec(cb, q, K, kernel=kernel).out


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("kernel", [4, 1, 3])
def test_inprocess_world(world, kernel):
    cb, q, full = _full(kernel=kernel)
    plan = ShardPlan(LAYERS, BATCH, KVH, world)
    ranks = []
    for r in range(world):
        ranks.append(OutputExchange(plan, GQ, r, "cuda:0", ranks=list(ranks)))
    shards = []
    for r in range(world):
        ids = plan.local_units(r).to("cuda")
        shards.append((B.subset(cb, ids), q.index_select(0, ids)))
    for step in range(2):
        expect = torch.empty_like(full)
        for r in range(world):
            sub, qr = shards[r]
            res = B.decode_step(sub, qr, K, kernel=kernel, exchange=ranks[r])
            assert _lib.lib().sikv_decode_last_kernel() == kernel
            expect[plan.local_units(r).to("cuda")] = res.out
        views = [x.wait() for x in ranks]
        torch.cuda.synchronize()
        ref = expect.to(torch.bfloat16).view(LAYERS, BATCH, KVH * GQ, 128)
        for r in range(world):
            assert torch.equal(views[r], ref), (world, kernel, step, r)
            assert int(ranks[r].counter.item()) == (step + 1) * LAYERS * BATCH * KVH * GQ
        # and the shards' outputs are the full run's (up to the split-merge order of the path)
        err = ((expect - full).norm(dim=-1) / full.norm(dim=-1)).max().item()
        assert err <= 1e-3


def test_inprocess_world_per_head_policy():
    cb, q, full = _full(per_head=True, kernel=4)
    world = 2
    plan = ShardPlan(LAYERS, BATCH, KVH, world)
    ranks = []
    for r in range(world):
        ranks.append(OutputExchange(plan, GQ, r, "cuda:0", ranks=list(ranks)))
    expect = torch.empty_like(full)
    for r in range(world):
        ids = plan.local_units(r).to("cuda")
        res = B.decode_step_per_head(B.subset(cb, ids), q.index_select(0, ids), K, kernel=4, exchange=ranks[r])
        expect[ids] = res.out
    views = [x.wait() for x in ranks]
    torch.cuda.synchronize()
    ref = expect.to(torch.bfloat16).view(LAYERS, BATCH, KVH * GQ, 128)
    for v in views:
        assert torch.equal(v, ref)


def test_exchange_validation():
    cb, q, _ = _full()
    plan = ShardPlan(LAYERS, BATCH, KVH, 1)
    x = OutputExchange(plan, GQ, 0, "cuda:0")
    with pytest.raises(ValueError, match="exchange built for"):
        x.cstruct(3, GQ)
    bad = _lib.Exchange()
    bad.npeers = 9

    class Bad:
        def cstruct(self, units, gq):
            return bad

    with pytest.raises(ValueError, match="npeers"):
        B.decode_step(cb, q, K, exchange=Bad())
    with pytest.raises(ValueError, match="null counter"):
        _lib.call("sikv_exchange_wait", None, 0, None)
    # world 1: the exchange is the model-layout copy of the step's outputs
    res = B.decode_step(cb, q, K, exchange=x)
    view = x.wait()
    torch.cuda.synchronize()
    assert torch.equal(view, res.out.to(torch.bfloat16).view(LAYERS, BATCH, KVH * GQ, 128))


# ---------------------------------------------------------------- two processes, CUDA IPC
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench as bn
        from paper_2603_14224_b200 import batch as Bb
        from paper_2603_14224_b200.shard import OutputExchange as OX
        from paper_2603_14224_b200.shard import ShardPlan as SP
        torch.cuda.set_device(0)
        plan = SP(LAYERS, BATCH, KVH, world)
        cb, qq = bn.build_cache(plan.local_units(rank).tolist(), L, GQ, SEED, torch.device("cuda", 0))
        x = OX(plan, GQ, rank, "cuda:0")
        for _ in range(2):
            res = Bb.decode_step(cb, qq, K, kernel=4, exchange=x)
            view = x.wait()
        torch.cuda.synchronize()
        q.put((rank, (view.cpu(), int(x.counter.item()), res.out.cpu(), plan.local_units(rank))))
        dist.barrier()                 # peers stop touching this rank's buffer before it is freed
        x.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc():
    import torch.multiprocessing as mp
    _, _, full = _full(kernel=4)
    ref = full.to(torch.bfloat16).view(LAYERS, BATCH, KVH * GQ, 128).cpu()
    world = 2
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, qu)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(qu.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    expect = torch.empty(LAYERS * BATCH * KVH, GQ, 128)
    for r in range(world):
        expect[res[r][3]] = res[r][2]
    expect = expect.to(torch.bfloat16).view(LAYERS, BATCH, KVH * GQ, 128)
    for r in range(world):
        view, cnt = res[r][0], res[r][1]
        assert torch.equal(view, expect), r
        assert cnt == 2 * LAYERS * BATCH * KVH * GQ
    err = ((expect.float() - ref.float()).norm(dim=-1) / ref.float().norm(dim=-1)).max().item()
    assert err <= 1e-2          # bf16 of the shards' outputs vs bf16 of the full run's


def test_bench_two_ranks_on_one_gpu():
    """bench.py --gpus 2 end to end (its own torchrun launch, the IPC exchange, the e2e
    loop, the JSON line), both ranks on cuda:0 (SIKV_BENCH_SHARE_GPU: gloo for the host-side
    collectives; the timings are not meaningful)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SIKV_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", "c1",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, env=env, timeout=600,
                       cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["output_gather"].startswith("fused")
    assert line["gpu_launches"] == 3 * 3      # per step: the decode kernel(s) + push (path 1) or not (path 4) + wait
