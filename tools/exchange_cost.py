"""Cost of the fused output exchange on one GPU: rank 0 of an N-rank shard of a config
decodes its units with and without the exchange epilogue storing to N peer buffers (all on
this GPU, so the stores go to local HBM instead of NVLink; the other ranks stay passive).

    python tools/exchange_cost.py [c2 8 [peers]] [--weak]

--weak: the bench's default weak scaling (batch x N, every GPU keeps the N = 1 unit count,
so each rank stores N times the N = 1 output volume).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402
from paper_2603_14224_b200.shard import OutputExchange, ShardPlan  # noqa: E402

weak = "--weak" in sys.argv
sys.argv = [a for a in sys.argv if a != "--weak"]
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
npeer = int(sys.argv[3]) if len(sys.argv) > 3 else world     # peers rank 0 stores to
layers, batch, kvh, gq, L, k, _ = bench.scaled_config(cfg, world, "weak" if weak else "strong")[0]
plan = ShardPlan(layers, batch, kvh, world)
dev = torch.device("cuda", 0)
cb, q = bench.build_cache(plan.local_units(0).tolist(), L, gq, 1234, dev)
out = torch.empty(plan.units_per_rank, gq, 128, device=dev)
ranks = []
for r in range(npeer):
    ranks.append(OutputExchange(plan, gq, r, dev, ranks=list(ranks)))
x0 = ranks[0]


def timed(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for rnd in range(2):
    t0 = timed(lambda: B.decode_step(cb, q, k, out=out))
    t1 = timed(lambda: B.decode_step(cb, q, k, out=out, exchange=x0))
    print(f"{cfg}{' weak' if weak else ''} rank 0 of {world} ({plan.units_per_rank} units): decode {t0:.4f} ms, with the fused exchange "
          f"to {npeer} buffers {t1:.4f} ms (+{(t1 - t0) * 1e3:.1f} us)", flush=True)
