"""Small decode workload for ncu: U units at C2 geometry, a few launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--units", type=int, default=592)
ap.add_argument("--L", type=int, default=32768)
ap.add_argument("--k", type=int, default=2048)
ap.add_argument("--gq", type=int, default=4)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cb, q = bench.build_cache(a.units, 0, a.L, a.gq, 1234, dev)
out = torch.empty(a.units, a.gq, 128, device=dev)
for _ in range(a.iters):
    B.decode_step(cb, q, a.k, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    B.decode_step(cb, q, a.k, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
gb = bench.algo_bytes_per_unit(a.L, a.k, a.gq) * a.units / 1e9
print(f"units={a.units} L={a.L} k={a.k}: {ms:.3f} ms/launch, {gb / ms * 1e3:.1f} GB/s algorithmic")
