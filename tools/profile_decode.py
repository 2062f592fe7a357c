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
ap.add_argument("--kernel", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cb, q = bench.build_cache(range(a.units), a.L, a.gq, 1234, dev)
out = torch.empty(a.units, a.gq, 128, device=dev)
for _ in range(a.iters):
    B.decode_step(cb, q, a.k, out=out, kernel=a.kernel)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    B.decode_step(cb, q, a.k, out=out, kernel=a.kernel)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
gb = bench.algo_bytes_per_unit(a.L, a.k, a.gq) * a.units / 1e9
print(f"units={a.units} L={a.L} k={a.k}: {ms:.3f} ms/launch, {gb / ms * 1e3:.1f} GB/s algorithmic")

if True:
    from paper_2603_14224_b200 import _lib
    clk = torch.zeros(a.units, 12, dtype=torch.int64, device=dev)
    _lib.call("sikv_debug_set_decode_profile", _lib.ptr(clk))
    B.decode_step(cb, q, a.k, out=out, kernel=a.kernel)
    torch.cuda.synchronize()
    _lib.call("sikv_debug_set_decode_profile", None)
    c = clk.cpu().numpy().astype("float64")
    names = ["setup", "B1+tau", "B2 score", "C select", "scan", "forced attn", "dyn attn", "wait merge", "merge"]
    pts = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9]
    tot = (c[:, 9] - c[:, 0]).mean()
    print(f"mean unit cycles {tot:.0f}")
    for i, n in enumerate(names):
        d = c[:, pts[i + 1]] - c[:, pts[i]]
        ok = (c[:, pts[i + 1]] > 0) & (c[:, pts[i]] > 0)
        print(f"  {n:12s} {d[ok].mean():10.0f} cycles ({100 * d[ok].mean() / tot:5.1f}%)  n={ok.sum()}")
