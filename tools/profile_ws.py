"""Per-unit phase clocks of the warp-specialised decode kernel (producer vs consumer).

    python tools/profile_ws.py [--units 4096] [--L 32768] [--k 2048] [--gq 4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import _lib  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--units", type=int, default=4096)
ap.add_argument("--L", type=int, default=32768)
ap.add_argument("--k", type=int, default=2048)
ap.add_argument("--gq", type=int, default=4)
ap.add_argument("--kernel", type=int, default=2)
ap.add_argument("--skip", type=int, default=0, help="debug skip bits (1: no attention)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
_lib.call("sikv_debug_set_ws_skip", a.skip)
cb, q = bench.build_cache(range(a.units), a.L, a.gq, 1234, dev)
out = torch.empty(a.units, a.gq, 128, device=dev)
for _ in range(3):
    B.decode_step(cb, q, a.k, out=out, kernel=a.kernel)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    B.decode_step(cb, q, a.k, out=out, kernel=a.kernel)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
gb = bench.algo_bytes_per_unit(a.L, a.k, a.gq) * a.units / 1e9
print(f"units={a.units} L={a.L} k={a.k} gq={a.gq}: {ms:.3f} ms/launch, {gb / ms * 1e3:.1f} GB/s algorithmic")

clk = torch.zeros(a.units, 12, dtype=torch.int64, device=dev)
_lib.call("sikv_debug_set_decode_profile", _lib.ptr(clk))
B.decode_step(cb, q, a.k, out=out, kernel=a.kernel)
torch.cuda.synchronize()
_lib.call("sikv_debug_set_decode_profile", None)
c = clk.cpu().numpy().astype(np.float64)
rows = [("P wait empty", 0, 1), ("P setup+table", 1, 2), ("P score+cand", 2, 3),
        ("C wait full", 4, 5), ("C select", 5, 6), ("C emit", 6, 7), ("C attention", 7, 8), ("C merge", 8, 9)]
pb = (c[:, 3] - c[:, 1]).mean()
cbusy = (c[:, 9] - c[:, 5]).mean()
print(f"producer busy/unit {pb:.0f} cycles, consumer busy/unit {cbusy:.0f} cycles")
for n, i, j in rows:
    ok = (c[:, i] > 0) & (c[:, j] > 0)
    d = c[ok, j] - c[ok, i]
    print(f"  {n:14s} mean {d.mean():9.0f}  p50 {np.median(d):9.0f}  max {d.max():9.0f}  n={ok.sum()}")
