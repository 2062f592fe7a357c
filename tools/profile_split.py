"""Per-unit phase clocks of decode_split_kernel (cluster rank 0): setup, scan (+ threshold),
cluster-wide k-th, ties / emission, attention, merge.
    python tools/profile_split.py [--units 32 --L 131072 --k 4096]"""
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
ap.add_argument("--units", type=int, default=32)
ap.add_argument("--L", type=int, default=131072)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--gq", type=int, default=4)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cb, q = bench.build_cache(range(a.units), a.L, a.gq, 1234, dev)
out = torch.empty(a.units, a.gq, 128, device=dev)
for _ in range(3):
    B.decode_step(cb, q, a.k, out=out, kernel=3)
clk = torch.zeros(a.units, 16, dtype=torch.int64, device=dev)
_lib.call("sikv_debug_set_decode_profile", _lib.ptr(clk))
B.decode_step(cb, q, a.k, out=out, kernel=3)
torch.cuda.synchronize()
_lib.call("sikv_debug_set_decode_profile", None)
c = clk.cpu().numpy().astype(np.float64)
for n, i, j in [("setup", 0, 1), ("sample+tau+scan", 1, 2), ("cluster k-th", 2, 3), ("ties+emit", 3, 4),
                ("attention", 4, 5), ("merge", 5, 6), ("total", 0, 6)]:
    d = c[:, j] - c[:, i]
    print(f"  {n:16s} mean {d.mean():9.0f}  max {d.max():9.0f}")
