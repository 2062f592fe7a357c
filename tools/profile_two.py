"""Per-unit phase clocks of decode_select_kernel (two-kernel path): setup, scoring +
candidates, selection + emission.   python tools/profile_two.py [--units 4096 --L 32768 --k 2048]"""
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
ap.add_argument("--cap", type=int, default=0)
ap.add_argument("--kernel", type=int, default=4)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cb, q = bench.build_cache(range(a.units), a.L, a.gq, 1234, dev)
out = torch.empty(a.units, a.gq, 128, device=dev)
for _ in range(3):
    B.decode_step(cb, q, a.k, out=out, kernel=a.kernel, cap=a.cap)
clk = torch.zeros(a.units, 16, dtype=torch.int64, device=dev)
_lib.call("sikv_debug_set_decode_profile", _lib.ptr(clk))
B.decode_step(cb, q, a.k, out=out, kernel=a.kernel, cap=a.cap)
torch.cuda.synchronize()
_lib.call("sikv_debug_set_decode_profile", None)
c = clk.cpu().numpy().astype(np.float64)
d = c[:, 2] - c[:, 1]
print("  score+cand deciles", np.percentile(d, [10, 50, 80, 90, 95, 99, 100]).astype(int).tolist())
grid = min(148, (a.units + 1) // 2)
grp = (np.arange(a.units) // grid) % 2
rows = [("wait inputs", 0, 4), ("bitmap+qbar+LUT", 4, 5), ("pair table", 5, 1), ("sample score", 1, 7),
                ("tau", 7, 8), ("scan (after tau)", 8, 2), ("setup+table", 0, 1), ("score+cand", 1, 2),
                ("select+emit", 2, 3), ("  k-th", 2, 12), ("  emit", 12, 13), ("  bitmaps/sel", 13, 3),
                ("unit total", 0, 3)]
for n, i, j in rows:
    d = c[:, j] - c[:, i]
    g0, g1 = d[grp == 0].mean(), d[grp == 1].mean()
    print(f"  {n:16s} mean {d.mean():9.0f}  p50 {np.median(d):9.0f}  max {d.max():9.0f}   group0 {g0:9.0f} group1 {g1:9.0f}")
att = clk.cpu().numpy()[:, 9]
print("  scan attempts (0 = first scan sufficed):", {int(v): int((att == v).sum()) for v in np.unique(att)})
tot, mw = clk.cpu().numpy()[:, 10], clk.cpu().numpy()[:, 11]
print(f"  candidates per unit: mean {tot.mean():.0f} min {tot.min()} max {tot.max()}; max per-warp segment {mw.max()}")
