"""Time decode paths 1 / 3 / 4 over unit counts at a fixed geometry (auto-dispatch tuning).
    python tools/dispatch_sweep.py --L 131072 --k 4096 --units 16 32 64 128 256"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=131072)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--gq", type=int, default=4)
ap.add_argument("--units", type=int, nargs="+", default=[16, 32, 64, 128, 256])
ap.add_argument("--kernels", type=int, nargs="+", default=[1, 3, 4])
a = ap.parse_args()
dev = torch.device("cuda", 0)
cb, q = bench.build_cache(range(max(a.units)), a.L, a.gq, 1234, dev)
for U in a.units:
    cb_u, q_u = B.subset(cb, list(range(U))), q[:U].contiguous()
    out = torch.empty(U, a.gq, 128, device=dev)
    row = []
    for kern in a.kernels + [0]:
        try:
            for _ in range(3):
                B.decode_step(cb_u, q_u, a.k, out=out, kernel=kern)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                B.decode_step(cb_u, q_u, a.k, out=out, kernel=kern)
            e1.record()
            torch.cuda.synchronize()
            row.append(f"k{kern if kern else 'auto'} {e0.elapsed_time(e1) / 20:.4f}")
        except Exception as ex:  # noqa: BLE001
            row.append(f"k{kern} n/a")
    print(f"L {a.L} units {U}: " + "  ".join(row), flush=True)
    del cb_u
