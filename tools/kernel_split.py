"""Per-kernel device time of the two-kernel decode path at a given unit count (C2 shape):
  python tools/kernel_split.py --units 512
The selection and attention kernels are timed on the launching stream with CUDA events."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--units", type=int, nargs="+", default=[512, 4096])
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--kernels", type=int, nargs="+", default=[4])
a = ap.parse_args()
dev = torch.device("cuda", 0)
for units in a.units:
    cb, q = bench.build_cache(range(units), 32768, 4, 1234, dev)
    out = torch.empty(units, 4, 128, device=dev)
    for kern in a.kernels:
        for _ in range(5):
            B.decode_step(cb, q, 2048, out=out, kernel=kern)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            B.decode_step(cb, q, 2048, out=out, kernel=kern)
        e1.record()
        torch.cuda.synchronize()
        res = B.decode_step(cb, q, 2048, kernel=kern, with_selection=True)
        torch.cuda.synchronize()
        same = ""
        if kern != a.kernels[0]:
            same = (f" out==k{a.kernels[0]}: {bool(torch.equal(res.out, ref.out))}"
                    f" sel==: {bool(torch.equal(res.selection, ref.selection))}")
        else:
            ref = res
        print(f"units {units} kernel {kern}: step {e0.elapsed_time(e1) / a.iters:.4f} ms{same}")
    del cb, q, out
    torch.cuda.empty_cache()
