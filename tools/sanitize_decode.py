"""Small decode workloads for compute-sanitizer (memcheck / racecheck) over every path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402

dev = torch.device("cuda", 0)
units = int(sys.argv[1]) if len(sys.argv) > 1 else 300
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
kernels = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4]
cb, q = bench.build_cache(range(units), L, 4, 77, dev)
for kern in kernels:
    for k, sel in ((256, True), (256, False), (L, False), (0, False)):
        r = B.decode_step(cb, q, k, with_selection=sel, with_lse=True, kernel=kern)
        torch.cuda.synchronize()
    print("kernel", kern, "ok")
