"""Time the decode kernels (1 = one CTA per unit, 3 = cluster split, 4 = two kernels)
on the bench configurations; prints ms per launch and algorithmic GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402

dev = torch.device("cuda", 0)
NIT = int(os.environ.get("NIT", "30"))
CAP = int(os.environ.get("CAP", "0"))   # candidate buffer entries (0 = the library's choice)
ONLY = [int(x) for x in os.environ["KERNELS"].split(",")] if "KERNELS" in os.environ else None
cfgs = sys.argv[1:] or ["c2", "c3", "c4"]
for name in cfgs:
    layers, batch, kvh, gq, L, k, _ = bench.CONFIGS[name]
    units = layers * batch * kvh
    cb, q = bench.build_cache(range(units), L, gq, 1234, dev)
    out = torch.empty(units, gq, 128, device=dev)
    for kern in ONLY or ([1, 3, 4] if units < 1000 else [1, 4]):
        try:
            for _ in range(3):
                B.decode_step(cb, q, k, out=out, kernel=kern, cap=CAP)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(NIT):
                B.decode_step(cb, q, k, out=out, kernel=kern, cap=CAP)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / NIT
            gb = bench.algo_bytes_per_unit(L, k, gq) * units / 1e9
            print(f"{name} kernel {kern} cap {CAP}: {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")
        except Exception as ex:  # noqa: BLE001
            print(f"{name} kernel {kern}: {ex}")
    del cb, q, out
    torch.cuda.empty_cache()
