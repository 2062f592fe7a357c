import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2603_14224_b200 import batch as B, _lib
cb, q = bench.build_cache(range(256), 131072, 4, 1234, torch.device("cuda", 0))
for kern, cap in [(1, 0), (4, 0), (4, 7000), (4, 8000), (4, 9000)]:
    try:
        r = B.decode_step(cb, q, 4096, with_diag=True, kernel=kern, cap=cap)
        torch.cuda.synchronize()
        d = r.diag.cpu()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        out = torch.empty_like(r.out)
        for _ in range(3): B.decode_step(cb, q, 4096, out=out, kernel=kern, cap=cap)
        e0.record()
        for _ in range(20): B.decode_step(cb, q, 4096, out=out, kernel=kern, cap=cap)
        e1.record(); torch.cuda.synchronize()
        print(kern, cap, "fallbacks", int(((d & 4) != 0).sum()), "ms", e0.elapsed_time(e1) / 20,
              "smem", _lib.lib().sikv_decode_smem_bytes(131072, 4096, 64, 4, cap), flush=True)
    except Exception as ex:
        print(kern, cap, "ERR", ex)
