import os, sys
sys.path.insert(0, "/root/repo")
import torch, bench
from paper_2603_14224_b200 import batch as B, _lib
dev = torch.device("cuda", 0)
cb, q = bench.build_cache(4096, 0, 32768, 4, 1234, dev)
out = torch.empty(4096, 4, 128, device=dev)
for skip in (0, 1):
    _lib.call("sikv_debug_set_ws_skip", skip)
    for _ in range(3): B.decode_step(cb, q, 2048, out=out, kernel=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): B.decode_step(cb, q, 2048, out=out, kernel=1)
    e1.record(); torch.cuda.synchronize()
    print("skip", skip, e0.elapsed_time(e1) / 10, "ms")
