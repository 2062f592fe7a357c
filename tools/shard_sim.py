"""Per-GPU decode time of the head-sharded step at N = 1, 2, 4, 8 GPUs, simulated on one GPU
(each rank decodes its ShardPlan share of the units on its auto path; the all-gather is not
included).   python tools/shard_sim.py [c2 c4 c3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import _lib  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402

dev = torch.device("cuda", 0)
KERNEL = int(os.environ.get("KERNEL", "0"))
for cfg in sys.argv[1:] or ["c2"]:
  layers, batch, kvh, gq, L, k, _ = bench.CONFIGS[cfg]
  units = layers * batch * kvh
  base = None
  for n in (1, 2, 4, 8):
      ul = units // n
      cb, q = bench.build_cache(range(ul), L, gq, 1234, dev)
      out = torch.empty(ul, gq, 128, device=dev)
      for _ in range(5):
          B.decode_step(cb, q, k, out=out, kernel=KERNEL)
      torch.cuda.synchronize()
      e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
      e0.record()
      for _ in range(50):
          B.decode_step(cb, q, k, out=out, kernel=KERNEL)
      e1.record()
      torch.cuda.synchronize()
      ms = e0.elapsed_time(e1) / 50
      base = base or ms
      print(f"{cfg} N={n}: {ul} units/GPU  {ms:.4f} ms  path {_lib.lib().sikv_decode_last_kernel()}  "
            f"speed-up {base / ms:.2f}x  efficiency {base / ms / n:.2f}")
      del cb, q, out
      torch.cuda.empty_cache()
