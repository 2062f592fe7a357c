"""Encoder workload for ncu: n units x L tokens of bf16 K/V."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_14224_b200 import _lib  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402
from paper_2603_14224_b200.synth import gen_units_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--units", type=int, default=8)
ap.add_argument("--L", type=int, default=131072)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cb = B.empty_batch(a.units, a.L, sink_count=64, device=dev)
ws = torch.empty(_lib.lib().sikv_encode_workspace_bytes(a.units, a.L, 128), dtype=torch.uint8, device=dev)
K, V = gen_units_torch(a.units, a.L, 128, 5, dev)
for _ in range(a.iters):
    B.prefill_into(cb, 0, K, V, workspace=ws, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    B.prefill_into(cb, 0, K, V, workspace=ws, check=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
th = a.units * a.L
print(f"encode {a.units}x{a.L}: {ms:.3f} ms, {th / ms / 1e3:.1f} M token-heads/s, {th * 624 / ms / 1e6:.1f} GB/s algorithmic")
