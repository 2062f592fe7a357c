"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck) over every decode
path and feature: kernels 1 / 3 / 4, selection on / off, k = 0 / all, ring appends, window
sinks, sign-only LUT, direct keys, per-q-head policy, the encoder and window-sink kernels.

    compute-sanitizer --tool memcheck python tools/sanitize_decode.py [units L]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402
from paper_2603_14224_b200.synth import gen_units_torch  # noqa: E402

dev = torch.device("cuda", 0)
units = int(sys.argv[1]) if len(sys.argv) > 1 else 300
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cb, q = bench.build_cache(range(units), L, 4, 77, dev)
for kern in (1, 3, 4):
    for k, sel in ((256, True), (256, False), (L, False), (0, False)):
        B.decode_step(cb, q, k, with_selection=sel, with_lse=True, kernel=kern)
        torch.cuda.synchronize()
    B.decode_step(cb, q, 256, with_selection=True, kernel=kern, sign_only=True)
    B.decode_step_per_head(cb, q, 128, with_selection=True, kernel=kern)
    torch.cuda.synchronize()
    print("kernel", kern, "ok", flush=True)
# ring appends (growth) then decode
for _ in range(20):
    B.append_batch(cb, torch.randn(units, 128, device=dev), torch.randn(units, 128, device=dev), check=False)
for kern in (1, 3, 4):
    B.decode_step(cb, q, 256, with_selection=True, kernel=kern)
torch.cuda.synchronize()
print("appends ok", flush=True)
# window sinks + direct keys through the encoder
K, V = gen_units_torch(8, L, 128, 5, dev)
W = torch.randn(8, 32, 128, device=dev)
cbw = B.prefill_batch(K, V, sink_count=64, window=W, sign_in_quant=False, bits=1)
qw = torch.randn(8, 4, 128, device=dev)
for kern in (1, 3, 4):
    B.decode_step(cbw, qw, 200, with_selection=True, kernel=kern)
torch.cuda.synchronize()
print("window sinks / direct / 1-bit ok", flush=True)
# 16-bit records (two-kernel path, split attention at 8 units)
cb16 = B.prefill_batch(K, V, sink_count=64, bits=16)
B.decode_step(cb16, qw, 200, with_selection=True, kernel=4)
torch.cuda.synchronize()
print("16-bit records ok", flush=True)
# 4- / 8-bit codes: reference-layout planes + sign-plane pass + dequantise / pack16
for b, siq in ((4, True), (8, False)):
    cbw4 = B.prefill_batch(K, V, sink_count=64, bits=b, sign_in_quant=siq, keep_reference=(b == 4))
    B.decode_step(cbw4, qw, 200, with_selection=True, kernel=4)
torch.cuda.synchronize()
print("4 / 8-bit codes ok", flush=True)
# a long unit: extra sample passes (>= 64K tokens) on the two-kernel path, split attention
cbl, ql = bench.build_cache(range(8), 65536, 4, 78, dev)
B.decode_step(cbl, ql, 2048, with_selection=True, kernel=4)
torch.cuda.synchronize()
print("long units ok", flush=True)
