"""One per-head drop-in decode (the reference's calling convention: select_tokens +
sparse_attention on one 32K-token head) for an ncu capture of the per-head kernels.
    ncu --set full -o perhead python tools/profile_perhead.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_14224_b200 as sk  # noqa: E402
from paper_2603_14224_b200.synth import gen_unit  # noqa: E402

L, k = 32768, 2048
u = gen_unit(L, 128, 2, 42)
K = torch.tensor(u.keys, dtype=torch.bfloat16, device="cuda")
V = torch.tensor(u.values, dtype=torch.bfloat16, device="cuda")
Q = torch.tensor(u.queries, device="cuda")
sk.api.set_device_input_checks(False)
cache = sk.prefill(K, V)
for i in range(2):
    sk.sparse_attention(Q[i], sk.select_tokens(cache, Q[i], k=k), cache)
torch.cuda.synchronize()
print("ok")
