"""Drive the per-head float64 kernels (lut / score / top-k / attend) on small inputs for
compute-sanitizer:  compute-sanitizer --tool racecheck python tools/sanitize_perhead.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_14224_b200 as sk  # noqa: E402
from paper_2603_14224_b200.synth import gen_unit  # noqa: E402

rng = np.random.default_rng(3)
for L in (100, 5000):
    for s in (rng.standard_normal(L), np.round(rng.standard_normal(L))):
        for k in (1, 40, L // 2):
            sk.top_k_select(s, k, sink=set(range(8)), recent=set(range(L - 4, L)))
for L, k in ((1024, 64), (4096, 256)):
    u = gen_unit(L, 128, 2, 9)
    cache = sk.prefill(torch.tensor(u.keys, dtype=torch.bfloat16, device="cuda"),
                       torch.tensor(u.values, dtype=torch.bfloat16, device="cuda"))
    for h in range(2):
        q = torch.tensor(u.queries[h], device="cuda")
        sk.sparse_attention(q, sk.select_tokens(cache, q, k=k), cache)
torch.cuda.synchronize()
print("per-head kernels ok")
