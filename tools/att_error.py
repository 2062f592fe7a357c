"""Measured attention error of the fused decode path against the float64 oracle on the same
selection, per configuration and decode kernel (max rel-L2, min cosine over units x heads).
Writes profiles/<round>/attention_error.json; the tests' tolerances are set from it.

    python tools/att_error.py [--out profiles/round2/attention_error.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import restate32 as R  # noqa: E402
from oracle import sikv_oracle as O  # noqa: E402
from paper_2603_14224_b200 import batch as B  # noqa: E402
from paper_2603_14224_b200.synth import gen_unit  # noqa: E402

CASES = [  # name, L, k, gq, kernels, units, bits, sign_in_quant
    ("c1 (4K, k 256, Gq 4)", 4096, 256, 4, (1, 3, 4), 8, 2, True),
    ("c2 geometry (32K, k 2048, Gq 4)", 32768, 2048, 4, (1, 3, 4), 6, 2, True),
    ("c4 geometry (8K, k 1024, Gq 7)", 8192, 1024, 7, (1, 3, 4), 8, 2, True),
    ("c3 geometry (128K, k 4096, Gq 4)", 131072, 4096, 4, (1, 3), 2, 2, True),
    ("direct keys 4K", 4096, 256, 4, (1, 4), 8, 2, False),
    ("direct keys 32K", 32768, 2048, 4, (1, 3, 4), 6, 2, False),
    ("1-bit 4K", 4096, 256, 4, (1, 4), 8, 1, True),
    ("1-bit 32K", 32768, 2048, 4, (1, 4), 4, 1, True),
    ("1-bit direct 32K", 32768, 2048, 4, (1, 4), 4, 1, False),
]
ap = argparse.ArgumentParser()
ap.add_argument("--out", default="profiles/round2/attention_error.json")
ap.add_argument("--variants-only", action="store_true")
a = ap.parse_args()
res = []
only = os.environ.get("ATT_ONLY")
for name, L, k, gq, kernels, n, bits, siq in CASES:
    if only and only not in name:
        continue
    units = [gen_unit(L, 128, gq, 5000 + i) for i in range(n)]
    K = torch.tensor(np.stack([u.keys for u in units]), dtype=torch.bfloat16, device="cuda")
    V = torch.tensor(np.stack([u.values for u in units]), dtype=torch.bfloat16, device="cuda")
    cb = B.prefill_batch(K, V, sink_count=64, bits=bits, sign_in_quant=siq)
    oc = [O.prefill(u.keys, u.values, sink_count=64, bits=bits, sign_in_quant=siq) for u in units]
    q = torch.tensor(np.stack([u.queries[:gq] for u in units]), dtype=torch.float32, device="cuda")
    for kern in kernels:
        r = B.decode_step(cb, q, k, with_selection=True, kernel=kern)
        out = r.out.cpu().numpy()
        rels, coss = [], []
        for i, c in enumerate(oc):
            idx = R.select32(c, u.queries[:gq].astype(np.float32) if False else q[i].cpu().numpy(), k)[0]
            assert np.array_equal(r.selection[i, : int(r.counts[i])].cpu().numpy(), idx)
            for h in range(gq):
                ref = O.sparse_attention(q[i, h].cpu().numpy().astype(np.float64), idx, c)
                rels.append(O.rel_l2(out[i, h], ref))
                coss.append(O.cosine(out[i, h], ref))
        rec = {"config": name, "bits": bits, "sign_in_quant": siq, "kernel": kern, "units": n, "heads": n * gq, "max_rel_l2": max(rels),
               "mean_rel_l2": float(np.mean(rels)), "min_cosine": min(coss)}
        print(json.dumps(rec), flush=True)
        res.append(rec)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    json.dump({"what": "fused decode attention vs float64 oracle on the same selection "
                       "(fp16 mma operands, fp32 accumulation, fp32 output)", "cases": res}, f, indent=1)
