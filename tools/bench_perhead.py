"""The per-head drop-in API (the reference's own calling convention) timed on the GPU against
the reference's CPU path (the oracle port) on the same unit: prefill, select_tokens +
sparse_attention per query head.  Prints one JSON line per configuration.

    python tools/bench_perhead.py [--tokens 4096 32768] [--queries 16]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_14224_b200 as sk  # noqa: E402
from oracle import sikv_oracle as O  # noqa: E402
from paper_2603_14224_b200.synth import gen_unit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, nargs="+", default=[4096, 32768])
ap.add_argument("--queries", type=int, default=16)
a = ap.parse_args()
for L in a.tokens:
    k = 256 if L <= 4096 else 2048
    u = gen_unit(L, 128, a.queries, 42)
    K = torch.tensor(u.keys, dtype=torch.bfloat16, device="cuda")
    V = torch.tensor(u.values, dtype=torch.bfloat16, device="cuda")
    Q = torch.tensor(u.queries, device="cuda")
    sk.api.set_device_input_checks(False)
    for _ in range(2):
        cache = sk.prefill(K, V)
        [sk.sparse_attention(Q[i], sk.select_tokens(cache, Q[i], k=k), cache) for i in range(a.queries)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cache = sk.prefill(K, V)
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t0
    t0 = time.perf_counter()
    outs = [sk.sparse_attention(Q[i], sk.select_tokens(cache, Q[i], k=k), cache) for i in range(a.queries)]
    torch.cuda.synchronize()
    t_dec = (time.perf_counter() - t0) / a.queries
    t0 = time.perf_counter()
    c = O.prefill(u.keys, u.values)
    c_pre = time.perf_counter() - t0
    t0 = time.perf_counter()
    n_cpu = min(a.queries, 4)
    for i in range(n_cpu):
        O.sparse_attention(u.queries[i], O.select(c, u.queries[i], k=k)[0], c)
    c_dec = (time.perf_counter() - t0) / n_cpu
    err = max(O.rel_l2(outs[i].out.cpu().numpy(), O.sparse_attention(u.queries[i], O.select(c, u.queries[i], k=k)[0], c))
              for i in range(2))
    print(json.dumps({"api": "per-head (float64 kernels, device calling convention)", "tokens": L, "k": k,
                      "gpu_prefill_ms": round(t_pre * 1e3, 3), "gpu_select_attend_ms": round(t_dec * 1e3, 3),
                      "cpu_prefill_ms": round(c_pre * 1e3, 1), "cpu_select_attend_ms": round(c_dec * 1e3, 1),
                      "speedup_decode": round(c_dec / t_dec, 1), "max_rel_l2_vs_cpu": err}), flush=True)
