"""Generate golden vectors by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports ``sikv`` from ``/root/reference/pkg/src`` (read-only, never copied),
feeds it bf16-rounded synthetic inputs (regenerable from the seed anywhere via
``paper_2603_14224_b200.synth.gen_unit``) and records its outputs:

* SHA-256 of every encoder plane (sign codes, payloads, fp16 scales / zeros),
  of the generated inputs and of the float64 score vector;
* the small float arrays (mu, alpha, centroids, LUT) and the selections /
  attention outputs in full.

The oracle (``oracle/sikv_oracle.py``) is pinned against this file by
``tests/test_oracle_golden.py``; the GPU tests then compare against the oracle.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import sikv  # noqa: E402  (the reference)
from sikv.harness.synth import gen_synthetic  # noqa: E402

from paper_2603_14224_b200.synth import bf16_round, gen_unit  # noqa: E402

# (name, tokens, dim, seed, bits, group, sinks, sign_in_quant, window, k, gq, appends)
CASES = [
    ("c1_u0", 4096, 128, 100, 2, 32, 64, True, False, 256, 4, 0),
    ("c1_u1", 4096, 128, 101, 2, 32, 64, True, False, 256, 4, 0),
    ("c1_u2", 4096, 128, 102, 2, 32, 64, True, False, 256, 4, 0),
    ("c1_u3", 4096, 128, 103, 2, 32, 64, True, False, 256, 4, 0),
    ("win_1k", 1024, 128, 7, 2, 32, 64, True, True, 96, 4, 0),
    ("append_2k", 2048, 128, 11, 2, 32, 64, True, False, 128, 4, 3),
    ("gq7_2k", 2048, 128, 12, 2, 32, 64, True, False, 200, 7, 0),
    ("b4_d64", 600, 64, 5, 4, 32, 16, True, False, 40, 2, 0),
    ("direct_d32", 300, 32, 6, 2, 16, 8, False, False, 30, 2, 0),
    ("b8_d32", 257, 32, 8, 8, 32, 4, True, False, 20, 1, 0),
    ("b1_d128", 512, 128, 9, 1, 32, 0, True, False, 64, 4, 0),
    ("lossless_d64", 256, 64, 10, 16, 32, 8, True, False, 32, 2, 0),
    ("c2_1unit", 32768, 128, 200, 2, 32, 64, True, False, 2048, 4, 0),
    # the fast path's variants at its geometry (D = 128, group 32)
    ("direct_d128", 2048, 128, 13, 2, 32, 64, False, False, 128, 4, 0),
    ("b1_sinks_d128", 2048, 128, 14, 1, 32, 64, True, False, 128, 4, 0),
    ("lossless_d128", 2048, 128, 15, 16, 32, 64, True, False, 128, 4, 0),
]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    out = {}
    arrays = {}
    for (name, L, D, seed, bits, group, sinks, siq, win, k, gq, appends) in CASES:
        nq = gq + appends
        mine = gen_unit(L, D, nq, seed)
        ref = gen_synthetic(L, D, nq, seed)
        # the reference generator and ours must draw identical numbers
        assert np.array_equal(bf16_round(ref.keys), mine.keys), name
        assert np.array_equal(bf16_round(ref.queries), mine.queries), name
        K, V, Q, W = mine.keys, mine.values, mine.queries, mine.window
        cfg = sikv.CacheConfig(bits=bits, group_size=group, sink_count=sinks, sign_in_quant=siq)
        cache = sikv.prefill(K, V, W if win else None, cfg)
        rec = dict(L=L, D=D, seed=seed, bits=bits, group=group, sinks=sinks, sign_in_quant=siq,
                   window=win, k=k, gq=gq, appends=appends,
                   inputs_sha=sha(np.stack([K.sum(0), V.sum(0)])) + sha(K) + sha(V),
                   codes_sha=sha(cache.codes.packed))
        planes = {}
        for tag, qt in (("kmag", cache.key_mag), ("kdirect", cache.key_direct),
                        ("values", cache.values)):
            if qt is not None:
                planes[tag] = dict(packed=sha(qt.packed), scales=sha(qt.scales), zeros=sha(qt.zeros))
        rec["planes"] = planes
        rec["sink_indices"] = cache.sink_indices.tolist()
        # decode-time appends use the queries after the first gq as new keys/values
        for a in range(appends):
            sikv.append_token(cache, Q[gq + a] * 0.5, Q[gq + a][::-1].copy())
        qh = Q[:gq]
        qbar = qh.sum(axis=0)
        lut = sikv.build_lut(qbar, cache.codebook)
        scores = sikv.score_tokens(lut, cache.codes)
        rec["scores_sha"] = sha(scores)
        sel = sikv.select_tokens(cache, qbar, k=k)
        rec["sel_counts"] = [sel.sink_count, sel.recent_count, sel.dynamic_count]
        outs = np.stack([sikv.sparse_attention(q, sel, cache).out for q in qh])
        per_head = [sikv.select_tokens(cache, q, k=k).indices.tolist() for q in qh]
        rec["per_head_sel"] = per_head
        if cache.config.lossless is False:
            budget_sel = sikv.select_tokens(cache, qbar, budget=k + 10)
            spars_sel = sikv.select_tokens(cache, qbar, sparsity=0.05, sign_only=True)
            rec["budget_sel"] = budget_sel.indices.tolist()
            rec["sparsity_signonly_sel"] = spars_sel.indices.tolist()
        rec["memory"] = sikv.memory_report(cache).total_bits
        rec["checksum"] = cache.checksum()
        out[name] = rec
        arrays[f"{name}/mu"] = cache.norm.mu
        arrays[f"{name}/alpha"] = cache.norm.alpha
        arrays[f"{name}/centroids"] = cache.codebook.centroids
        arrays[f"{name}/lut"] = lut.table
        arrays[f"{name}/sel"] = sel.indices
        arrays[f"{name}/attn"] = outs
        print(name, "done", flush=True)

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden_arrays.npz"), **arrays)


if __name__ == "__main__":
    main()
