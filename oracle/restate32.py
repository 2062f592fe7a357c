"""float32 restatement of the GPU fast-path scoring arithmetic (TEST INFRASTRUCTURE ONLY).

The fused decode kernel (``paper_2603_14224_b200/csrc/decode.cu``) scores tokens
in float32 with a fixed, stated order so that its top-k set can be checked
exactly.  This module states that order in numpy so tests can reproduce the
kernel's scores bit for bit from the oracle's planes:

1. GQA group-sum query (north_star "per-(batch, KV-head) top-k"):
   ``qbar = ((q_0 + q_1) + q_2) + ...`` in float32.  By linearity of the LUT this is
   ``select_tokens(cache, sum_h q_h, k)`` of the reference (cache.py:290-309).
2. Centroids rounded once to float32 from the float64 codebook (codebook.py:128-160).
3. ``LUT[g][c] = (qbar0*c0 + qbar2*c2) + (qbar1*c1 + qbar3*c3)`` in float32,
   every product rounded, no FMA — the same pairing as the reference's einsum
   (retrieval.py:50).
4. Pair table ``P[p][b] = LUT[2p][b & 15] + LUT[2p+1][b >> 4]`` for the byte
   ``b`` of packed code pair ``p`` (bitpack layout: low nibble = group 2p).
5. Token score = sequential float32 sum of the 16 pair entries starting at pair
   ``r = t mod 16`` and wrapping: ``P[r] + P[r+1] + ... + P[r+15 mod 16]``.
   (The kernel walks the pairs in this rotated order so the 16 lanes of a half
   warp always hit 16 different shared-memory banks.)
6. Top-k over non-forced tokens, descending score, ties -> lower index,
   -0.0 == +0.0 (retrieval.py:127-161).
"""

from __future__ import annotations

import numpy as np

from . import sikv_oracle as O


def group_query(qs: np.ndarray) -> np.ndarray:
    """float32 left-to-right sum over the GQA heads of one KV head."""
    qs = np.asarray(qs, dtype=np.float32)
    acc = qs[0].copy()
    for h in range(1, qs.shape[0]):
        acc = (acc + qs[h]).astype(np.float32)
    return acc


def lut32(qbar: np.ndarray, centroids64: np.ndarray) -> np.ndarray:
    c = centroids64.astype(np.float32)
    G = c.shape[0]
    q = np.asarray(qbar, dtype=np.float32).reshape(G, 1, 4)
    p = (q * c).astype(np.float32)
    return ((p[..., 0] + p[..., 2]) + (p[..., 1] + p[..., 3])).astype(np.float32)


def pair_table(table: np.ndarray) -> np.ndarray:
    """(G/2, 256) float32 pair table."""
    G = table.shape[0]
    b = np.arange(256)
    return (table[0::2][:, b & 15] + table[1::2][:, b >> 4]).astype(np.float32)


def scores32(table: np.ndarray, packed_codes: np.ndarray) -> np.ndarray:
    """Rotated sequential float32 pair sums, one per token."""
    P = pair_table(table)
    npair = P.shape[0]
    L = packed_codes.shape[0]
    t = np.arange(L)
    r = t % npair
    s = P[r, packed_codes[t, r]].astype(np.float32)
    for i in range(1, npair):
        p = (r + i) % npair
        s = (s + P[p, packed_codes[t, p]]).astype(np.float32)
    return s


def select32(cache: O.OracleCache, qs: np.ndarray, k: int):
    """Group-sum fp32 selection on an oracle cache; returns (indices, counts...)."""
    qbar = group_query(qs)
    s = scores32(lut32(qbar, cache.centroids), cache.packed_codes).astype(np.float64)
    s = np.concatenate([s, np.full(len(cache.recent_k), -np.inf)])
    return O.top_k(s, k, sink=cache.sinks, recent=cache.recents())
