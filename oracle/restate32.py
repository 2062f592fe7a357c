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


def sign_lut32(qbar: np.ndarray, groups: int) -> np.ndarray:
    """Sign-only LUT (build_sign_lut, retrieval.py:54-62) in the same float32 pairing as
    lut32, with the code's +-1 pattern (element i <-> bit 3 - i) in place of the centroid:
    the products are exact, ``(s0 q0 + s2 q2) + (s1 q1 + s3 q3)``."""
    pat = (((np.arange(16)[:, None] >> O._SH) & 1) * 2 - 1).astype(np.float32)   # (16, 4)
    q = np.asarray(qbar, dtype=np.float32).reshape(groups, 1, 4)
    p = (q * pat[None]).astype(np.float32)
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


def select32(cache: O.OracleCache, qs: np.ndarray, k: int, sign_only: bool = False):
    """Group-sum fp32 selection on an oracle cache; returns (indices, counts...)."""
    qbar = group_query(qs)
    table = sign_lut32(qbar, cache.centroids.shape[0]) if sign_only else lut32(qbar, cache.centroids)
    s = scores32(table, cache.packed_codes).astype(np.float64)
    s = np.concatenate([s, np.full(len(cache.recent_k), -np.inf)])
    return O.top_k(s, k, sink=cache.sinks, recent=cache.recents())


# --------------------------------------------------------------------------- certified bound
U32 = 2.0 ** -24
U64 = 2.0 ** -53


def _gamma(n: int, u: float) -> float:
    return n * u / (1.0 - n * u)


def score_error_bound(cache: O.OracleCache, qs: np.ndarray, sign_only: bool = False) -> float:
    """A bound B with |scores32(t) - s64(t)| <= B for every prefill token t, where s64 is the
    reference's float64 score of the group-sum query (select_tokens(cache, sum_h q_h),
    cache.py:290-309) and scores32 the fast path's float32 order above.

    Standard forward error analysis (Higham, ch. 3), per group g and code c:
      qbar:   |fl32(sum_h q_h) - sum_h q_h| <= gamma_{Gq-1} sum_h |q_h|          (per channel)
      LUT:    fl32 centroids (1 rounding), 4 products + 3 adds -> gamma_4 relative on
              sum_i |qbar_i c_i|, plus the qbar error times |c|;
      pairs:  one add (u |P|);  score: 15 sequential adds, gamma_15 on sum_p |P_p|;
      and the reference's own float64 rounding (gamma_40 in double on the same sums).
    The bound is uniform over tokens: every term is maximised over the 16 codes of a group."""
    qs = np.asarray(qs, dtype=np.float64)
    gq = qs.shape[0]
    qbar = group_query(qs).astype(np.float64)
    dq = _gamma(max(gq - 1, 0), U32) * np.abs(qs).sum(axis=0)           # per channel
    c = np.ones_like(cache.centroids) if sign_only else np.abs(cache.centroids)   # (G, 16, 4)
    G = c.shape[0]
    qa = np.abs(qbar).reshape(G, 1, 4)
    dqa = dq.reshape(G, 1, 4)
    e_lut = ((dqa + (_gamma(4, U32) + U32) * qa) * c * (1 + U32)).sum(axis=2)   # (G, 16)
    mag = (qa * c).sum(axis=2) * (1 + _gamma(5, U32))                   # |LUT| bound
    e_lut_max = e_lut.max(axis=1)
    mag_max = mag.max(axis=1)
    pair_mag = mag_max[0::2] + mag_max[1::2]
    B = e_lut_max.sum() + U32 * pair_mag.sum() + _gamma(15, U32) * pair_mag.sum() * (1 + U32)
    B += _gamma(40, U64) * (np.abs(qs).sum(axis=0).reshape(G, 1, 4) * c).sum(axis=2).max(axis=1).sum()
    return float(B * 1.01)


def certified_selection_check(cache: O.OracleCache, qs: np.ndarray, k: int, got: np.ndarray,
                              sign_only: bool = False):
    """Compare a fast-path selection with the reference's float64 selection of the group-sum
    query.  Returns (ok, n_diff, gap, bound): the sets must be equal, except that tokens whose
    float64 score lies within 2B of the float64 k-th score (B = score_error_bound) may swap —
    there the float32 order cannot certify which side of the boundary they fall on."""
    q64 = np.asarray(qs, dtype=np.float64).sum(axis=0)
    ref = O.select(cache, q64, k, sign_only=sign_only)[0]
    got = np.asarray(got)
    diff = np.setxor1d(ref, got)
    B = score_error_bound(cache, qs, sign_only)
    if diff.size == 0:
        return True, 0, np.inf, B
    G = cache.centroids.shape[0]
    s64 = O.score(O.sign_lut(q64, G) if sign_only else O.lut(q64, cache.centroids), cache.codes)
    dyn = np.setdiff1d(ref, np.concatenate([cache.sinks, np.arange(cache.L, cache.L + len(cache.recent_k))]))
    kth = s64[dyn].min()
    gap = float(np.abs(s64[diff[diff < cache.L]] - kth).max()) if np.any(diff < cache.L) else np.inf
    return bool(gap <= 2 * B), int(diff.size), gap, B
