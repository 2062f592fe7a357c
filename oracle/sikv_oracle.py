"""CPU oracle for the self-indexing KV-cache decode path (TEST INFRASTRUCTURE ONLY).

This module is a float64 numpy restatement of the reference package
(``/root/reference/pkg/src/sikv``) for the functions on the hot path. It is the
checker the GPU path is compared against; it is never called by the product
(``paper_2603_14224_b200``), only by ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by importing the real reference in the build
container (``tests/golden/make_golden.py``) and against the hand-derived known
answers in the reference's own tests. The reference itself cannot travel to the
GPU box, so this restatement is what runs there.

Every function cites the reference file:line it restates. Arithmetic order is
kept where it decides bits:

* column mean = sequential row accumulation then one division
  (numpy ``add.reduce`` over axis 0, ``normalize.py:59``);
* LUT entries = ``(q0*c0 + q2*c2) + (q1*c1 + q3*c3)`` — the order numpy's
  ``einsum("gd,gcd->gc")`` uses on this host (two-lane SIMD accumulation,
  measured in the build container, ``retrieval.py:50``);
* token scores = numpy ``sum(axis=1)`` (8-way unrolled pairwise sum,
  ``retrieval.py:77``), restated explicitly in :func:`pairwise_rows`;
* codebook = sequential ``np.add.at`` scatter (``codebook.py:150-151``);
* float16 parameters = direct float64 -> float16 rounding (``quantizer.py:98-99``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SUB = 4            # subvector width (codebook.py:21)
NCODE = 16         # codes per group (codebook.py:22)
_W = np.array([8, 4, 2, 1], dtype=np.uint8)      # MSB-first weights (codebook.py:25)
_SH = np.array([3, 2, 1, 0], dtype=np.uint8)
_TINY = np.float16(2.0 ** -24)                    # quantizer.py:31


# --------------------------------------------------------------------------- bit packing
def pack(codes: np.ndarray, bits: int) -> np.ndarray:
    """Row-wise little-endian packing, element 0 in the low bits (bitpack.py:27-48)."""
    codes = np.asarray(codes)
    assert bits in (1, 2, 4, 8)
    if codes.size and (codes.min() < 0 or codes.max() >= (1 << bits)):
        raise ValueError(f"codes out of range for {bits}-bit packing")
    rows, n = codes.shape
    per = 8 // bits
    width = -(-n // per)
    buf = np.zeros((rows, width * per), dtype=np.uint16)
    buf[:, :n] = codes
    out = np.zeros((rows, width), dtype=np.uint16)
    for m in range(per):
        out |= buf[:, m::per] << (bits * m)
    return out.astype(np.uint8)


def unpack(packed: np.ndarray, bits: int, n: int) -> np.ndarray:
    """Inverse of :func:`pack` (bitpack.py:51-67)."""
    packed = np.asarray(packed, dtype=np.uint8)
    per = 8 // bits
    mask = (1 << bits) - 1
    out = np.empty((packed.shape[0], packed.shape[1] * per), dtype=np.uint8)
    for m in range(per):
        out[:, m::per] = (packed >> (bits * m)) & mask
    return out[:, :n]


# --------------------------------------------------------------------------- encoder
def channel_stats(K: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """mu = column mean, alpha = max |K - mu| per column (normalize.py:56-61)."""
    K = np.asarray(K, dtype=np.float64)
    # np.add.reduce over axis 0 accumulates row after row (sequential per
    # column); verified bit-identical to an explicit row loop in the build container.
    mu = np.add.reduce(K, axis=0) / K.shape[0]
    alpha = np.abs(K - mu).max(axis=0)
    return mu, alpha


def sign_codes(Kp: np.ndarray) -> np.ndarray:
    """4-bit MSB-first sign code per 4-wide subvector, sign(0) = +1 (codebook.py:116-125)."""
    L, D = Kp.shape
    sub = (Kp.reshape(L, D // SUB, SUB) >= 0).astype(np.uint8)
    return (sub * _W).sum(axis=2).astype(np.uint8)


def codebook(Kp: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """One-pass centroid means, empty cluster = 0 (codebook.py:128-160)."""
    L, D = Kp.shape
    G = D // SUB
    sums = np.zeros((G, NCODE, SUB))
    cnt = np.zeros((G, NCODE), dtype=np.int64)
    gi = np.broadcast_to(np.arange(G), (L, G))
    np.add.at(sums, (gi, codes), Kp.reshape(L, G, SUB))
    np.add.at(cnt, (gi, codes), 1)
    out = np.zeros_like(sums)
    np.divide(sums, cnt[:, :, None], out=out, where=cnt[:, :, None] > 0)
    return out


def narrow(scales: np.ndarray, zeros: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """float16 narrowing with the underflow clamp (quantizer.py:97-103)."""
    s16 = scales.astype(np.float16)
    z16 = zeros.astype(np.float16)
    if not (np.isfinite(s16).all() and np.isfinite(z16).all()):
        raise ValueError("group min/max exceed the 16-bit parameter range")
    s16 = np.where((scales > 0) & (s16 == 0), _TINY, s16)
    return s16, z16


@dataclass
class QPlane:
    """Packed B-bit payload plus float16 scale / zero-point (quantizer.py:52-94)."""
    packed: np.ndarray
    scales: np.ndarray
    zeros: np.ndarray
    bits: int
    group: int
    dim: int

    def codes(self, rows=None) -> np.ndarray:
        p = self.packed if rows is None else self.packed[np.asarray(rows)]
        return unpack(p, self.bits, self.dim)


def quantize(X: np.ndarray, bits: int, group: int) -> QPlane:
    """Token-wise, group-wise asymmetric quantization (quantizer.py:106-140)."""
    X = np.asarray(X, dtype=np.float64)
    L, D = X.shape
    if D % group:
        raise ValueError(f"channel count {D} not divisible by group_size {group}")
    lv = (1 << bits) - 1
    xg = X.reshape(L, D // group, group)
    lo = xg.min(axis=2)
    hi = xg.max(axis=2)
    s16, z16 = narrow((hi - lo) / lv, lo)
    qs = s16.astype(np.float64)[:, :, None]
    zp = z16.astype(np.float64)[:, :, None]
    live = qs > 0
    t = np.zeros_like(xg)
    np.divide(xg - zp, qs, out=t, where=live)
    c = np.clip(np.floor(t + 0.5), 0, lv)
    c = np.where(live, c, 0.0).astype(np.uint8).reshape(L, D)
    return QPlane(pack(c, bits), s16, z16, bits, group, D)


def dequantize(q: QPlane, rows=None) -> np.ndarray:
    """qs * code + zp (quantizer.py:143-152)."""
    c = q.codes(rows).astype(np.float64)
    sel = slice(None) if rows is None else np.asarray(rows)
    n = c.shape[0]
    s = q.scales[sel].astype(np.float64)
    z = q.zeros[sel].astype(np.float64)
    g = c.reshape(n, q.dim // q.group, q.group)
    return (g * s[:, :, None] + z[:, :, None]).reshape(n, q.dim)


def quantize_key_mags(Kp: np.ndarray, alpha: np.ndarray, bits: int, group: int) -> QPlane:
    """Quantize |K'| / alpha, alpha == 0 channels -> 0 (quantizer.py:155-170)."""
    m = np.abs(Kp) / np.where(alpha == 0, 1.0, alpha)
    m[:, alpha == 0] = 0.0
    if m.max(initial=0.0) > 1.0 + 1e-9:
        raise ValueError("alpha does not dominate |keys_norm|")
    return quantize(m, bits, group)


def sign_plane(codes: np.ndarray) -> np.ndarray:
    """-1/+1 signs decoded from the 4-bit codes (codebook.py:82-86)."""
    b = (codes[:, :, None] >> _SH) & 1
    return b.reshape(codes.shape[0], -1).astype(np.float64) * 2.0 - 1.0


def dequantize_keys(q: QPlane, alpha: np.ndarray, codes: np.ndarray, rows=None) -> np.ndarray:
    """K' = sign * alpha * (qs*c + zp) (quantizer.py:173-184)."""
    sel = codes if rows is None else codes[np.asarray(rows)]
    return sign_plane(sel) * alpha[None, :] * dequantize(q, rows)


# --------------------------------------------------------------------------- cache
@dataclass
class OracleCache:
    """One head's compressed cache (cache.py:78-182), first-S or window sinks."""
    dim: int
    L: int
    mu: np.ndarray
    alpha: np.ndarray
    codes: np.ndarray            # (L, G) uint8, unpacked
    centroids: np.ndarray        # (G, 16, 4) float64
    kmag: QPlane | None
    kdirect: QPlane | None
    vq: QPlane | None
    kfull: np.ndarray | None
    vfull: np.ndarray | None
    sinks: np.ndarray
    sink_k: np.ndarray
    sink_v: np.ndarray
    bits: int
    sign_in_quant: bool = True
    recent_k: list = field(default_factory=list)
    recent_v: list = field(default_factory=list)

    @property
    def length(self) -> int:
        return self.L + len(self.recent_k)

    @property
    def packed_codes(self) -> np.ndarray:
        return pack(self.codes, 4)

    def recents(self) -> np.ndarray:
        return np.arange(self.L, self.length, dtype=np.int64)

    def forced(self) -> np.ndarray:
        return np.union1d(self.sinks, self.recents())

    def gather(self, idx) -> tuple[np.ndarray, np.ndarray]:
        """Row dispatch recent / sink / dequant (cache.py:118-158)."""
        idx = np.asarray(idx, dtype=np.int64)
        Kr = np.empty((idx.size, self.dim))
        Vr = np.empty((idx.size, self.dim))
        rec = idx >= self.L
        snk = ~rec & np.isin(idx, self.sinks)
        dyn = ~rec & ~snk
        if rec.any():
            rel = idx[rec] - self.L
            Kr[rec] = np.stack([self.recent_k[i] for i in rel])
            Vr[rec] = np.stack([self.recent_v[i] for i in rel])
        if snk.any():
            pos = np.searchsorted(self.sinks, idx[snk])
            Kr[snk] = self.sink_k[pos]
            Vr[snk] = self.sink_v[pos]
        if dyn.any():
            rows = idx[dyn]
            if self.bits == 16:
                Kr[dyn] = self.kfull[rows]
                Vr[dyn] = self.vfull[rows]
            else:
                if self.sign_in_quant:
                    Kr[dyn] = dequantize_keys(self.kmag, self.alpha, self.codes, rows)
                else:
                    Kr[dyn] = dequantize(self.kdirect, rows)
                Vr[dyn] = dequantize(self.vq, rows)
        return Kr, Vr


def window_sinks(Kp: np.ndarray, W: np.ndarray, count: int, pool: int = 7) -> np.ndarray:
    """SnapKV-style vote + max-pool + stable top-count (cache.py:185-209)."""
    from scipy.ndimage import maximum_filter1d
    if count == 0:
        return np.empty(0, dtype=np.int64)
    L = Kp.shape[0]
    if count >= L:
        return np.arange(L, dtype=np.int64)
    lg = (Kp @ W.T) / np.sqrt(Kp.shape[1])
    lg -= lg.max(axis=0, keepdims=True)
    w = np.exp(lg)
    w /= w.sum(axis=0, keepdims=True)
    pooled = maximum_filter1d(w.sum(axis=1), size=pool, mode="nearest")
    return np.sort(np.argsort(-pooled, kind="stable")[:count]).astype(np.int64)


def prefill(K, V, *, bits: int = 2, group: int = 32, sink_count: int = 64,
            sign_in_quant: bool = True, window=None) -> OracleCache:
    """Stats -> centre -> codes -> codebook -> quantize -> sinks (cache.py:212-271)."""
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    L, D = K.shape
    mu, alpha = channel_stats(K)
    Kp = K - mu
    codes = sign_codes(Kp)
    cent = codebook(Kp, codes)
    kmag = kdirect = vq = kfull = vfull = None
    if bits == 16:
        kfull, vfull = Kp.copy(), V.copy()
    else:
        if sign_in_quant:
            kmag = quantize_key_mags(Kp, alpha, bits, group)
        else:
            kdirect = quantize(Kp, bits, group)
        vq = quantize(V, bits, group)
    if sink_count == 0:
        sinks = np.empty(0, dtype=np.int64)
    elif window is not None:
        sinks = window_sinks(Kp, np.asarray(window, dtype=np.float64), sink_count)
    else:
        sinks = np.arange(min(sink_count, L), dtype=np.int64)
    return OracleCache(D, L, mu, alpha, codes, cent, kmag, kdirect, vq, kfull, vfull,
                       sinks, Kp[sinks].copy(), V[sinks].copy(), bits, sign_in_quant)


def append(cache: OracleCache, k, v) -> None:
    """Recent buffer gets (k - mu, v) at full precision (cache.py:274-287)."""
    cache.recent_k.append(np.asarray(k, dtype=np.float64) - cache.mu)
    cache.recent_v.append(np.asarray(v, dtype=np.float64).copy())


# --------------------------------------------------------------------------- retrieval
def lut(q: np.ndarray, centroids: np.ndarray) -> np.ndarray:
    """LUT[g][c] = q_g . centroid[g][c] (retrieval.py:46-51), einsum's pairing order."""
    G = centroids.shape[0]
    qg = np.asarray(q, dtype=np.float64).reshape(G, 1, SUB)
    p = qg * centroids
    return (p[..., 0] + p[..., 2]) + (p[..., 1] + p[..., 3])


def sign_lut(q: np.ndarray, G: int) -> np.ndarray:
    """Ablation LUT against raw +-1 patterns (retrieval.py:54-62).

    The reference's ``(G,4) @ (4,16)`` matmul sums the four exact products
    left to right for G > 1 and as (a0 + a2) + (a1 + a3) for G == 1 (the
    matrix-vector BLAS path); both orders measured in the build container."""
    pats = ((np.arange(NCODE)[:, None] >> _SH) & 1).astype(np.float64) * 2 - 1
    p = np.asarray(q, dtype=np.float64).reshape(G, 1, SUB) * pats[None]
    if G == 1:
        return (p[..., 0] + p[..., 2]) + (p[..., 1] + p[..., 3])
    return ((p[..., 0] + p[..., 1]) + p[..., 2]) + p[..., 3]


def pairwise_rows(x: np.ndarray) -> np.ndarray:
    """numpy's pairwise row sum for n <= 128 (8 strided accumulators, then a tree,
    then the remainder left to right) — the order of ``x.sum(axis=1)``."""
    n = x.shape[1]
    if n < 8:
        r = x[:, 0].copy()
        for i in range(1, n):
            r = r + x[:, i]
        return r
    assert n <= 128
    acc = [x[:, j].copy() for j in range(8)]
    i = 8
    while i < n - (n % 8):
        for j in range(8):
            acc[j] = acc[j] + x[:, i + j]
        i += 8
    res = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))
    while i < n:
        res = res + x[:, i]
        i += 1
    return res


def score(table: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """Sum of looked-up entries per token (retrieval.py:65-77)."""
    G = table.shape[0]
    return pairwise_rows(table[np.arange(G)[None, :], codes])


def top_k(scores, k: int, sink=(), recent=()) -> tuple[np.ndarray, int, int, int]:
    """Forced union + exact top-k, ties -> lower index (retrieval.py:127-161).

    Returns (sorted indices, sink_count, recent_count, dynamic_count)."""
    s = np.asarray(scores, dtype=np.float64)
    if k < 0:
        raise ValueError(f"k must be non-negative, got {k}")
    L = s.shape[0]
    snk = np.unique(np.asarray(list(sink) if not isinstance(sink, np.ndarray) else sink,
                               dtype=np.int64))
    rec = np.unique(np.asarray(list(recent) if not isinstance(recent, np.ndarray) else recent,
                               dtype=np.int64))
    for name, a in (("sink", snk), ("recent", rec)):
        if a.size and (a.min() < 0 or a.max() >= L):
            raise ValueError(f"{name} indices out of range [0, {L})")
    forced = np.union1d(snk, rec)
    keep = np.ones(L, dtype=bool)
    keep[forced] = False
    cand = np.flatnonzero(keep)
    ke = min(k, cand.size)
    dyn = cand[np.argsort(-s[cand], kind="stable")[:ke]] if ke > 0 else np.empty(0, np.int64)
    idx = np.sort(np.concatenate([forced, dyn])).astype(np.int64)
    return idx, int(snk.size), int(np.setdiff1d(rec, snk).size), int(ke)


def resolve_k(length: int, forced: int, budget=None, sparsity=None) -> int:
    """Budget / sparsity -> dynamic k (retrieval.py:164-181)."""
    if (budget is None) == (sparsity is None):
        raise ValueError("exactly one of budget and sparsity must be set")
    if budget is not None:
        if budget < 0:
            raise ValueError("budget must be non-negative")
        return max(int(budget) - forced, 0)
    if not 0.0 <= sparsity <= 1.0:
        raise ValueError("sparsity must be in [0, 1]")
    return max(int(np.floor(sparsity * length + 0.5)) - forced, 1)


def select(cache: OracleCache, q, k=None, budget=None, sparsity=None, sign_only=False):
    """LUT -> scores -> recents -inf -> top-k (cache.py:290-309)."""
    q = np.asarray(q, dtype=np.float64)
    G = cache.centroids.shape[0]
    table = sign_lut(q, G) if sign_only else lut(q, cache.centroids)
    s = np.concatenate([score(table, cache.codes), np.full(len(cache.recent_k), -np.inf)])
    if k is None:
        k = resolve_k(cache.length, cache.forced().size, budget, sparsity)
    return top_k(s, k, sink=cache.sinks, recent=cache.recents())


def attend(q, K: np.ndarray, V: np.ndarray) -> np.ndarray:
    """Max-stabilised softmax(K q / sqrt(D)) V (attention.py:35-39)."""
    lg = (K @ np.asarray(q, dtype=np.float64)) / np.sqrt(K.shape[1])
    w = np.exp(lg - lg.max())
    w /= w.sum()
    return w @ V


def sparse_attention(q, indices, cache: OracleCache) -> np.ndarray:
    """Attention over the gathered selection (attention.py:52-62)."""
    if len(indices) == 0:
        raise ValueError("selection is empty")
    Kr, Vr = cache.gather(indices)
    return attend(q, Kr, Vr)


def rel_l2(x, ref) -> float:
    """Relative L2 error with ``ref`` as reference (attention.py:65-86)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.linalg.norm(x - ref)
    n = np.linalg.norm(ref)
    return 0.0 if d == 0 else (float("inf") if n == 0 else float(d / n))


def cosine(x, ref) -> float:
    x = np.asarray(x, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    nx, ny = np.linalg.norm(x), np.linalg.norm(ref)
    if nx == 0 and ny == 0:
        return 1.0
    if nx == 0 or ny == 0:
        return 0.0
    return float(x @ ref / (nx * ny))
