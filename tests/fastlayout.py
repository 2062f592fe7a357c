"""numpy inverse of the fast HBM layout (test helper): fast planes -> reference planes.

Mirrors the permutations in paper_2603_14224_b200/csrc/common.cuh (kpay_pos, vpay_pos,
ksgn_pos) and the rotated sign plane, so the tests can check the fast layout bit-exactly
against the oracle's reference-layout planes.
"""

import numpy as np


def kpay_pos(ch):
    s, r = ch >> 4, ch & 15
    e, rr = (r >> 3) & 1, r & 7
    t4, hi = rr >> 1, rr & 1
    u, i = s >> 2, ((s & 3) << 1) | e
    return 2 * t4 + u, 2 * i + 16 * hi


def ksgn_pos(ch):
    s, r = ch >> 4, ch & 15
    e, rr = (r >> 3) & 1, r & 7
    t4, hi = rr >> 1, rr & 1
    u, i = s >> 2, ((s & 3) << 1) | e
    return t4, 8 * u + i + 16 * hi


def vpay_pos(ch):
    m, r = ch >> 4, ch & 15
    g, e = r & 7, r >> 3
    return g, 8 * (m >> 1) + 2 * (2 * (m & 1) + e)


def unrotate_signs(signs_fast: np.ndarray) -> np.ndarray:
    """[L, 16] rotated -> reference packed codes [L, 16]."""
    L = signs_fast.shape[0]
    t = np.arange(L)[:, None]
    i = np.arange(16)[None, :]
    out = np.empty_like(signs_fast)
    out[t, (t + i) % 16] = signs_fast[t, i]
    return out


def records_to_reference(recs: np.ndarray):
    """[L, 128] u8 records -> (kq codes [L,128], vq codes [L,128], kpar [L,4,2] u16,
    vpar [L,4,2] u16, negative-sign mask [L,128] bool)."""
    w = recs.view(np.uint32)           # [L, 32]
    L = recs.shape[0]
    kc = np.empty((L, 128), np.uint8)
    vc = np.empty((L, 128), np.uint8)
    neg = np.empty((L, 128), bool)
    for ch in range(128):
        wd, bt = kpay_pos(ch)
        kc[:, ch] = (w[:, wd] >> bt) & 3
        wd, bt = vpay_pos(ch)
        vc[:, ch] = (w[:, 8 + wd] >> bt) & 3
        wd, bt = ksgn_pos(ch)
        neg[:, ch] = ((w[:, 24 + wd] >> bt) & 1).astype(bool)
    kpar = recs[:, 64:80].copy().view(np.uint16).reshape(L, 4, 2)
    vpar = recs[:, 80:96].copy().view(np.uint16).reshape(L, 4, 2)
    assert (w[:, 28:] == 0).all()
    return kc, vc, kpar, vpar, neg
