"""numpy inverse of the fast HBM layout (test helper): fast planes -> reference planes.

Mirrors the permutations in paper_2603_14224_b200/csrc/common.cuh (k4_pos, vpay_pos) and
the rotated sign plane, so the tests can check the fast layout bit-exactly against the
oracle's reference-layout planes.
"""

import numpy as np


def k4_pos(ch):
    """K nibble (e2m1: sign at bit 3, code at bits 0-1) of channel ch: (word, bit)."""
    j, n = ch >> 5, ch & 31
    ss, e, rr = n >> 4, (n >> 3) & 1, n & 7
    return 4 * (rr >> 1) + j, 16 * ss + 8 * e + 4 * (rr & 1)


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
    vpar [L,4,2] u16, negative-sign mask [L,128] bool).  K params are stored as (2 qs, zp)."""
    w = recs.view(np.uint32)           # [L, 32]
    L = recs.shape[0]
    kc = np.empty((L, 128), np.uint8)
    vc = np.empty((L, 128), np.uint8)
    neg = np.empty((L, 128), bool)
    for ch in range(128):
        wd, bt = k4_pos(ch)
        nib = (w[:, wd] >> bt) & 15
        assert ((nib & 4) == 0).all()
        kc[:, ch] = nib & 3
        neg[:, ch] = (nib & 8).astype(bool)
        wd, bt = vpay_pos(ch)
        vc[:, ch] = (w[:, 16 + wd] >> bt) & 3
    kp = recs[:, 96:112].copy().view(np.uint16).reshape(L, 4, 2)
    qs2 = kp[..., 0].view(np.float16)
    kpar = kp.copy()
    kpar[..., 0] = (qs2 / np.float16(2)).astype(np.float16).view(np.uint16)
    assert (kpar[..., 0].view(np.float16) * np.float16(2) == qs2).all()
    vpar = recs[:, 112:128].copy().view(np.uint16).reshape(L, 4, 2)
    return kc, vc, kpar, vpar, neg


def records16_to_arrays(recs: np.ndarray):
    """[L, 512] u8 16-bit records -> (K^ [L, 128] fp16, V [L, 128] fp16) in channel order
    (inverse of common.cuh k16_off / v16_off)."""
    L = recs.shape[0]
    h = recs.view(np.uint16)                    # [L, 256]
    ch = np.arange(128)
    s, e, t4 = ch >> 4, (ch >> 3) & 1, (ch & 7) >> 1
    koff = 64 * t4 + 4 * (2 * s + e) + 2 * (ch & 1)
    m, r = ch >> 4, ch & 15
    voff = 256 + 32 * (r & 7) + 4 * m + 2 * (r >> 3)
    return h[:, koff // 2].view(np.float16).reshape(L, 128), h[:, voff // 2].view(np.float16).reshape(L, 128)
