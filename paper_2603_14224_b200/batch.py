"""Batched B200 decode path: many decode units (layer x batch x KV head) in one launch.

This is the hot path the benchmark measures.  A :class:`CacheBatch` holds U units that
share a prefill length L in the fast HBM layout:

* ``signs``  [U, L, 16]  u8   — sign plane (the retrieval index), rotated by t mod 16;
* ``recs``   [U, L, 128] u8   — per-token record: 2-bit K magnitudes and V in mma.sync
  fragment order, fp16 (scale, zero) per 32-channel group, K sign words;
* ``cent32`` [U, 32, 16, 4] f32, ``alpha32`` [U, 128] f32 — codebook and key scale;
* sinks (first ``sink_count`` positions, cache.py:253-254) and the recent ring as float32
  centred K' / V rows.

``decode_step`` = per unit ``select_tokens(cache, sum_h q_h, k)`` + ``sparse_attention``
for every query head of the GQA group (cache.py:290-309, attention.py:52-62), fused.
"""

from __future__ import annotations

import ctypes as C

from dataclasses import dataclass, field

import torch

from . import _lib as L_

FD = 128


@dataclass
class CacheBatch:
    units: int
    tokens: int
    mu64: torch.Tensor
    alpha64: torch.Tensor
    mu32: torch.Tensor
    alpha32: torch.Tensor
    cent64: torch.Tensor
    cent32: torch.Tensor
    signs: torch.Tensor
    recs: torch.Tensor
    sink_idx: torch.Tensor
    sink_k: torch.Tensor
    sink_v: torch.Tensor
    recent_k: torch.Tensor                    # [U, capacity, 128] float32 centred K' rows
    recent_v: torch.Tensor                    # [U, capacity, 128] float32 V rows
    recent_n: torch.Tensor                    # [U] int32 recent rows per unit (device)
    ffrag: torch.Tensor                       # [U, blocks, FBLK] int32 forced-row fragments + row scales
    recent_host: torch.Tensor = None          # [U] int64 host mirror of recent_n (appends are host-issued)
    ref: dict = field(default_factory=dict)   # optional reference-layout planes
    bits: int = 2                             # payload bits: 2, 1 (same record, codes in 2-bit fields),
                                              # 16 (fp16 K^ / V records of 512 B, the "16 bits" variant) or
                                              # 4 / 8 (codes dequantised at prefill into those 512-B records)
    sign_in_quant: bool = True                # False: keys quantised directly (cache.py:241-244)

    @property
    def sinks(self) -> int:
        return int(self.sink_idx.shape[1])

    @property
    def recent_capacity(self) -> int:
        return int(self.recent_k.shape[1])

    @property
    def recent(self) -> int:
        """The largest recent-row count over the units."""
        return int(self.recent_host.max()) if self.units else 0

    @property
    def length(self) -> int:
        return self.tokens + self.recent

    def fast_bytes(self) -> int:
        return self.signs.numel() + self.recs.numel()


def _frag_blocks(sinks: int, capacity: int) -> int:
    return L_.lib().sikv_forced_blocks(sinks, capacity)


def empty_batch(units: int, tokens: int, *, sink_count: int = 64, recent_capacity: int = 0,
                keep_reference: bool = False, device=None, bits: int = 2, sign_in_quant: bool = True) -> CacheBatch:
    """An empty batch of `units` caches of `tokens` prefill tokens.  Fast-path variants
    (cache.py:52-75): bits 2 or 1 (the 1-bit codes use the same record, in its 2-bit fields),
    sign_in_quant True (|K'| / alpha codes + sign plane) or False (direct signed K' codes), or
    bits 16 (K' / alpha-hat and V stored in fp16: 512-B records, the two-kernel path), or bits
    4 / 8 (the reference's 4- / 8-bit codes, dequantised once at prefill into the same fp16
    records: the decode reads 512 B per selected token as at bits 16)."""
    if bits not in (1, 2, 4, 8, 16):
        raise NotImplementedError("the fast path supports bits 1, 2, 4, 8 and 16")
    dev = device or L_.require_cuda()
    S = min(sink_count, tokens)
    f32 = dict(device=dev, dtype=torch.float32)
    f64 = dict(device=dev, dtype=torch.float64)
    u8 = dict(device=dev, dtype=torch.uint8)
    cb = CacheBatch(
        units=units, tokens=tokens,
        mu64=torch.empty(units, FD, **f64), alpha64=torch.empty(units, FD, **f64),
        mu32=torch.empty(units, FD, **f32), alpha32=torch.empty(units, FD, **f32),
        cent64=torch.empty(units, 32, 16, 4, **f64), cent32=torch.empty(units, 32, 16, 4, **f32),
        signs=torch.empty(units, tokens, 16, **u8),
        recs=torch.empty(units, tokens, 512 if bits >= 4 else 128, **u8),
        sink_idx=torch.arange(S, device=dev, dtype=torch.int32).repeat(units, 1),
        sink_k=torch.empty(units, S, FD, **f32), sink_v=torch.empty(units, S, FD, **f32),
        recent_k=torch.zeros(units, recent_capacity, FD, **f32),
        recent_v=torch.zeros(units, recent_capacity, FD, **f32),
        recent_n=torch.zeros(units, device=dev, dtype=torch.int32),
        ffrag=torch.zeros(units, _frag_blocks(S, recent_capacity), L_.lib().sikv_forced_block_words(),
                          device=dev, dtype=torch.int32),
        recent_host=torch.zeros(units, dtype=torch.int64), bits=bits, sign_in_quant=bool(sign_in_quant),
    )
    if keep_reference and bits != 16:
        cb.ref = dict(
            codes=torch.empty(units, tokens, 16, **u8),
            kq=torch.empty(units, tokens, 16 * bits, **u8), vq=torch.empty(units, tokens, 16 * bits, **u8),
            ks=torch.empty(units, tokens, 4, device=dev, dtype=torch.float16),
            kz=torch.empty(units, tokens, 4, device=dev, dtype=torch.float16),
            vs=torch.empty(units, tokens, 4, device=dev, dtype=torch.float16),
            vz=torch.empty(units, tokens, 4, device=dev, dtype=torch.float16),
        )
    return cb


def subset(cb: CacheBatch, ids) -> CacheBatch:
    """A new CacheBatch holding units `ids` of `cb` (copies; e.g. one rank's shard)."""
    ix = torch.as_tensor(ids, dtype=torch.long, device=cb.signs.device)
    take = lambda t: t.index_select(0, ix)  # noqa: E731
    return CacheBatch(
        units=int(ix.numel()), tokens=cb.tokens, mu64=take(cb.mu64), alpha64=take(cb.alpha64), mu32=take(cb.mu32),
        alpha32=take(cb.alpha32), cent64=take(cb.cent64), cent32=take(cb.cent32), signs=take(cb.signs),
        recs=take(cb.recs), sink_idx=take(cb.sink_idx), sink_k=take(cb.sink_k), sink_v=take(cb.sink_v),
        recent_k=take(cb.recent_k), recent_v=take(cb.recent_v), recent_n=take(cb.recent_n), ffrag=take(cb.ffrag),
        recent_host=cb.recent_host.index_select(0, ix.cpu()), ref={k: take(v) for k, v in cb.ref.items()},
        bits=cb.bits, sign_in_quant=cb.sign_in_quant)


def _sl(t: torch.Tensor | None, u0: int, n: int):
    return None if t is None else t[u0:u0 + n]


def prefill_into(cb: CacheBatch, u0: int, keys: torch.Tensor, values: torch.Tensor,
                 workspace: torch.Tensor | None = None, check: bool = True, window: torch.Tensor | None = None,
                 pool_width: int = 7) -> None:
    """Compress raw K/V [n, L, 128] (bf16/f32/f64, on device) into units u0..u0+n-1.

    Replaces prefill (cache.py:212-271) with bits=2, group_size=32, sign_in_quant=True,
    batched over units.  Sinks: the first S positions, or with `window` [n, w, 128] the
    SnapKV-style window sinks of each unit (select_sink_tokens, cache.py:185-209, on the GPU in
    float64: snapkv.cu).  Mixed K / V dtypes are promoted to the wider one (the reference
    converts both to float64)."""
    n, L, D = keys.shape
    if values.shape != keys.shape:
        raise ValueError(f"keys and values must match, got {tuple(keys.shape)} and {tuple(values.shape)}")
    if D != FD or L != cb.tokens:
        raise ValueError(f"expected [n, {cb.tokens}, {FD}] keys, got {tuple(keys.shape)}")
    if keys.dtype != values.dtype:
        wide = torch.promote_types(keys.dtype, values.dtype)
        keys, values = keys.to(wide), values.to(wide)
    keys = keys.contiguous()
    values = values.contiguous()
    dt = L_.dtype_code(keys)
    need = L_.lib().sikv_encode_workspace_bytes(n, L, D)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=keys.device)
    status = torch.zeros(1, dtype=torch.int32, device=keys.device)
    if cb.bits in (4, 8):
        _prefill_wide(cb, u0, keys, values, dt, workspace, status)
    else:
        _prefill_fast(cb, u0, keys, values, dt, workspace, status)
    S = cb.sinks
    if window is not None and 0 < S < L:
        if window.dim() != 3 or window.shape[0] != n or window.shape[2] != D:
            raise ValueError(f"window must be [{n}, w, {D}], got {tuple(window.shape)}")
        win = window.to(device=keys.device, dtype=torch.float64).contiguous()
        wneed = L_.lib().sikv_window_sinks_workspace_bytes(n, L, win.shape[1])
        wws = workspace if workspace is not None and workspace.numel() >= wneed else \
            torch.empty(wneed, dtype=torch.uint8, device=keys.device)
        sidx = torch.empty(n, S, dtype=torch.int32, device=keys.device)
        L_.call("sikv_window_sinks", L_.ptr(keys), dt, n, L, D, L_.ptr(_sl(cb.mu64, u0, n)), L_.ptr(win),
                win.shape[1], S, pool_width, L_.ptr(sidx), L_.ptr(wws), wws.numel(), L_.stream())
        cb.sink_idx[u0:u0 + n] = sidx
    if S:
        L_.call("sikv_gather_rows", L_.ptr(keys), L_.ptr(values), dt, n, L, D,
                L_.ptr(cb.sink_idx[u0:u0 + n].contiguous()), S, L_.ptr(_sl(cb.mu64, u0, n)),
                L_.ptr(_sl(cb.sink_k, u0, n)), L_.ptr(_sl(cb.sink_v, u0, n)), 0, L_.stream())
    _pack_forced(cb, u0, n, 0, cb.ffrag.shape[1] * 16, status)
    if check:
        L_.raise_status(status, "keys")


def _prefill_fast(cb: CacheBatch, u0: int, keys, values, dt: int, workspace, status) -> None:
    """bits 1 / 2 (fused encoder: sign plane + 128-B records) and 16 (sign plane + pack16)."""
    n, L, D = keys.shape
    r = cb.ref
    r16 = cb.bits == 16
    L_.call("sikv_encode", L_.ptr(keys), L_.ptr(values), dt, n, L, D, 0 if r16 else cb.bits, 32,
            int(cb.sign_in_quant), 3, None,
            L_.ptr(_sl(cb.mu64, u0, n)), L_.ptr(_sl(cb.alpha64, u0, n)), L_.ptr(_sl(cb.mu32, u0, n)),
            L_.ptr(_sl(cb.alpha32, u0, n)), L_.ptr(_sl(cb.cent64, u0, n)), L_.ptr(_sl(cb.cent32, u0, n)),
            L_.ptr(_sl(r.get("codes"), u0, n)), L_.ptr(_sl(r.get("kq"), u0, n)),
            L_.ptr(_sl(r.get("ks"), u0, n)), L_.ptr(_sl(r.get("kz"), u0, n)),
            L_.ptr(_sl(r.get("vq"), u0, n)), L_.ptr(_sl(r.get("vs"), u0, n)),
            L_.ptr(_sl(r.get("vz"), u0, n)), L_.ptr(_sl(cb.signs, u0, n)),
            None if r16 else L_.ptr(_sl(cb.recs, u0, n)),
            L_.ptr(workspace), workspace.numel(), L_.ptr(status), L_.stream())
    if r16:
        # codes + codebook came from the encoder; the sign plane and the fp16 records here
        L_.call("sikv_pack16", L_.ptr(keys), L_.ptr(values), dt, n, L, L_.ptr(_sl(cb.mu64, u0, n)),
                L_.ptr(_sl(cb.alpha32, u0, n)), L_.ptr(_sl(cb.recs, u0, n)), L_.ptr(status), L_.stream())
    if not cb.sign_in_quant and not r16:
        # direct keys: the record dequantises to K' itself, so the attention's alpha-hat is 1
        # (16-bit records hold K' / alpha-hat whatever the key mode: alpha-hat stays)
        cb.alpha32[u0:u0 + n] = 1.0


def _prefill_wide(cb: CacheBatch, u0: int, keys, values, dt: int, workspace, status) -> None:
    """bits 4 / 8 (cache.py:52-75 with QuantConfig(bits=4|8)): the encoder writes the
    reference-layout planes (codes, key magnitudes or direct keys, values, fp16 scales / zeros:
    quantizer.py:106-184, bit-exact), a second pass writes the rotated sign plane the scoring
    kernels read; then every row is dequantised on the device exactly as cache.gather does
    (K' = sign * alpha * (qs c + zp), V = qs c + zp, cache.py:118-158, float64) and stored once
    as the 16-bit path's fp16 records (K' / alpha-hat, V): the decode is the bits-16 decode."""
    n, L, D = keys.shape
    dev = keys.device
    u8 = dict(device=dev, dtype=torch.uint8)
    f16 = dict(device=dev, dtype=torch.float16)
    b = cb.bits
    if cb.ref:
        pl = {k: v[u0:u0 + n] for k, v in cb.ref.items()}
    else:
        pl = dict(codes=torch.empty(n, L, 16, **u8), kq=torch.empty(n, L, 16 * b, **u8),
                  ks=torch.empty(n, L, 4, **f16), kz=torch.empty(n, L, 4, **f16),
                  vq=torch.empty(n, L, 16 * b, **u8), vs=torch.empty(n, L, 4, **f16),
                  vz=torch.empty(n, L, 4, **f16))
    mu64, al64 = _sl(cb.mu64, u0, n), _sl(cb.alpha64, u0, n)
    # pass 1: statistics, codebook and the reference-layout b-bit planes
    L_.call("sikv_encode", L_.ptr(keys), L_.ptr(values), dt, n, L, D, b, 32, int(cb.sign_in_quant), 3, None,
            L_.ptr(mu64), L_.ptr(al64), L_.ptr(_sl(cb.mu32, u0, n)), L_.ptr(_sl(cb.alpha32, u0, n)),
            L_.ptr(_sl(cb.cent64, u0, n)), L_.ptr(_sl(cb.cent32, u0, n)),
            L_.ptr(pl["codes"]), L_.ptr(pl["kq"]), L_.ptr(pl["ks"]), L_.ptr(pl["kz"]),
            L_.ptr(pl["vq"]), L_.ptr(pl["vs"]), L_.ptr(pl["vz"]), None, None,
            L_.ptr(workspace), workspace.numel(), L_.ptr(status), L_.stream())
    # pass 2: the rotated sign plane (bits 0 = sign plane only; its codebook copy is discarded)
    c64 = torch.empty(n, 32, 16, 4, device=dev, dtype=torch.float64)
    c32 = torch.empty(n, 32, 16, 4, device=dev, dtype=torch.float32)
    L_.call("sikv_encode", L_.ptr(keys), L_.ptr(values), dt, n, L, D, 0, 32, int(cb.sign_in_quant), 2, None,
            L_.ptr(mu64), L_.ptr(al64), None, None, L_.ptr(c64), L_.ptr(c32),
            None, None, None, None, None, None, None, L_.ptr(_sl(cb.signs, u0, n)), None,
            L_.ptr(workspace), workspace.numel(), L_.ptr(status), L_.stream())
    if not cb.sign_in_quant:
        cb.alpha32[u0:u0 + n] = 1.0          # direct keys: the records hold K' itself
    # dequantise in unit chunks (float64 K', V temporaries bounded at ~512 MiB) and pack
    rows = torch.arange(L, device=dev, dtype=torch.int64)
    zero_mu = torch.zeros(n, D, device=dev, dtype=torch.float64)
    chunk = max(1, (1 << 29) // (2 * L * D * 8))
    for c0 in range(0, n, chunk):
        m = min(chunk, n - c0)
        kd = torch.empty(m, L, D, device=dev, dtype=torch.float64)
        vd = torch.empty(m, L, D, device=dev, dtype=torch.float64)
        pa = [L_.ptr(pl[x][c0:c0 + m]) for x in ("codes", "kq", "ks", "kz", "vq", "vs", "vz")]
        for which, out in ((1, kd), (0, vd)):
            L_.call("sikv_dequant_rows", *pa, None, None, L_.ptr(al64[c0:c0 + m]), b, 32, int(cb.sign_in_quant),
                    m, L, D, L_.ptr(rows), L, which, L_.ptr(out), L_.stream())
        L_.call("sikv_pack16", L_.ptr(kd), L_.ptr(vd), 1, m, L, L_.ptr(zero_mu[c0:c0 + m]),
                L_.ptr(cb.alpha32[u0 + c0:u0 + c0 + m]), L_.ptr(cb.recs[u0 + c0:u0 + c0 + m]), L_.ptr(status),
                L_.stream())


def _pack_forced(cb: CacheBatch, u0: int, n: int, row_begin: int, row_end: int, status=None) -> None:
    L_.call("sikv_pack_forced", L_.ptr(_sl(cb.sink_k, u0, n)), L_.ptr(_sl(cb.sink_v, u0, n)), cb.sinks,
            L_.ptr(_sl(cb.recent_k, u0, n)), L_.ptr(_sl(cb.recent_v, u0, n)), cb.recent_capacity,
            L_.ptr(_sl(cb.recent_n, u0, n)), 0, L_.ptr(_sl(cb.alpha32, u0, n)), n,
            L_.ptr(_sl(cb.ffrag, u0, n)), cb.ffrag.shape[1], row_begin, row_end, L_.ptr(status), L_.stream())


def prefill_batch(keys: torch.Tensor, values: torch.Tensor, *, sink_count: int = 64,
                  recent_capacity: int = 0, keep_reference: bool = False, window: torch.Tensor | None = None,
                  pool_width: int = 7, bits: int = 2, sign_in_quant: bool = True) -> CacheBatch:
    U, L, D = keys.shape
    cb = empty_batch(U, L, sink_count=sink_count, recent_capacity=recent_capacity,
                     keep_reference=keep_reference, device=keys.device, bits=bits, sign_in_quant=sign_in_quant)
    prefill_into(cb, 0, keys, values, window=window, pool_width=pool_width)
    return cb


def reserve_recent(cb: CacheBatch, capacity: int) -> None:
    """Grow the recent-row ring to at least `capacity` rows per unit (amortised doubling by
    the appends; call it up front to keep reallocation out of a timed decode loop).  The
    stored rows and their packed fragment blocks are copied; the new blocks start empty."""
    old = cb.recent_capacity
    if capacity <= old:
        return
    cap = max(capacity, 2 * old, 16)
    cap = (cap + 15) // 16 * 16
    U, dev = cb.units, cb.recent_k.device
    rk = torch.zeros(U, cap, FD, device=dev, dtype=torch.float32)
    rv = torch.zeros(U, cap, FD, device=dev, dtype=torch.float32)
    rk[:, :old] = cb.recent_k
    rv[:, :old] = cb.recent_v
    fr = torch.zeros(U, _frag_blocks(cb.sinks, cap), cb.ffrag.shape[2], device=dev, dtype=torch.int32)
    fr[:, :cb.ffrag.shape[1]] = cb.ffrag
    cb.recent_k, cb.recent_v, cb.ffrag = rk, rv, fr


def append_batch(cb: CacheBatch, k: torch.Tensor, v: torch.Tensor, units=None, *, check: bool = True) -> None:
    """append_token (cache.py:274-287) for every unit, or for the units `units` (distinct ids):
    row i of k / v [n, 128] becomes the next recent row of its unit, centred with the frozen
    prefill mu, force-included in every later decode step (scored -inf, cache.py:302).  The
    ring grows by doubling when a unit fills it.  check=True reads the device status word
    (one sync) and raises ValueError for non-finite rows like the reference; check=False
    keeps the append fully asynchronous."""
    ids = None if units is None else torch.as_tensor(units, dtype=torch.long)
    n = cb.units if ids is None else int(ids.numel())
    if k.shape != (n, FD) or v.shape != (n, FD):
        raise ValueError(f"k and v must have shape ({n}, {FD})")
    if ids is not None and (ids.numel() != torch.unique(ids).numel() or
                            (ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= cb.units))):
        raise ValueError("units must be distinct ids in range")
    if k.dtype != v.dtype:
        wide = torch.promote_types(k.dtype, v.dtype)
        k, v = k.to(wide), v.to(wide)
    k = k.contiguous()
    v = v.contiguous()
    host = cb.recent_host if ids is None else cb.recent_host[ids]
    need = int(host.max()) + 1 if n else 0
    if need > cb.recent_capacity:
        reserve_recent(cb, need)
    dev_ids = None if ids is None else ids.to(device=k.device, dtype=torch.int32)
    status = torch.zeros(1, dtype=torch.int32, device=k.device)
    L_.call("sikv_append_forced", L_.ptr(k), L_.ptr(v), L_.dtype_code(k), n, L_.ptr(dev_ids), L_.ptr(cb.mu64),
            L_.ptr(cb.alpha32), L_.ptr(cb.sink_k), L_.ptr(cb.sink_v), cb.sinks, L_.ptr(cb.recent_k),
            L_.ptr(cb.recent_v), cb.recent_capacity, L_.ptr(cb.recent_n), L_.ptr(cb.ffrag), cb.ffrag.shape[1],
            L_.ptr(status), L_.stream())
    if ids is None:
        cb.recent_host += 1
    else:
        cb.recent_host[ids] += 1
    if check:
        L_.raise_status(status, "appended token")


@dataclass
class DecodeOutput:
    out: torch.Tensor                 # [U, Gq, 128] float32
    lse: torch.Tensor | None          # [U, Gq] natural-log partition function of the logits
    selection: torch.Tensor | None    # [U, stride] int32 sorted indices (first counts[u] valid)
    counts: torch.Tensor | None       # [U] int32
    diag: torch.Tensor | None         # [U] int32


_WS: dict = {}


def _workspace(units: int, tokens: int, k: int, sinks: int, device) -> torch.Tensor:
    """Decode scratch (fallback bitmaps, dynamic lists), cached per (device, stream): steps on
    one stream reuse it in order; steps on different streams never share one."""
    need = L_.lib().sikv_decode_workspace_bytes_k(units, tokens, k, sinks)
    dev = device.index if device.index is not None else torch.cuda.current_device()
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def decode_step(cb: CacheBatch, q: torch.Tensor, k: int, *, cap: int = 0, with_selection: bool = False,
                with_lse: bool = False, with_diag: bool = False, out: torch.Tensor | None = None,
                sel_buf: torch.Tensor | None = None, kernel: int = 0, append=None,
                sign_only: bool = False, unit_map=None, exchange=None) -> DecodeOutput:
    """One fused decode step over all units; q is [U, Gq, 128] (float32 or bf16).

    unit_map ([Uq] ints, each < cb.units): query unit i reads cache unit unit_map[i] (q, out and
    the selection are per query unit); see decode_step_per_head.
    sign_only=True scores with the sign-only LUT (select_tokens(..., sign_only=True),
    retrieval.py:54-62).  append=(k, v) first appends one token per unit ([U, 128] rows, append_batch without the
    status sync), so a generation step is one call.  kernel: 0 auto, 1 one CTA per unit,
    3 each unit split across a CTA cluster (long contexts, few units), 4 two kernels
    (selection with two unit groups per SM, then attention).
    exchange (shard.OutputExchange): the multi-GPU output all-gather fused into the step; every
    rank's outputs land as bf16 in every rank's exchange buffer (exchange.wait() orders a
    stream after the step of every rank)."""
    if append is not None:
        append_batch(cb, append[0], append[1], check=False)
    umap = None
    U = cb.units
    if unit_map is not None:
        um = torch.as_tensor(unit_map)
        if um.dim() != 1:
            raise ValueError("unit_map must be 1-D")
        if not um.is_cuda and um.numel() and (int(um.min()) < 0 or int(um.max()) >= cb.units):
            raise ValueError(f"unit_map ids must be in [0, {cb.units})")
        umap = um.to(device=cb.signs.device, dtype=torch.int32).contiguous()
        U = int(umap.numel())
    if q.dim() != 3 or q.shape[0] != U or q.shape[2] != FD:
        raise ValueError(f"q must be [{U}, Gq, {FD}], got {tuple(q.shape)}")
    Gq = q.shape[1]
    if k < 0:
        raise ValueError(f"k must be non-negative, got {k}")
    qf = q if q.dtype == torch.float32 and q.is_contiguous() else q.float().contiguous()
    dev = q.device
    if out is None:
        out = torch.empty(U, Gq, FD, device=dev, dtype=torch.float32)
    elif (out.dtype != torch.float32 or tuple(out.shape) != (U, Gq, FD) or not out.is_contiguous()
          or out.device != dev):
        raise ValueError(f"out must be a contiguous float32 [{U}, {Gq}, {FD}] tensor on {dev}")
    lse = torch.empty(U, Gq, device=dev, dtype=torch.float32) if with_lse else None
    R = cb.recent
    sel = cnt = None
    stride = 0
    if with_selection:
        need = cb.sinks + min(k, cb.tokens - cb.sinks) + R
        if sel_buf is None:
            sel = torch.empty(U, max(need, 1), device=dev, dtype=torch.int32)
        elif (sel_buf.dtype != torch.int32 or sel_buf.dim() != 2 or sel_buf.shape[0] != U
              or sel_buf.shape[1] < need or not sel_buf.is_contiguous() or sel_buf.device != dev):
            raise ValueError(f"sel_buf must be a contiguous int32 [{U}, >= {need}] tensor on {dev}")
        else:
            sel = sel_buf
        stride = int(sel.shape[1])
        cnt = torch.empty(U, device=dev, dtype=torch.int32)
    diag = torch.empty(U, device=dev, dtype=torch.int32) if with_diag else None
    ws = _workspace(U, cb.tokens, k, cb.sinks, dev)
    args = (L_.ptr(cb.signs), L_.ptr(cb.recs), L_.ptr(cb.cent32), L_.ptr(cb.alpha32),
            L_.ptr(cb.sink_idx), cb.sinks, L_.ptr(cb.ffrag), cb.ffrag.shape[1], L_.ptr(cb.recent_n), R,
            L_.ptr(qf), U, cb.tokens, Gq, k, cap,
            L_.ptr(out), L_.ptr(lse), L_.ptr(sel), stride, L_.ptr(cnt),
            L_.ptr(diag), L_.ptr(ws), ws.numel(), L_.ptr(umap), int(sign_only) | (2 if cb.bits >= 4 else 0), kernel)
    if exchange is None:
        L_.call("sikv_decode_step", *args, L_.stream())
    else:
        L_.call("sikv_decode_step_x", *args, C.byref(exchange.cstruct(U, Gq)), L_.stream())
    return DecodeOutput(out, lse, sel, cnt, diag)


_UMAPS: dict = {}


def decode_step_per_head(cb: CacheBatch, q: torch.Tensor, k: int, *, out: torch.Tensor | None = None,
                         **kw) -> DecodeOutput:
    """The per-q-head selection policy (cache.py:290-309 with each query head's own query):
    every query head selects its own top-k over its KV head's cache and attends to it.  q is
    [U, Gq, 128]; out [U, Gq, 128]; selection / counts per (unit, head) as [U * Gq, ...]."""
    U, Gq, D = q.shape
    if U != cb.units or D != FD:
        raise ValueError(f"q must be [{cb.units}, Gq, {FD}], got {tuple(q.shape)}")
    key = (U, Gq, q.device)
    umap = _UMAPS.get(key)
    if umap is None:
        umap = torch.arange(U, dtype=torch.int32).repeat_interleave(Gq).to(q.device)
        _UMAPS[key] = umap
    o = None if out is None else out.view(U * Gq, 1, D)
    res = decode_step(cb, q.reshape(U * Gq, 1, D), k, unit_map=umap, out=o, **kw)
    lse = None if res.lse is None else res.lse.view(U, Gq)
    return DecodeOutput(res.out.view(U, Gq, D), lse, res.selection, res.counts, res.diag)


def score_fast(cb: CacheBatch, q: torch.Tensor, sign_only: bool = False) -> torch.Tensor:
    """float32 fast-path scores of every prefill token (group-summed query) [U, L]."""
    qf = q.float().contiguous()
    out = torch.empty(cb.units, cb.tokens, device=q.device, dtype=torch.float32)
    L_.call("sikv_score_fast", L_.ptr(cb.signs), L_.ptr(cb.cent32), L_.ptr(qf), q.shape[1], cb.units,
            cb.tokens, int(sign_only), L_.ptr(out), L_.stream())
    return out


def decode_smem_bytes(tokens: int, k: int, sinks: int, gq: int, cap: int = 0) -> int:
    return L_.lib().sikv_decode_smem_bytes(tokens, k, sinks, gq, cap)
