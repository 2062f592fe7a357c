"""Drop-in replacement of the reference package's Python API (``sikv``), backed by CUDA.

Same names, arguments, dataclasses and ValueError messages as
``/root/reference/pkg/src/sikv/__init__.py:11-100``.  Every numeric step runs in
``libsikv_b200.so`` on the GPU (inputs are moved to the current CUDA device; results are
torch tensors there); there is no CPU fallback.  The per-head functions reproduce the
reference's float64 arithmetic in the reference's own order wherever the order decides
bits, so sign codes, payloads, fp16 parameters, mu / alpha, LUTs, scores
and top-k selections are bit-identical to the reference on the same inputs; attention is
float64 with a different summation order (agreement ~1e-15 relative).

The batched B200 hot path (many units, one fused kernel) is :mod:`.batch`.
"""

from __future__ import annotations

import hashlib
import math
from contextlib import contextmanager
from dataclasses import asdict, dataclass, field
from typing import Iterator

import numpy as np
import torch

from . import _lib as L_

SUBVECTOR_DIM = 4
CODEBOOK_SIZE = 16
PACKABLE_BITS = (1, 2, 4, 8)
PARAM_BITS = 16
FULL_PRECISION_BITS = 16
PARAM_PRECISION_BITS = 16
INDEX_BITS = 32
LOSSLESS_BITS = 16
DEFAULT_SINK_COUNT = 64
DEFAULT_POOL_WIDTH = 7


# ============================================================================ op counters
@dataclass
class OpCounters:
    """Analytic work counters (instrument.py:16-28), tallied from the shapes each call
    processes, as the reference does."""
    lut_lookups: int = 0
    lut_adds: int = 0
    score_muls: int = 0
    dense_muls: int = 0
    dense_adds: int = 0
    codebook_subvector_reads: int = 0
    kmeans_subvector_reads: int = 0
    dequant_rows: int = 0

    def as_dict(self) -> dict[str, int]:
        return asdict(self)


_active: list[OpCounters] = []


def tally(counter: str, amount: int) -> None:
    for c in _active:
        setattr(c, counter, getattr(c, counter) + amount)


@contextmanager
def collect() -> Iterator[OpCounters]:
    c = OpCounters()
    _active.append(c)
    try:
        yield c
    finally:
        _active.remove(c)


# ============================================================================ input handling
def _dev() -> torch.device:
    return L_.require_cuda()


# Input validation follows the reference (ValueError at call time).  Host arrays are checked on
# the host before they are uploaded (no device sync).  Device tensors need one device->host
# read per check; set_device_input_checks(False) skips those (the caller vouches for its
# tensors) so chained GPU calls stay asynchronous.
_DEVICE_CHECKS = True


def set_device_input_checks(on: bool) -> None:
    global _DEVICE_CHECKS
    _DEVICE_CHECKS = bool(on)


def _finite(t: torch.Tensor, host) -> bool:
    if host is not None:
        return bool(np.isfinite(host).all())
    return not _DEVICE_CHECKS or bool(torch.isfinite(t).all())


def _tensor(x, dtype=torch.float64) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(_dev())
        return t if dtype is None else t.to(dtype)
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=_dev()).to(dtype or torch.float64)


def _as_matrix(x, name: str = "matrix", keep_dtype: bool = False) -> torch.Tensor:
    """normalize.py:16-24 validation; keep_dtype keeps bf16/f32 inputs for the encoder."""
    host = None if isinstance(x, torch.Tensor) else np.asarray(x, dtype=np.float64)
    t = x.to(_dev()) if host is None else torch.as_tensor(host, device=_dev())
    if not keep_dtype or t.dtype not in (torch.float32, torch.float64, torch.bfloat16):
        t = t.to(torch.float64)
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
    if t.shape[0] < 1:
        raise ValueError(f"{name} must contain at least one row")
    if not _finite(t, host):
        raise ValueError(f"{name} contains non-finite entries")
    return t.contiguous()


def _as_query(q, dim: int | None = None) -> torch.Tensor:
    """retrieval.py:20-28."""
    host = None if isinstance(q, torch.Tensor) else np.asarray(q, dtype=np.float64)
    t = _tensor(q if host is None else host)
    if t.dim() != 1:
        raise ValueError(f"query must be 1-D, got shape {tuple(t.shape)}")
    if dim is not None and t.shape[0] != dim:
        raise ValueError(f"query has {t.shape[0]} channels, expected {dim}")
    if not _finite(t, host):
        raise ValueError("query contains non-finite entries")
    return t.contiguous()


def _ws(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=_dev())


def _status() -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=_dev())


def _rows(rows, n: int) -> torch.Tensor:
    if isinstance(rows, torch.Tensor):
        r = rows.to(_dev()).to(torch.int64).reshape(-1).contiguous()
        bad = _DEVICE_CHECKS and r.numel() and (int(r.min()) < 0 or int(r.max()) >= n)
    else:
        h = np.asarray(rows, dtype=np.int64).reshape(-1)
        bad = h.size and (h.min() < 0 or h.max() >= n)
        r = torch.as_tensor(h, device=_dev())
    if bad:
        raise ValueError(f"rows out of range [0, {n})")
    return r


# ============================================================================ bit packing
def packed_row_bytes(num_elements: int, bits: int) -> int:
    if bits not in PACKABLE_BITS:
        raise ValueError(f"bits must be one of {PACKABLE_BITS}, got {bits}")
    return -(-num_elements * bits // 8)


def _unpack(packed: torch.Tensor, bits: int, n: int) -> torch.Tensor:
    per = 8 // bits
    mask = (1 << bits) - 1
    shifts = torch.arange(per, device=packed.device, dtype=torch.uint8) * bits
    lanes = (packed.unsqueeze(-1) >> shifts) & mask
    return lanes.reshape(packed.shape[0], -1)[:, :n].contiguous()


def _pack(codes: torch.Tensor, bits: int) -> torch.Tensor:
    rows, n = codes.shape
    per = 8 // bits
    width = -(-n // per)
    buf = torch.zeros(rows, width * per, dtype=torch.int32, device=codes.device)
    buf[:, :n] = codes.to(torch.int32)
    shifts = torch.arange(per, device=codes.device, dtype=torch.int32) * bits
    return (buf.reshape(rows, width, per) << shifts).sum(-1).to(torch.uint8)


def pack_rows(codes, bits: int) -> torch.Tensor:
    """bitpack.py:27-48: rows of bits-bit codes -> uint8, lowest element in the low bits."""
    if bits not in PACKABLE_BITS:
        raise ValueError(f"bits must be one of {PACKABLE_BITS}, got {bits}")
    if isinstance(codes, torch.Tensor):
        c = codes.to(_dev())
        integer = not (c.is_floating_point() or c.is_complex() or c.dtype == torch.bool)
        lo_hi = (int(c.min()), int(c.max())) if c.numel() and integer else (0, 0)
    else:
        a = np.asarray(codes)
        integer = np.issubdtype(a.dtype, np.integer)
        lo_hi = (int(a.min()), int(a.max())) if a.size and integer else (0, 0)
        c = torch.as_tensor(a.astype(np.int64) if integer else a, device=_dev())
    if c.dim() != 2:
        raise ValueError(f"expected a 2-D code array, got shape {tuple(c.shape)}")
    if not integer:
        raise ValueError(f"codes must be integers, got dtype {c.dtype}")
    if lo_hi[0] < 0 or lo_hi[1] >= (1 << bits):
        raise ValueError(f"codes out of range for {bits}-bit packing")
    return _pack(c, bits)


def unpack_rows(packed, bits: int, num_elements: int) -> torch.Tensor:
    """bitpack.py:51-67: inverse of pack_rows, (rows, num_elements) uint8."""
    if bits not in PACKABLE_BITS:
        raise ValueError(f"bits must be one of {PACKABLE_BITS}, got {bits}")
    p = packed.to(_dev()).to(torch.uint8) if isinstance(packed, torch.Tensor) else \
        torch.as_tensor(np.asarray(packed, dtype=np.uint8), device=_dev())
    if p.dim() != 2:
        raise ValueError(f"expected a 2-D packed array, got shape {tuple(p.shape)}")
    want = packed_row_bytes(num_elements, bits)
    if p.shape[1] != want:
        raise ValueError(f"packed row has {p.shape[1]} bytes, expected {want} for {num_elements} elements "
                         f"at {bits} bits")
    return _unpack(p, bits, num_elements)


# ============================================================================ normalize
@dataclass(frozen=True, eq=False)
class NormalizationState:
    """normalize.py:27-53."""
    mu: torch.Tensor
    alpha: torch.Tensor

    def __post_init__(self) -> None:
        mu = _tensor(self.mu)
        alpha = _tensor(self.alpha)
        if mu.dim() != 1 or alpha.dim() != 1 or mu.shape != alpha.shape:
            raise ValueError(f"mu and alpha must be 1-D with equal length, got {tuple(mu.shape)} and {tuple(alpha.shape)}")
        if bool((alpha < 0).any()):
            raise ValueError("alpha must be non-negative")
        object.__setattr__(self, "mu", mu.contiguous())
        object.__setattr__(self, "alpha", alpha.contiguous())

    @property
    def dim(self) -> int:
        return int(self.mu.shape[0])


def _encode(keys: torch.Tensor, values: torch.Tensor, *, bits: int, group: int, siq: int, what: int,
            mu: torch.Tensor | None = None, alpha: torch.Tensor | None = None, codes_in=None,
            want_codes=False, want_k=False, want_v=False, want_cb=False):
    """One-unit call of the encoder; returns a dict of the requested planes."""
    Lk, D = keys.shape
    dev = keys.device
    if D > 128:
        raise NotImplementedError("dim > 128 is not supported by the encoder")
    out = {}
    mu64 = mu.contiguous() if mu is not None else torch.empty(D, dtype=torch.float64, device=dev)
    al64 = alpha.contiguous() if alpha is not None else torch.empty(D, dtype=torch.float64, device=dev)
    G = D // 4
    qb = bits if bits in PACKABLE_BITS else 2
    payb = packed_row_bytes(D, qb)
    ng = D // group if bits in PACKABLE_BITS else 1
    codes = torch.empty(Lk, -(-G // 2), dtype=torch.uint8, device=dev) if want_codes else None
    kq = torch.empty(Lk, payb, dtype=torch.uint8, device=dev) if want_k else None
    ks = torch.empty(Lk, ng, dtype=torch.float16, device=dev) if want_k else None
    kz = torch.empty(Lk, ng, dtype=torch.float16, device=dev) if want_k else None
    vq = torch.empty(Lk, payb, dtype=torch.uint8, device=dev) if want_v else None
    vs = torch.empty(Lk, ng, dtype=torch.float16, device=dev) if want_v else None
    vz = torch.empty(Lk, ng, dtype=torch.float16, device=dev) if want_v else None
    c64 = torch.empty(G, 16, 4, dtype=torch.float64, device=dev) if (what & 2) else None
    ws = _ws(L_.lib().sikv_encode_workspace_bytes(1, Lk, D))
    st = _status()
    L_.call("sikv_encode", L_.ptr(keys), L_.ptr(values), L_.dtype_code(keys), 1, Lk, D,
            bits if bits in PACKABLE_BITS else 0, group, siq, what, L_.ptr(codes_in), L_.ptr(mu64),
            L_.ptr(al64), None, None, L_.ptr(c64), None, L_.ptr(codes), L_.ptr(kq), L_.ptr(ks), L_.ptr(kz),
            L_.ptr(vq), L_.ptr(vs), L_.ptr(vz), None, None, L_.ptr(ws), ws.numel(), L_.ptr(st), L_.stream())
    out.update(mu=mu64, alpha=al64, codes=codes, kq=kq, ks=ks, kz=kz, vq=vq, vs=vs, vz=vz, cent=c64, status=st)
    return out


def compute_channel_stats(keys) -> NormalizationState:
    """normalize.py:56-61 (float64-exact, see encode.cu)."""
    K = _as_matrix(keys, "keys", keep_dtype=True)
    r = _encode(K, K, bits=2, group=4, siq=0, what=1)
    L_.raise_status(r["status"], "keys")
    return NormalizationState(mu=r["mu"], alpha=r["alpha"])


def apply_normalization(keys, state: NormalizationState) -> torch.Tensor:
    """normalize.py:64-69."""
    K = _as_matrix(keys, "keys", keep_dtype=True)
    if K.shape[1] != state.dim:
        raise ValueError(f"keys have {K.shape[1]} channels, state has {state.dim}")
    out = torch.empty(K.shape, dtype=torch.float64, device=K.device)
    L_.call("sikv_center", L_.ptr(K), L_.dtype_code(K), 1, K.shape[0], K.shape[1], L_.ptr(state.mu),
            L_.ptr(out), L_.stream())
    return out


def sign_entropy(signs) -> torch.Tensor:
    """normalize.py:72-88 (a metric, not on the decode path)."""
    S = _tensor(signs)
    if S.dim() != 2 or S.shape[0] < 1:
        raise ValueError(f"signs must be a non-empty 2-D matrix, got shape {tuple(S.shape)}")
    if not bool(((S == -1.0) | (S == 1.0)).all()):
        raise ValueError("sign matrix entries must be -1 or +1")
    p = (S > 0).to(torch.float64).mean(dim=0)
    out = torch.zeros_like(p)
    m = (p > 0) & (p < 1)
    pi = p[m]
    out[m] = -(pi * torch.log2(pi) + (1 - pi) * torch.log2(1 - pi))
    return out


# ============================================================================ codebook
@dataclass(frozen=True, eq=False)
class SignCodeMatrix:
    """codebook.py:50-90; packed [L, ceil(G/2)] uint8 on the device."""
    packed: torch.Tensor
    num_tokens: int
    num_groups: int

    def __post_init__(self) -> None:
        expected = (self.num_tokens, -(-self.num_groups // 2))
        if tuple(self.packed.shape) != expected or self.packed.dtype != torch.uint8:
            raise ValueError(f"packed array must be uint8 with shape {expected}, got {self.packed.dtype} "
                             f"{tuple(self.packed.shape)}")

    @classmethod
    def from_codes(cls, codes) -> "SignCodeMatrix":
        c = codes.to(_dev()) if isinstance(codes, torch.Tensor) else torch.as_tensor(np.asarray(codes), device=_dev())
        if c.numel() and (int(c.min()) < 0 or int(c.max()) >= 16):
            raise ValueError("codes out of range for 4-bit packing")
        return cls(packed=_pack(c, 4), num_tokens=int(c.shape[0]), num_groups=int(c.shape[1]))

    def unpack(self, rows=None) -> torch.Tensor:
        p = self.packed if rows is None else self.packed[_rows(rows, self.num_tokens)]
        return _unpack(p, 4, self.num_groups)

    def sign_plane(self, rows=None) -> torch.Tensor:
        c = self.unpack(rows)
        sh = torch.tensor([3, 2, 1, 0], device=c.device, dtype=torch.uint8)
        b = (c.unsqueeze(-1) >> sh) & 1
        return b.reshape(c.shape[0], -1).to(torch.float64) * 2.0 - 1.0

    @property
    def bit_cost(self) -> int:
        return self.num_tokens * self.num_groups * SUBVECTOR_DIM


@dataclass(frozen=True, eq=False)
class Codebook:
    """codebook.py:93-113."""
    centroids: torch.Tensor

    def __post_init__(self) -> None:
        s = tuple(self.centroids.shape)
        if len(s) != 3 or s[1] != CODEBOOK_SIZE or s[2] != SUBVECTOR_DIM:
            raise ValueError(f"centroids must have shape (G, {CODEBOOK_SIZE}, {SUBVECTOR_DIM}), got {s}")

    @property
    def num_groups(self) -> int:
        return int(self.centroids.shape[0])


def sign_pattern_vectors() -> torch.Tensor:
    """codebook.py:39-47."""
    c = torch.arange(CODEBOOK_SIZE, device=_dev())
    sh = torch.tensor([3, 2, 1, 0], device=c.device)
    return ((c[:, None] >> sh) & 1).to(torch.float64) * 2.0 - 1.0


def _zero_stats(D: int):
    z = torch.zeros(D, dtype=torch.float64, device=_dev())
    return z, z.clone()


def encode_keys(keys_norm) -> SignCodeMatrix:
    """codebook.py:116-125."""
    K = _as_matrix(keys_norm, "keys_norm", keep_dtype=True)
    L, D = K.shape
    if D < SUBVECTOR_DIM or D % SUBVECTOR_DIM != 0:
        raise ValueError(f"channel count {D} must be a positive multiple of {SUBVECTOR_DIM}")
    mu, al = _zero_stats(D)
    r = _encode(K, K, bits=0, group=4, siq=0, what=2, mu=mu, alpha=al, want_codes=True)
    return SignCodeMatrix(packed=r["codes"], num_tokens=L, num_groups=D // 4)


def encode_sign_code(subvector) -> int:
    """codebook.py:29-36."""
    v = _tensor(subvector)
    if tuple(v.shape) != (SUBVECTOR_DIM,):
        raise ValueError(f"subvector must have shape ({SUBVECTOR_DIM},), got {tuple(v.shape)}")
    if not bool(torch.isfinite(v).all()):
        raise ValueError("subvector contains non-finite entries")
    return int(encode_keys(v[None]).unpack()[0, 0])


def build_codebook(keys_norm, codes: SignCodeMatrix) -> Codebook:
    """codebook.py:128-160 (fixed-order float64 partial sums; centroids match the
    reference's to ~1e-15 relative and their float32 roundings bit for bit)."""
    K = _as_matrix(keys_norm, "keys_norm", keep_dtype=True)
    L, D = K.shape
    G = D // SUBVECTOR_DIM
    if D % SUBVECTOR_DIM != 0 or codes.num_tokens != L or codes.num_groups != G:
        raise ValueError(f"codes describe {codes.num_tokens}x{codes.num_groups} groups, keys are {L}x{D}")
    mu, al = _zero_stats(D)
    r = _encode(K, K, bits=0, group=4, siq=0, what=2, mu=mu, alpha=al, codes_in=codes.packed.contiguous())
    tally("codebook_subvector_reads", L * G)
    return Codebook(centroids=r["cent"])


# ============================================================================ quantizer
@dataclass(frozen=True)
class QuantConfig:
    """quantizer.py:36-49."""
    bits: int = 2
    group_size: int = 32

    def __post_init__(self) -> None:
        if self.bits not in PACKABLE_BITS:
            raise ValueError(f"bits must be one of {PACKABLE_BITS}, got {self.bits}")
        if self.group_size < 1:
            raise ValueError(f"group_size must be positive, got {self.group_size}")

    @property
    def levels(self) -> int:
        return (1 << self.bits) - 1


@dataclass(frozen=True, eq=False)
class QuantizedTensor:
    """quantizer.py:52-94 (device tensors)."""
    packed: torch.Tensor
    scales: torch.Tensor
    zeros: torch.Tensor
    bits: int
    group_size: int
    num_tokens: int
    num_channels: int

    def __post_init__(self) -> None:
        L, D = self.num_tokens, self.num_channels
        ng = D // self.group_size
        if tuple(self.packed.shape) != (L, packed_row_bytes(D, self.bits)):
            raise ValueError(f"packed has shape {tuple(self.packed.shape)}, inconsistent with {L}x{D}")
        if tuple(self.scales.shape) != (L, ng) or tuple(self.zeros.shape) != (L, ng):
            raise ValueError("scales/zeros must have shape (num_tokens, num_groups)")
        if self.scales.dtype != torch.float16 or self.zeros.dtype != torch.float16:
            raise ValueError("scales/zeros must be float16")

    @property
    def num_groups(self) -> int:
        return self.num_channels // self.group_size

    def codes(self, rows=None) -> torch.Tensor:
        p = self.packed if rows is None else self.packed[_rows(rows, self.num_tokens)]
        return _unpack(p, self.bits, self.num_channels)

    @property
    def code_bits(self) -> int:
        return self.bits * self.num_tokens * self.num_channels

    @property
    def param_bits(self) -> int:
        return 2 * PARAM_BITS * self.num_tokens * self.num_groups


def _check_group(D: int, cfg: QuantConfig) -> None:
    if D % cfg.group_size != 0:
        raise ValueError(f"channel count {D} not divisible by group_size {cfg.group_size}")
    if cfg.group_size > 128 or cfg.group_size & (cfg.group_size - 1) or cfg.group_size < 4:
        raise NotImplementedError("group_size must be a power of two in [4, 128]")


def quantize_values(values, config: QuantConfig) -> QuantizedTensor:
    """quantizer.py:106-140."""
    V = _as_matrix(values, "values", keep_dtype=True)
    L, D = V.shape
    _check_group(D, config)
    if D % 4:
        raise NotImplementedError("channel count must be a multiple of 4")
    mu, al = _zero_stats(D)
    r = _encode(V, V, bits=config.bits, group=config.group_size, siq=0, what=2, mu=mu, alpha=al, want_v=True)
    L_.raise_status(r["status"], "values")
    return QuantizedTensor(r["vq"], r["vs"], r["vz"], config.bits, config.group_size, L, D)


def _planes_args(kq, vq, codes, alpha, bits, gs, siq, kfull=None, vfull=None):
    return (L_.ptr(codes), L_.ptr(kq.packed if kq else None), L_.ptr(kq.scales if kq else None),
            L_.ptr(kq.zeros if kq else None), L_.ptr(vq.packed if vq else None), L_.ptr(vq.scales if vq else None),
            L_.ptr(vq.zeros if vq else None), L_.ptr(kfull), L_.ptr(vfull), L_.ptr(alpha), bits, gs, siq)


def dequantize_values(q: QuantizedTensor, rows=None) -> torch.Tensor:
    """quantizer.py:143-152."""
    r = torch.arange(q.num_tokens, device=_dev()) if rows is None else _rows(rows, q.num_tokens)
    out = torch.empty(r.numel(), q.num_channels, dtype=torch.float64, device=_dev())
    tally("dequant_rows", r.numel())
    if r.numel():
        L_.call("sikv_dequant_rows", *_planes_args(None, q, None, None, q.bits, q.group_size, 0), 1, q.num_tokens,
                q.num_channels, L_.ptr(r), r.numel(), 0, L_.ptr(out), L_.stream())
    return out


def quantize_key_magnitudes(keys_norm, alpha, config: QuantConfig) -> QuantizedTensor:
    """quantizer.py:155-170."""
    K = _as_matrix(keys_norm, "keys_norm", keep_dtype=True)
    a = _tensor(alpha)
    if tuple(a.shape) != (K.shape[1],):
        raise ValueError(f"alpha must have shape ({K.shape[1]},), got {tuple(a.shape)}")
    L, D = K.shape
    _check_group(D, config)
    if D % 4:
        raise NotImplementedError("channel count must be a multiple of 4")
    mu = torch.zeros(D, dtype=torch.float64, device=_dev())
    r = _encode(K, K, bits=config.bits, group=config.group_size, siq=1, what=2, mu=mu, alpha=a.contiguous(),
                want_k=True)
    s = int(r["status"].item())
    if s & 2:
        raise ValueError("alpha does not dominate |keys_norm|; stats were computed elsewhere")
    L_.raise_status(r["status"], "keys_norm")
    return QuantizedTensor(r["kq"], r["ks"], r["kz"], config.bits, config.group_size, L, D)


def dequantize_keys(q: QuantizedTensor, alpha, signs: SignCodeMatrix, rows=None) -> torch.Tensor:
    """quantizer.py:173-184."""
    a = _tensor(alpha)
    if tuple(a.shape) != (q.num_channels,):
        raise ValueError(f"alpha must have shape ({q.num_channels},), got {tuple(a.shape)}")
    if signs.num_tokens != q.num_tokens or signs.num_groups * 4 != q.num_channels:
        raise ValueError(f"sign codes describe {signs.num_tokens}x{signs.num_groups * 4}, "
                         f"quantized tensor is {q.num_tokens}x{q.num_channels}")
    r = torch.arange(q.num_tokens, device=_dev()) if rows is None else _rows(rows, q.num_tokens)
    out = torch.empty(r.numel(), q.num_channels, dtype=torch.float64, device=_dev())
    tally("dequant_rows", r.numel())
    if r.numel():
        L_.call("sikv_dequant_rows", *_planes_args(q, q, signs.packed, a.contiguous(), q.bits, q.group_size, 1),
                1, q.num_tokens, q.num_channels, L_.ptr(r), r.numel(), 1, L_.ptr(out), L_.stream())
    return out


# ============================================================================ retrieval
@dataclass(frozen=True, eq=False)
class LookupTable:
    """retrieval.py:31-43."""
    table: torch.Tensor

    def __post_init__(self) -> None:
        if self.table.dim() != 2 or self.table.shape[1] != CODEBOOK_SIZE:
            raise ValueError(f"table must have shape (G, {CODEBOOK_SIZE}), got {tuple(self.table.shape)}")

    @property
    def num_groups(self) -> int:
        return int(self.table.shape[0])


def build_lut(q, codebook: Codebook) -> LookupTable:
    """retrieval.py:46-51 (float64, the reference's einsum pairing)."""
    G = codebook.num_groups
    qq = _as_query(q, dim=G * SUBVECTOR_DIM)
    out = torch.empty(G, 16, dtype=torch.float64, device=qq.device)
    L_.call("sikv_build_lut_f64", L_.ptr(qq), L_.ptr(codebook.centroids.contiguous()), 1, G, 0, L_.ptr(out),
            L_.stream())
    return LookupTable(table=out)


def build_sign_lut(q, num_groups: int) -> LookupTable:
    """retrieval.py:54-62."""
    qq = _as_query(q, dim=num_groups * SUBVECTOR_DIM)
    out = torch.empty(num_groups, 16, dtype=torch.float64, device=qq.device)
    L_.call("sikv_build_lut_f64", L_.ptr(qq), None, 1, num_groups, 1, L_.ptr(out), L_.stream())
    return LookupTable(table=out)


def score_tokens(lut: LookupTable, codes: SignCodeMatrix) -> torch.Tensor:
    """retrieval.py:65-77 (float64, numpy's pairwise summation order)."""
    if codes.num_groups != lut.num_groups:
        raise ValueError(f"codes have {codes.num_groups} groups, lookup table has {lut.num_groups}")
    L, G = codes.num_tokens, codes.num_groups
    out = torch.empty(L, dtype=torch.float64, device=_dev())
    if L:
        L_.call("sikv_score_f64", L_.ptr(lut.table.contiguous()), L_.ptr(codes.packed), 1, G, L, L_.ptr(out),
                L_.stream())
    tally("lut_lookups", L * G)
    tally("lut_adds", L * (G - 1) if G else 0)
    tally("score_muls", 0)
    return out


def dense_scores(q, keys_norm) -> torch.Tensor:
    """retrieval.py:80-89: the exact q . K'^T oracle (a cuBLAS float64 GEMV)."""
    K = _tensor(keys_norm)
    if K.dim() != 2:
        raise ValueError(f"keys_norm must be 2-D, got shape {tuple(K.shape)}")
    qq = _as_query(q, dim=K.shape[1])
    L, D = K.shape
    tally("dense_muls", L * D)
    tally("dense_adds", L * (D - 1) if D else 0)
    return K @ qq


@dataclass(frozen=True, eq=False)
class TokenSelection:
    """retrieval.py:92-113."""
    indices: torch.Tensor
    sink_count: int
    recent_count: int
    dynamic_count: int
    _valid: bool = field(default=False, repr=False)   # made by top_k_select: indices known in range

    def __post_init__(self) -> None:
        if self.indices.dim() != 1:
            raise ValueError("indices must be 1-D")
        if self.sink_count + self.recent_count + self.dynamic_count != self.indices.shape[0]:
            raise ValueError("breakdown counts do not sum to the selection size")

    def __len__(self) -> int:
        return int(self.indices.shape[0])


def _as_index_set(indices, length: int, name: str):
    """retrieval.py:116-124: (device index set or None, host copy or None).  Host inputs are
    checked and deduplicated on the host and not uploaded (the caller uploads what it needs)."""
    if isinstance(indices, torch.Tensor):
        idx = torch.unique(indices.to(_dev()).to(torch.int64).reshape(-1))
        if _DEVICE_CHECKS and idx.numel() and (int(idx.min()) < 0 or int(idx.max()) >= length):
            raise ValueError(f"{name} indices out of range [0, {length})")
        return idx, None
    h = np.unique(np.asarray(indices if isinstance(indices, np.ndarray) else sorted(indices), dtype=np.int64))
    if h.size and (h[0] < 0 or h[-1] >= length):
        raise ValueError(f"{name} indices out of range [0, {length})")
    return None, h


def top_k_select(scores, k: int, sink=(), recent=()) -> TokenSelection:
    """retrieval.py:127-161: exact top-k on the GPU, ties -> lower index."""
    s = _tensor(scores)
    if s.dim() != 1:
        raise ValueError(f"scores must be 1-D, got shape {tuple(s.shape)}")
    if k < 0:
        raise ValueError(f"k must be non-negative, got {k}")
    L = int(s.shape[0])
    sink_idx, sink_h = _as_index_set(sink, L, "sink")
    recent_idx, recent_h = _as_index_set(recent, L, "recent")
    if sink_h is not None and recent_h is not None:
        # host sets: union on the host, one upload
        forced = torch.as_tensor(np.union1d(sink_h, recent_h).astype(np.int32), device=_dev())
    else:
        if sink_idx is None:
            sink_idx = torch.as_tensor(sink_h, device=_dev())
        if recent_idx is None:
            recent_idx = torch.as_tensor(recent_h, device=_dev())
        forced = torch.unique(torch.cat([sink_idx, recent_idx])).to(torch.int32).contiguous()
    F = int(forced.numel())
    keff = min(k, L - F)
    n = F + max(keff, 0)
    out = torch.empty(max(n, 1), dtype=torch.int32, device=_dev())
    counts = torch.zeros(2, dtype=torch.int32, device=_dev())
    if L:
        ws = _ws(L_.lib().sikv_topk_workspace_bytes(1, L))
        L_.call("sikv_topk", L_.ptr(s.contiguous()), 0, 1, L, L_.ptr(forced) if F else None, F, k, L_.ptr(ws),
                L_.ptr(out), max(n, 1), L_.ptr(counts), L_.stream())
    n_sink = int(sink_h.size) if sink_h is not None else int(sink_idx.numel())
    if sink_h is not None and recent_h is not None:
        recent_only = int(np.isin(recent_h, sink_h, invert=True).sum()) if recent_h.size else 0
    elif not recent_idx.numel():
        recent_only = 0
    else:
        recent_only = int(torch.isin(recent_idx, sink_idx, invert=True).sum())
    return TokenSelection(indices=out[:n].to(torch.int64), sink_count=n_sink,
                          recent_count=recent_only, dynamic_count=max(keff, 0), _valid=True)


def resolve_dynamic_k(length: int, forced_count: int, budget: int | None = None,
                      sparsity: float | None = None) -> int:
    """retrieval.py:164-181."""
    if (budget is None) == (sparsity is None):
        raise ValueError("exactly one of budget and sparsity must be set")
    if budget is not None:
        if budget < 0:
            raise ValueError(f"budget must be non-negative, got {budget}")
        return max(int(budget) - forced_count, 0)
    if not 0.0 <= sparsity <= 1.0:
        raise ValueError(f"sparsity must be in [0, 1], got {sparsity}")
    target = int(math.floor(sparsity * length + 0.5))
    return max(target - forced_count, 1)


# ============================================================================ cache
@dataclass(frozen=True)
class CacheConfig:
    """cache.py:52-75."""
    bits: int = 2
    group_size: int = 32
    sink_count: int = DEFAULT_SINK_COUNT
    sign_in_quant: bool = True
    sink_pool_width: int = DEFAULT_POOL_WIDTH

    def __post_init__(self) -> None:
        if self.bits not in (1, 2, 4, 8, LOSSLESS_BITS):
            raise ValueError(f"bits must be 1, 2, 4, 8 or {LOSSLESS_BITS}, got {self.bits}")
        if self.sink_count < 0:
            raise ValueError(f"sink_count must be non-negative, got {self.sink_count}")
        if self.sink_pool_width < 1 or self.sink_pool_width % 2 == 0:
            raise ValueError("sink_pool_width must be odd and positive")

    @property
    def lossless(self) -> bool:
        return self.bits == LOSSLESS_BITS


@dataclass(eq=False)
class SelfIndexingCache:
    """One head's compressed cache (cache.py:78-182), planes on the device."""
    config: CacheConfig
    dim: int
    prefill_length: int
    norm: NormalizationState
    codes: SignCodeMatrix
    codebook: Codebook
    key_mag: QuantizedTensor | None
    key_direct: QuantizedTensor | None
    values: QuantizedTensor | None
    kprime_full: torch.Tensor | None
    values_full: torch.Tensor | None
    sink_indices: torch.Tensor
    sink_k: torch.Tensor
    sink_v: torch.Tensor
    _recent_k: torch.Tensor = None
    _recent_v: torch.Tensor = None
    _n_recent: int = 0

    def __post_init__(self) -> None:
        if self._recent_k is None:
            self._recent_k = torch.empty(16, self.dim, dtype=torch.float64, device=_dev())
            self._recent_v = torch.empty(16, self.dim, dtype=torch.float64, device=_dev())

    @property
    def length(self) -> int:
        return self.prefill_length + self._n_recent

    @property
    def recent_count(self) -> int:
        return self._n_recent

    def sink_host(self) -> np.ndarray:
        """The sink indices as a host array (read once: they are fixed at prefill)."""
        h = self.__dict__.get("_sink_h")
        if h is None:
            h = self.sink_indices.cpu().numpy().astype(np.int64)
            self.__dict__["_sink_h"] = h
        return h

    def recent_indices(self) -> torch.Tensor:
        return torch.arange(self.prefill_length, self.length, dtype=torch.int64, device=_dev())

    def forced_indices(self) -> torch.Tensor:
        return torch.unique(torch.cat([self.sink_indices, self.recent_indices()]))

    def _planes(self):
        kq = self.key_mag if self.config.sign_in_quant else self.key_direct
        return _planes_args(kq, self.values, self.codes.packed, self.norm.alpha, self.config.bits,
                            self.config.group_size, int(self.config.sign_in_quant),
                            self.kprime_full, self.values_full)

    def gather(self, indices) -> tuple[torch.Tensor, torch.Tensor]:
        """cache.py:118-158: K' and V rows, dequantising only dynamic rows."""
        idx = _tensor(indices, torch.int64)
        if idx.dim() != 1:
            raise ValueError("indices must be 1-D")
        if idx.numel() and (int(idx.min()) < 0 or int(idx.max()) >= self.length):
            raise ValueError(f"indices out of range [0, {self.length})")
        K = torch.empty(idx.numel(), self.dim, dtype=torch.float64, device=_dev())
        V = torch.empty_like(K)
        rec = idx >= self.prefill_length
        snk = ~rec & torch.isin(idx, self.sink_indices)
        dyn = ~rec & ~snk
        if bool(rec.any()):
            rel = idx[rec] - self.prefill_length
            K[rec] = self._recent_k[rel]
            V[rec] = self._recent_v[rel]
        if bool(snk.any()):
            pos = torch.searchsorted(self.sink_indices, idx[snk])
            K[snk] = self.sink_k[pos]
            V[snk] = self.sink_v[pos]
        if bool(dyn.any()):
            rows = idx[dyn].contiguous()
            n = rows.numel()
            kk = torch.empty(n, self.dim, dtype=torch.float64, device=_dev())
            vv = torch.empty_like(kk)
            tally("dequant_rows", 0 if self.config.lossless else 2 * n)
            L_.call("sikv_dequant_rows", *self._planes(), 1, self.prefill_length, self.dim, L_.ptr(rows), n, 1,
                    L_.ptr(kk), L_.stream())
            L_.call("sikv_dequant_rows", *self._planes(), 1, self.prefill_length, self.dim, L_.ptr(rows), n, 0,
                    L_.ptr(vv), L_.stream())
            K[dyn] = kk
            V[dyn] = vv
        return K, V

    def checksum(self) -> str:
        """cache.py:160-182: SHA-256 over every stored plane."""
        h = hashlib.sha256()
        arrs = [self.norm.mu, self.norm.alpha, self.codes.packed, self.codebook.centroids, self.sink_indices,
                self.sink_k, self.sink_v, self._recent_k[: self._n_recent], self._recent_v[: self._n_recent]]
        for q in (self.key_mag, self.key_direct, self.values):
            if q is not None:
                arrs += [q.packed, q.scales, q.zeros]
        for a in (self.kprime_full, self.values_full):
            if a is not None:
                arrs.append(a)
        for a in arrs:
            h.update(a.contiguous().cpu().numpy().tobytes())
        return h.hexdigest()


def select_sink_tokens(keys_norm, query_window, count: int, pool_width: int = DEFAULT_POOL_WIDTH) -> torch.Tensor:
    """cache.py:185-209: SnapKV-style sinks (snapkv.cu: float64 K' W^T, column softmax, votes,
    edge-replicated max-pool, stable top-count, one C-ABI call)."""
    if count == 0:
        return torch.empty(0, dtype=torch.int64, device=_dev())
    K = _as_matrix(keys_norm, "keys_norm")
    W = _as_matrix(query_window, "query_window")
    if W.shape[1] != K.shape[1]:
        raise ValueError(f"window queries have {W.shape[1]} channels, keys have {K.shape[1]}")
    L, D = K.shape
    if count >= L:
        return torch.arange(L, dtype=torch.int64, device=_dev())
    mu0 = torch.zeros(D, dtype=torch.float64, device=K.device)
    ws = torch.empty(L_.lib().sikv_window_sinks_workspace_bytes(1, L, W.shape[0]), dtype=torch.uint8, device=K.device)
    out = torch.empty(count, dtype=torch.int32, device=K.device)
    L_.call("sikv_window_sinks", L_.ptr(K.contiguous()), L_.IN_F64, 1, L, D, L_.ptr(mu0), L_.ptr(W.contiguous()),
            W.shape[0], count, pool_width, L_.ptr(out), L_.ptr(ws), ws.numel(), L_.stream())
    return out.to(torch.int64)


def prefill(keys, values, query_window=None, config: CacheConfig = CacheConfig()) -> SelfIndexingCache:
    """cache.py:212-271."""
    K = _as_matrix(keys, "keys", keep_dtype=True)
    V = _as_matrix(values, "values", keep_dtype=True)
    if K.shape != V.shape:
        raise ValueError(f"keys and values must match, got {tuple(K.shape)} and {tuple(V.shape)}")
    L, D = K.shape
    if D % 4 != 0:
        raise ValueError(f"channel count {D} must be divisible by 4")
    if not config.lossless and D % config.group_size != 0:
        raise ValueError(f"channel count {D} not divisible by group_size {config.group_size}")
    if V.dtype != K.dtype:            # the reference converts both to float64: never round one down
        wide = torch.promote_types(K.dtype, V.dtype)
        K, V = K.to(wide), V.to(wide)
    bits = 0 if config.lossless else config.bits
    siq = int(config.sign_in_quant)
    r = _encode(K, V, bits=bits, group=config.group_size if bits else 4, siq=siq, what=3, want_codes=True,
                want_k=bits > 0, want_v=bits > 0)
    st = int(r["status"].item())
    if st & 4:
        raise ValueError("keys contains non-finite entries")
    if st & 2:
        raise ValueError("alpha does not dominate |keys_norm|; stats were computed elsewhere")
    if st & 1:
        raise ValueError("group min/max exceed the 16-bit parameter range")
    norm = NormalizationState(mu=r["mu"], alpha=r["alpha"])
    codes = SignCodeMatrix(packed=r["codes"], num_tokens=L, num_groups=D // 4)
    codebook = Codebook(centroids=r["cent"])
    key_mag = key_direct = values_q = kfull = vfull = None
    if config.lossless:
        kfull = apply_normalization(K, norm)
        vfull = V.to(torch.float64).clone()
    else:
        kq = QuantizedTensor(r["kq"], r["ks"], r["kz"], bits, config.group_size, L, D)
        if siq:
            key_mag = kq
        else:
            key_direct = kq
        values_q = QuantizedTensor(r["vq"], r["vs"], r["vz"], bits, config.group_size, L, D)
    if config.sink_count == 0:
        sinks = torch.empty(0, dtype=torch.int64, device=_dev())
    elif query_window is not None:
        sinks = select_sink_tokens(apply_normalization(K, norm), query_window, config.sink_count,
                                   config.sink_pool_width)
    else:
        sinks = torch.arange(min(config.sink_count, L), dtype=torch.int64, device=_dev())
    S = int(sinks.numel())
    sk = torch.empty(S, D, dtype=torch.float64, device=_dev())
    sv = torch.empty_like(sk)
    if S:
        L_.call("sikv_gather_rows", L_.ptr(K), L_.ptr(V), L_.dtype_code(K), 1, L, D,
                L_.ptr(sinks.to(torch.int32).contiguous()), S, L_.ptr(norm.mu), L_.ptr(sk), L_.ptr(sv), 1,
                L_.stream())
    return SelfIndexingCache(config=config, dim=D, prefill_length=L, norm=norm, codes=codes, codebook=codebook,
                             key_mag=key_mag, key_direct=key_direct, values=values_q, kprime_full=kfull,
                             values_full=vfull, sink_indices=sinks, sink_k=sk, sink_v=sv)


def append_token(cache: SelfIndexingCache, k, v) -> None:
    """cache.py:274-287: (k - mu, v) into the recent buffer at full precision."""
    kk = _tensor(k)
    vv = _tensor(v)
    if tuple(kk.shape) != (cache.dim,) or tuple(vv.shape) != (cache.dim,):
        raise ValueError(f"k and v must have shape ({cache.dim},)")
    if not (bool(torch.isfinite(kk).all()) and bool(torch.isfinite(vv).all())):
        raise ValueError("appended token contains non-finite entries")
    n = cache._n_recent
    if n >= cache._recent_k.shape[0]:
        grow = max(16, cache._recent_k.shape[0])
        cache._recent_k = torch.cat([cache._recent_k, torch.empty_like(cache._recent_k[:grow])])
        cache._recent_v = torch.cat([cache._recent_v, torch.empty_like(cache._recent_v[:grow])])
    st = _status()
    L_.call("sikv_append", L_.ptr(kk.contiguous()), L_.ptr(vv.contiguous()), 1, 1, cache.dim, L_.ptr(cache.norm.mu),
            L_.ptr(cache._recent_k), L_.ptr(cache._recent_v), cache._recent_k.shape[0], n, 1, L_.ptr(st),
            L_.stream())
    cache._n_recent = n + 1


def select_tokens(cache: SelfIndexingCache, q, k: int | None = None, budget: int | None = None,
                  sparsity: float | None = None, sign_only: bool = False) -> TokenSelection:
    """cache.py:290-309: LUT -> scores -> recents at -inf -> exact top-k."""
    qq = _as_query(q, dim=cache.dim)
    lut = build_sign_lut(qq, cache.codes.num_groups) if sign_only else build_lut(qq, cache.codebook)
    pre = score_tokens(lut, cache.codes)
    scores = torch.cat([pre, torch.full((cache.recent_count,), -math.inf, dtype=torch.float64, device=_dev())])
    if k is None:
        nforced = int(np.union1d(cache.sink_host(), np.arange(cache.prefill_length, cache.length)).size)
        k = resolve_dynamic_k(cache.length, nforced, budget=budget, sparsity=sparsity)
    elif budget is not None or sparsity is not None:
        raise ValueError("give exactly one of k, budget and sparsity")
    return top_k_select(scores, k, sink=cache.sink_host(), recent=np.arange(cache.prefill_length, cache.length))


# ============================================================================ attention
@dataclass(frozen=True, eq=False)
class AttentionOutput:
    """attention.py:23-26.  weights_checksum: a float, or a 0-d device tensor for outputs of
    sparse_attention (no host sync; float(...) reads it)."""
    out: torch.Tensor
    weights_checksum: float


@dataclass(frozen=True, eq=False)
class ErrorReport:
    cosine_sim: float
    rel_l2: float


def _softmax_attend(q, K, V) -> AttentionOutput:
    logits = (K @ q) / math.sqrt(K.shape[1])
    w = torch.exp(logits - logits.max())
    w = w / w.sum()
    return AttentionOutput(out=w @ V, weights_checksum=float(w.sum()))


def exact_attention(q, keys, values) -> AttentionOutput:
    """attention.py:42-49: full attention oracle (cuBLAS float64)."""
    K = _as_matrix(keys, "keys")
    V = _as_matrix(values, "values")
    if K.shape != V.shape:
        raise ValueError(f"keys and values must match, got {tuple(K.shape)} and {tuple(V.shape)}")
    return _softmax_attend(_as_query(q, dim=K.shape[1]), K, V)


def sparse_attention(q, selection: TokenSelection, cache: SelfIndexingCache) -> AttentionOutput:
    """attention.py:52-62: float64 attention over the selection, gathering and
    dequantising only the selected rows on the GPU."""
    if len(selection) == 0:
        raise ValueError("selection is empty")
    qq = _as_query(q, dim=cache.dim)
    si = selection.indices
    idx = (si.to(_dev()) if isinstance(si, torch.Tensor) else
           torch.as_tensor(np.asarray(si, dtype=np.int64), device=_dev())).to(torch.int32).contiguous()
    n = int(idx.numel())
    if not selection._valid and n and _DEVICE_CHECKS and (int(idx.min()) < 0 or int(idx.max()) >= cache.length):
        raise ValueError(f"indices out of range [0, {cache.length})")
    cnt = torch.full((1,), n, dtype=torch.int32, device=_dev())
    ws = torch.empty((L_.lib().sikv_attend_f64_workspace_bytes(1, 1, n) + 7) // 8, dtype=torch.float64,
                     device=_dev())
    out = torch.empty(cache.dim, dtype=torch.float64, device=_dev())
    chk = torch.empty((), dtype=torch.float64, device=_dev())
    S = int(cache.sink_indices.numel())
    # dequantised rows = the selection's dynamic (non-forced) rows (cache.py:118-158)
    ndyn = selection.dynamic_count if selection._valid else \
        int(np.isin(idx.cpu().numpy(), np.union1d(cache.sink_host(), np.arange(cache.prefill_length, cache.length)),
                    invert=True).sum())
    tally("dequant_rows", 0 if cache.config.lossless else 2 * ndyn)
    L_.call("sikv_attend_f64", *cache._planes(), 1, cache.prefill_length, cache.dim, L_.ptr(qq), 1, L_.ptr(idx),
            L_.ptr(cnt), n, L_.ptr(cache.sink_indices.to(torch.int32).contiguous()) if S else None, S,
            L_.ptr(cache.sink_k), L_.ptr(cache.sink_v), L_.ptr(cache._recent_k), L_.ptr(cache._recent_v),
            cache._recent_k.shape[0], L_.ptr(ws), L_.ptr(out), L_.ptr(chk), L_.stream())
    # the checksum stays on the device (a 0-d tensor, read when used): no host sync here
    return AttentionOutput(out=out, weights_checksum=chk)


def output_error(a: AttentionOutput, b: AttentionOutput) -> ErrorReport:
    """attention.py:65-86."""
    x = _tensor(a.out)
    y = _tensor(b.out)
    if x.shape != y.shape:
        raise ValueError(f"outputs must have equal shape, got {tuple(x.shape)} and {tuple(y.shape)}")
    nx, ny = float(torch.linalg.norm(x)), float(torch.linalg.norm(y))
    if nx == 0.0 and ny == 0.0:
        cos = 1.0
    elif nx == 0.0 or ny == 0.0:
        cos = 0.0
    else:
        cos = float(torch.dot(x, y)) / (nx * ny)
    d = float(torch.linalg.norm(x - y))
    rel = 0.0 if d == 0.0 else (math.inf if ny == 0.0 else d / ny)
    return ErrorReport(cosine_sim=cos, rel_l2=rel)


# ============================================================================ accounting
@dataclass(frozen=True)
class MemoryReport:
    """cache.py:312-336."""
    sign_bits: int
    payload_bits: int
    param_bits: int
    fixed_bits: int
    recent_bits: int
    total_bits: int
    baseline_bits: int
    savings_fraction: float

    @property
    def variable_bits(self) -> int:
        return self.sign_bits + self.payload_bits + self.param_bits

    @property
    def compression_ratio(self) -> float:
        return self.baseline_bits / self.variable_bits


def memory_report_from_shapes(tokens: int, dim: int, bits: int = 2, group_size: int = 32,
                              sink_count: int = DEFAULT_SINK_COUNT, recent_count: int = 0) -> MemoryReport:
    """cache.py:339-371 (integer shape arithmetic)."""
    if tokens < 1 or dim < 4 or dim % 4 != 0:
        raise ValueError(f"invalid shape {tokens}x{dim}: dim must be a positive multiple of 4")
    if bits != LOSSLESS_BITS and dim % group_size != 0:
        raise ValueError(f"channel count {dim} not divisible by group_size {group_size}")
    L, D = tokens, dim
    sign = L * D
    payload = 2 * bits * L * D
    param = 0 if bits == LOSSLESS_BITS else 2 * (D // group_size) * L * 2 * PARAM_PRECISION_BITS
    fixed = (D // 4) * 16 * 4 * FULL_PRECISION_BITS + 2 * D * FULL_PRECISION_BITS + \
        sink_count * (2 * D * FULL_PRECISION_BITS + INDEX_BITS)
    recent = recent_count * 2 * D * FULL_PRECISION_BITS
    base = 2 * L * D * FULL_PRECISION_BITS
    var = sign + payload + param
    return MemoryReport(sign, payload, param, fixed, recent, var + fixed + recent, base, 1.0 - var / base)


def memory_report(cache: SelfIndexingCache) -> MemoryReport:
    """cache.py:374-383."""
    return memory_report_from_shapes(tokens=cache.prefill_length, dim=cache.dim, bits=cache.config.bits,
                                     group_size=cache.config.group_size, sink_count=int(cache.sink_indices.numel()),
                                     recent_count=cache.recent_count)
