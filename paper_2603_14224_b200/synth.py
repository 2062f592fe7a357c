"""Synthetic K/V/Q workloads (harness, not the hot path).

Two generators of the same distribution as the reference harness
(``harness/synth.py:34-80``): per-channel lognormal scales with a +-0.5 sigma
offset for keys, standard normal values, and queries that are 50% a rescaled key
row plus 0.25 noise, 50% standard normal.

* :func:`gen_unit` — numpy, draws in exactly the reference generator's order, so
  a seed gives the same arrays as ``sikv.harness.synth.gen_synthetic`` (checked
  against a recorded hash in ``tests/golden``).  Used for parity tests.
* :func:`gen_units_torch` — the same distribution drawn on the GPU with a seeded
  Philox ``torch.Generator``, for bench-sized inputs (C2 is 4096 units x 32K
  tokens, 68 GB of raw bf16 K/V, generated layer by layer and discarded after
  encoding).

All values are rounded to bfloat16 (the model dtype), so the float64 reference
sees exactly the numbers the GPU sees.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bfloat16 (ties to even) via float32, return float64."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


@dataclass
class Unit:
    keys: np.ndarray        # (L, D) float64, bf16-exact
    values: np.ndarray      # (L, D)
    queries: np.ndarray     # (n, D)
    window: np.ndarray      # (w, D)
    paired: np.ndarray      # (n,) row a query was drawn from, or -1


def gen_unit(tokens: int, dim: int, queries: int, seed: int, *, offset: float = 0.5,
             correlated: float = 0.5, noise: float = 0.25, window: int = 32,
             spread: float = 0.5, bf16: bool = True) -> Unit:
    rng = np.random.default_rng(seed)
    scale = np.exp(spread * rng.standard_normal(dim))
    shift = offset * scale * np.where(rng.random(dim) < 0.5, -1.0, 1.0)
    K = rng.standard_normal((tokens, dim)) * scale + shift
    V = rng.standard_normal((tokens, dim))

    def draw(n):
        out = np.empty((n, dim))
        row_of = np.full(n, -1, dtype=np.int64)
        for i in range(n):
            if rng.random() < correlated:
                r = int(rng.integers(tokens))
                out[i] = K[r] * (np.sqrt(dim) / np.linalg.norm(K[r]))
                out[i] += noise * rng.standard_normal(dim)
                row_of[i] = r
            else:
                out[i] = rng.standard_normal(dim)
        return out, row_of

    Q, paired = draw(queries)
    W, _ = draw(window)
    if bf16:
        K, V, Q, W = (bf16_round(a) for a in (K, V, Q, W))
    return Unit(K, V, Q, W, paired)


def gen_units_torch(units: int, tokens: int, dim: int, seed: int, device, *,
                    offset: float = 0.5, spread: float = 0.5, dtype=None):
    """(units, tokens, dim) bf16 K and V on ``device``; per-unit channel scales/offsets."""
    import torch
    dtype = dtype or torch.bfloat16
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    scale = torch.exp(spread * torch.randn(units, 1, dim, generator=g, device=device))
    sign = torch.where(torch.rand(units, 1, dim, generator=g, device=device) < 0.5, -1.0, 1.0)
    K = torch.randn(units, tokens, dim, generator=g, device=device)
    K.mul_(scale).add_(offset * scale * sign)
    V = torch.randn(units, tokens, dim, generator=g, device=device)
    return K.to(dtype), V.to(dtype)


def gen_units_by_id(ids, tokens: int, dim: int, seed: int, device, *, offset: float = 0.5,
                    spread: float = 0.5, dtype=None):
    """(len(ids), tokens, dim) bf16 K and V: unit i drawn from its own Philox stream seeded
    with ``seed + ids[i]``, so a unit's content depends only on its global id (a sharded
    rank regenerates exactly the units of the single-GPU run)."""
    import torch
    dtype = dtype or torch.bfloat16
    ids = [int(i) for i in ids]
    K = torch.empty(len(ids), tokens, dim, device=device, dtype=dtype)
    V = torch.empty_like(K)
    for j, gid in enumerate(ids):
        k, v = gen_units_torch(1, tokens, dim, seed + gid, device, offset=offset, spread=spread, dtype=dtype)
        K[j].copy_(k[0])
        V[j].copy_(v[0])
    return K, V


def gen_queries_by_id(keys, ids, heads: int, seed: int, **kw):
    """(len(ids), heads, dim) queries, unit i from the stream ``seed + ids[i]``."""
    import torch
    return torch.cat([gen_queries_torch(keys[j:j + 1], heads, seed + int(gid), **kw) for j, gid in enumerate(ids)])


def gen_queries_torch(keys, heads: int, seed: int, *, correlated: float = 0.5,
                      noise: float = 0.25):
    """(units, heads, dim) queries: per head, half are a rescaled key row + noise."""
    import torch
    U, L, D = keys.shape
    dev = keys.device
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    rows = torch.randint(0, L, (U, heads), generator=g, device=dev)
    base = keys.float()[torch.arange(U, device=dev)[:, None], rows]
    base = base * (D ** 0.5) / base.norm(dim=-1, keepdim=True).clamp_min(1e-30)
    base = base + noise * torch.randn(U, heads, D, generator=g, device=dev)
    rnd = torch.randn(U, heads, D, generator=g, device=dev)
    pick = torch.rand(U, heads, 1, generator=g, device=dev) < correlated
    return torch.where(pick, base, rnd).to(torch.bfloat16)
