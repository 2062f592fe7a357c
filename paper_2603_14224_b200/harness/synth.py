"""Synthetic K/V/query workloads (reference: sikv/harness/synth.py:18-80).

``gen_synthetic`` returns the reference's workload record; the arrays are drawn by
:func:`paper_2603_14224_b200.synth.gen_unit`, which consumes the same numpy Generator stream in
the same order (checked against the reference's recorded hash in tests/golden), so a seed
gives byte-identical arrays."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..synth import gen_unit


@dataclass(frozen=True, eq=False)
class SyntheticWorkload:
    keys: np.ndarray
    values: np.ndarray
    queries: np.ndarray
    window: np.ndarray
    paired_rows: np.ndarray

    @property
    def tokens(self) -> int:
        return int(self.keys.shape[0])

    @property
    def dim(self) -> int:
        return int(self.keys.shape[1])


def gen_synthetic(tokens: int, dim: int, query_count: int, seed: int, channel_offset: float = 0.5,
                  correlated_fraction: float = 0.5, query_noise: float = 0.25, window: int = 32,
                  channel_scale_spread: float = 0.5) -> SyntheticWorkload:
    if tokens < 1 or dim < 1:
        raise ValueError(f"tokens and dim must be positive, got {tokens}, {dim}")
    if not 0.0 <= correlated_fraction <= 1.0:
        raise ValueError(f"correlated_fraction must be in [0, 1], got {correlated_fraction}")
    u = gen_unit(tokens, dim, query_count, seed, offset=channel_offset, correlated=correlated_fraction,
                 noise=query_noise, window=window, spread=channel_scale_spread, bf16=False)
    return SyntheticWorkload(keys=u.keys, values=u.values, queries=u.queries, window=u.window,
                             paired_rows=u.paired)
