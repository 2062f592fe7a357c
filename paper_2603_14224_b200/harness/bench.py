"""Benchmark runners (reference: sikv/harness/bench.py:1-293): retrieval recall, attention
fidelity and operation-count micro benchmarks, one flat JSON-able record each.

Every runner builds its cache and selections with this package's GPU implementation (through
the host-array API, :mod:`paper_2603_14224_b200.hostapi`).  ``run_recall_bench_fused`` also
measures recall of the batched fused decode path (``batch.decode_step``: float32 scoring,
exact top-k) over every query of the workload at once.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from .. import hostapi as sk
from ..api import tally
from .synth import SyntheticWorkload, gen_synthetic

ABLATIONS = ("full", "no_sign_quant", "sign_only_retrieval", "no_sink")
RECORD_KEYS = ("bench", "seed", "L", "D", "bits", "budget", "ablation", "recall_at_k", "cosine_mean",
               "cosine_std", "bits_per_token", "savings_fraction", "wall_ms", "op_counts")
SUBVECTOR = 4


@dataclass(frozen=True)
class BenchConfig:
    tokens: int = 4096
    dim: int = 128
    seed: int = 0
    bits: int = 2
    group_size: int = 32
    sink_count: int = 64
    budget: int | None = None
    sparsity: float | None = None
    ablation: str = "full"
    query_count: int = 16
    channel_offset: float = 0.5
    correlated_fraction: float = 0.5
    query_noise: float = 0.25
    window: int = 32

    def __post_init__(self) -> None:
        if (self.budget is None) == (self.sparsity is None):
            raise ValueError("exactly one of budget and sparsity must be set")
        if self.ablation not in ABLATIONS:
            raise ValueError(f"ablation must be one of {ABLATIONS}, got {self.ablation!r}")

    @property
    def target_tokens(self) -> int:
        """Kept tokens in total (forced ones included)."""
        return self.budget if self.budget is not None else int(np.floor(self.sparsity * self.tokens + 0.5))


def make_workload(cfg: BenchConfig) -> SyntheticWorkload:
    return gen_synthetic(cfg.tokens, cfg.dim, cfg.query_count, cfg.seed, channel_offset=cfg.channel_offset,
                         correlated_fraction=cfg.correlated_fraction, query_noise=cfg.query_noise,
                         window=cfg.window)


def cache_config_for(cfg: BenchConfig, ablation: str | None = None):
    ab = cfg.ablation if ablation is None else ablation
    return sk.CacheConfig(bits=cfg.bits, group_size=cfg.group_size,
                          sink_count=0 if ab == "no_sink" else cfg.sink_count,
                          sign_in_quant=ab != "no_sign_quant")


def build_cache(cfg: BenchConfig, workload: SyntheticWorkload, ablation: str | None = None):
    return sk.prefill(workload.keys, workload.values, query_window=workload.window,
                      config=cache_config_for(cfg, ablation))


def make_record(bench: str, cfg: BenchConfig, **metrics) -> dict:
    extra = set(metrics) - set(RECORD_KEYS)
    if extra:
        raise ValueError(f"unknown record keys: {sorted(extra)}")
    rec = {key: None for key in RECORD_KEYS}
    rec.update(bench=bench, seed=cfg.seed, L=cfg.tokens, D=cfg.dim, bits=cfg.bits, budget=cfg.target_tokens,
               ablation=cfg.ablation, **metrics)
    return rec


def _dynamic_k(cfg: BenchConfig, cache) -> int:
    forced = int(cache.forced_indices().size)
    k = sk.resolve_dynamic_k(cache.length, forced, budget=cfg.budget, sparsity=cfg.sparsity)
    room = cache.length - forced
    if k > room:
        warnings.warn(f"budget exceeds cache length; clamping dynamic k from {k} to {room}")
        k = room
    return k


def _exact_top(q, keys_norm, candidates: np.ndarray, k: int) -> set:
    exact = sk.dense_scores(q, keys_norm)
    return set(candidates[np.argsort(-exact[candidates], kind="stable")[:k]].tolist())


def run_recall_bench(cfg: BenchConfig, workload: SyntheticWorkload | None = None) -> list[dict]:
    """Recall@k of compressed-domain selection against the exact-score top-k, plus a uniform
    random baseline over the same candidates (expected ~ k / L)."""
    work = make_workload(cfg) if workload is None else workload
    cache = build_cache(cfg, work)
    keys_norm = sk.apply_normalization(work.keys, cache.norm)
    forced = cache.forced_indices()
    candidates = np.setdiff1d(np.arange(cache.length), forced)
    k = _dynamic_k(cfg, cache)
    if k < 1:
        raise ValueError("budget leaves no dynamic tokens; recall@k is undefined")
    sign_only = cfg.ablation == "sign_only_retrieval"
    rng = np.random.default_rng((cfg.seed, 0xBA5E))
    hits, rand_hits = [], []
    t0 = time.perf_counter()
    for q in work.queries:
        top = _exact_top(q, keys_norm, candidates, k)
        sel = sk.select_tokens(cache, q, k=k, sign_only=sign_only)
        hits.append(len(top.intersection(np.setdiff1d(sel.indices, forced).tolist())) / k)
        rand_hits.append(len(top.intersection(rng.choice(candidates, size=k, replace=False).tolist())) / k)
    wall = (time.perf_counter() - t0) * 1e3
    rep = sk.memory_report(cache)
    method = make_record("recall", cfg, recall_at_k=float(np.mean(hits)),
                         bits_per_token=rep.variable_bits // cache.prefill_length,
                         savings_fraction=rep.savings_fraction, wall_ms=wall)
    baseline = dict(method, ablation="random_baseline", recall_at_k=float(np.mean(rand_hits)))
    return [method, baseline]


def run_recall_bench_fused(cfg: BenchConfig, workloads: list[SyntheticWorkload]) -> dict:
    """Recall@k of the batched fused decode path (one unit per (workload, query), Gq = 1,
    first-S sinks, bits 2 / group 32): float32 LUT scoring + exact top-k on the GPU."""
    from .. import batch as B
    if cfg.bits != 2 or cfg.group_size != 32 or cfg.dim != 128 or cfg.ablation != "full":
        raise ValueError("the fused path is D = 128, 2-bit, group 32, full method")
    dev = torch.device("cuda", torch.cuda.current_device())
    K = torch.tensor(np.stack([w.keys for w in workloads]), device=dev)
    V = torch.tensor(np.stack([w.values for w in workloads]), device=dev)
    cb = B.prefill_batch(K, V, sink_count=cfg.sink_count)
    nq = workloads[0].queries.shape[0]
    big = B.subset(cb, np.repeat(np.arange(len(workloads)), nq))
    q = torch.tensor(np.concatenate([w.queries for w in workloads])[:, None, :], device=dev)
    S = cb.sinks
    k = max(cfg.target_tokens - S, 0)
    t0 = time.perf_counter()
    res = B.decode_step(big, q, k, with_selection=True)
    sel = res.selection.cpu().numpy()
    wall = (time.perf_counter() - t0) * 1e3
    hits = []
    for i, w in enumerate(workloads):
        kn = w.keys - w.keys.mean(axis=0)
        cand = np.arange(S, w.tokens)
        for j in range(nq):
            top = set(cand[np.argsort(-(kn[cand] @ w.queries[j]), kind="stable")[:k]].tolist())
            hits.append(len(top.intersection(sel[i * nq + j, S:S + k].tolist())) / k)
    return make_record("recall", cfg, recall_at_k=float(np.mean(hits)), bits_per_token=896 if cfg.dim == 128 else None,
                       savings_fraction=0.78125, wall_ms=wall)


def run_attention_bench(cfg: BenchConfig, workload: SyntheticWorkload | None = None) -> dict:
    """Cosine similarity of sparse attention against exact attention over the whole cache."""
    work = make_workload(cfg) if workload is None else workload
    cache = build_cache(cfg, work)
    keys_norm = sk.apply_normalization(work.keys, cache.norm)
    k = _dynamic_k(cfg, cache)
    sign_only = cfg.ablation == "sign_only_retrieval"
    cos = []
    t0 = time.perf_counter()
    for q in work.queries:
        sel = sk.select_tokens(cache, q, k=k, sign_only=sign_only)
        approx = sk.sparse_attention(q, sel, cache)
        cos.append(sk.output_error(approx, sk.exact_attention(q, keys_norm, work.values)).cosine_sim)
    wall = (time.perf_counter() - t0) * 1e3
    rep = sk.memory_report(cache)
    return make_record("attn", cfg, cosine_mean=float(np.mean(cos)), cosine_std=float(np.std(cos)),
                       bits_per_token=rep.variable_bits // cache.prefill_length,
                       savings_fraction=rep.savings_fraction, wall_ms=wall)


def kmeans_codebook(keys_norm, iterations: int = 20, seed: int = 0) -> np.ndarray:
    """Lloyd's k-means per 4-channel group (the iterative comparator of the one-pass sign
    codebook), on the GPU in float64; every iteration rescans all L x G subvectors."""
    X = np.asarray(keys_norm, dtype=np.float64)
    L, D = X.shape
    G = D // SUBVECTOR
    dev = torch.device("cuda", torch.cuda.current_device())
    sub = torch.tensor(X.reshape(L, G, SUBVECTOR), device=dev)
    start = np.random.default_rng(seed).choice(L, size=16, replace=L < 16)
    cent = sub[torch.as_tensor(start, device=dev)].permute(1, 0, 2).contiguous()        # (G, 16, 4)
    for _ in range(iterations):
        d2 = ((sub[:, :, None, :] - cent[None]) ** 2).sum(-1)                           # (L, G, 16)
        assign = d2.argmin(dim=2)
        tally("kmeans_subvector_reads", L * G)
        # cluster sums as a one-hot contraction (deterministic, unlike scatter-add atomics)
        onehot = torch.nn.functional.one_hot(assign, 16).to(torch.float64)             # (L, G, 16)
        sums = torch.einsum("lgk,lgd->gkd", onehot, sub)
        cnt = onehot.sum(dim=0)[:, :, None]
        cent = torch.where(cnt > 0, sums / cnt.clamp_min(1), cent)
    return cent.cpu().numpy()


def run_micro_bench(cfg: BenchConfig, workload: SyntheticWorkload | None = None) -> dict:
    """Operation counts and wall-clock ratios of the three hot stages: LUT vs dense scoring,
    the one-pass codebook vs 20 k-means iterations, sparse vs full attention."""
    work = make_workload(cfg) if workload is None else workload
    cache = build_cache(cfg, work)
    keys_norm = sk.apply_normalization(work.keys, cache.norm)
    k = _dynamic_k(cfg, cache)
    q0 = work.queries[0]
    with sk.collect() as lut_ops:
        sk.select_tokens(cache, q0, k=k)
    with sk.collect() as dense_ops:
        sk.dense_scores(q0, keys_norm)

    def timed(fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) * 1e3

    with sk.collect() as build_ops:
        onepass = timed(lambda: sk.build_codebook(keys_norm, sk.encode_keys(keys_norm)))
    with sk.collect() as km_ops:
        kmeans = timed(lambda: kmeans_codebook(keys_norm, iterations=20, seed=cfg.seed))
    sels = [sk.select_tokens(cache, q, k=k) for q in work.queries]
    sparse = timed(lambda: [sk.sparse_attention(q, s, cache) for q, s in zip(work.queries, sels)])
    full = timed(lambda: [sk.exact_attention(q, keys_norm, work.values) for q in work.queries])
    rep = sk.memory_report(cache)
    return make_record(
        "micro", cfg, bits_per_token=rep.variable_bits // cache.prefill_length,
        savings_fraction=rep.savings_fraction,
        wall_ms={"onepass_build": onepass, "kmeans20_build": kmeans, "sparse_attention": sparse,
                 "full_attention": full},
        op_counts={"lut_lookups": lut_ops.lut_lookups, "lut_adds": lut_ops.lut_adds,
                   "score_muls": lut_ops.score_muls, "dense_muls": dense_ops.dense_muls,
                   "dense_adds": dense_ops.dense_adds, "onepass_subvector_reads": build_ops.codebook_subvector_reads,
                   "kmeans_subvector_reads": km_ops.kmeans_subvector_reads})
