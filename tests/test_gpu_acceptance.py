"""The reference's acceptance criteria on the B200 fused path, plus the certified comparison of
fused selections with the float64 reference selection.

  * c02 ADC exactness (/root/reference/pkg/tests/test_acceptance.py:62-91): on centroid-aligned
    caches the fused float32 scoring kernel equals exact q.K'^T, 1000 queries;
  * c09 recall dominance (test_acceptance.py:213-233): recall@160 of the fused decode step's
    selections (k = 160, no sinks, L = 4096, 50 seeds x 4 queries) >= 0.43 (the reference's
    committed floor) and >= 10x uniform, and above sign-only scoring;
  * certified selection: fused selections equal the float64 reference sets except for tokens
    whose float64 score sits within 2B of the k-th (B = restate32.score_error_bound).
"""

import numpy as np
import pytest
import torch

import paper_2603_14224_b200 as sk
from oracle import restate32 as R
from oracle import sikv_oracle as O
from paper_2603_14224_b200 import _lib
from paper_2603_14224_b200 import batch as B
from paper_2603_14224_b200.synth import gen_unit

pytestmark = pytest.mark.gpu


def _patterns():
    c = np.arange(16)
    return np.stack([np.where((c >> (3 - i)) & 1, 1.0, -1.0) for i in range(4)], axis=1)   # sign(0) = +1 code bits


def test_c02_adc_exactness_fused_scoring():
    rng = np.random.default_rng(2024)
    L, D = 1024, 128
    G = D // 4
    templates = np.abs(rng.standard_normal((G, 16, 4))) * _patterns()[None]
    choice = rng.integers(0, 16, size=(L, G))
    Kp = templates[np.arange(G)[None, :], choice].reshape(L, D)
    dev = torch.device("cuda", 0)
    K = torch.tensor(Kp, device=dev)
    # encode K' as given (mu = 0: the reference test builds codes / codebook on K' directly)
    mu = torch.zeros(D, dtype=torch.float64, device=dev)
    alpha = K.abs().amax(dim=0)
    cb = B.empty_batch(1, L, sink_count=0, keep_reference=True, device=dev)
    ws = torch.empty(_lib.lib().sikv_encode_workspace_bytes(1, L, D), dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    r = cb.ref
    _lib.call("sikv_encode", _lib.ptr(K), _lib.ptr(K), _lib.IN_F64, 1, L, D, 2, 32, 1, 2, None, _lib.ptr(mu),
              _lib.ptr(alpha), _lib.ptr(cb.mu32), _lib.ptr(cb.alpha32), _lib.ptr(cb.cent64), _lib.ptr(cb.cent32),
              _lib.ptr(r["codes"]), _lib.ptr(r["kq"]), _lib.ptr(r["ks"]), _lib.ptr(r["kz"]), _lib.ptr(r["vq"]),
              _lib.ptr(r["vs"]), _lib.ptr(r["vz"]), _lib.ptr(cb.signs), _lib.ptr(cb.recs), _lib.ptr(ws), ws.numel(),
              _lib.ptr(st), _lib.stream())
    _lib.raise_status(st, "keys")
    np.testing.assert_array_equal(r["codes"][0].cpu().numpy(), O.pack(choice, 4))   # every cluster is pure
    n = 1000
    Q = rng.standard_normal((n, D))
    big = B.subset(cb, [0] * n)
    s = B.score_fast(big, torch.tensor(Q[:, None, :], dtype=torch.float32, device=dev)).cpu().numpy()
    exact = Q.astype(np.float32).astype(np.float64) @ Kp.T
    worst = float((np.abs(s - exact).max(axis=1) / np.abs(exact).max(axis=1)).max())
    print(f"[c02 fused] worst relative score error {worst:.2e} over {n} queries")
    assert worst <= 1e-5


def test_c09_recall_dominance_fused():
    seeds, nq, L, k = 50, 4, 4096, 160
    dev = torch.device("cuda", 0)
    units = [gen_unit(L, 128, nq, s, bf16=False) for s in range(seeds)]
    K = torch.tensor(np.stack([u.keys for u in units]), device=dev)
    V = torch.tensor(np.stack([u.values for u in units]), device=dev)
    cb = B.prefill_batch(K, V, sink_count=0)
    big = B.subset(cb, np.repeat(np.arange(seeds), nq))            # one unit per (seed, query), Gq = 1
    q = torch.tensor(np.concatenate([u.queries for u in units])[:, None, :], device=dev)
    res = B.decode_step(big, q, k, with_selection=True)
    sel = res.selection.cpu().numpy()
    assert (res.counts.cpu().numpy() == k).all()
    full, sign_only, rand = [], [], []
    rng = np.random.default_rng(9)
    for s, u in enumerate(units):
        Kp = u.keys - u.keys.mean(axis=0)
        cache = sk.prefill(u.keys, u.values, None, sk.CacheConfig(sink_count=0))
        for j in range(nq):
            qv = u.queries[j]
            exact_top = set(np.argsort(-(Kp @ qv), kind="stable")[:k].tolist())
            full.append(len(exact_top.intersection(sel[s * nq + j].tolist())) / k)
            so = sk.select_tokens(cache, qv, k=k, sign_only=True).indices.cpu().numpy()
            sign_only.append(len(exact_top.intersection(so.tolist())) / k)
            rand.append(len(exact_top.intersection(rng.choice(L, size=k, replace=False).tolist())) / k)
    mean_recall = float(np.mean(full))
    uniform = k / L
    print(f"[c09 fused] recall@{k} {mean_recall:.4f} ({mean_recall / uniform:.1f}x uniform), "
          f"sign-only {np.mean(sign_only):.4f}")
    assert mean_recall >= 10 * uniform
    assert mean_recall >= 0.43                    # the reference's committed regression floor
    assert np.mean(full) > np.mean(sign_only)
    assert np.mean(rand) == pytest.approx(uniform, abs=0.01)


@pytest.mark.parametrize("L,k,gq,kernel", [(4096, 256, 4, 1), (32768, 2048, 4, 4), (8192, 1024, 7, 4),
                                          (131072, 4096, 4, 3)])
def test_selection_certified_against_float64_reference(L, k, gq, kernel):
    """Fused (float32) selections vs the reference's float64 select_tokens(cache, sum_h q_h, k):
    identical sets unless the float64 k-th boundary gap is within the certified float32 error
    bound.  The measured overlap is printed."""
    seeds = [900 + i for i in range(4 if L <= 32768 else 2)]
    units = [gen_unit(L, 128, gq, s) for s in seeds]
    dev = torch.device("cuda", 0)
    K = torch.tensor(np.stack([u.keys for u in units]), dtype=torch.bfloat16, device=dev)
    V = torch.tensor(np.stack([u.values for u in units]), dtype=torch.bfloat16, device=dev)
    cb = B.prefill_batch(K, V, sink_count=64)
    q = torch.tensor(np.stack([u.queries[:gq] for u in units]), dtype=torch.float32, device=dev)
    res = B.decode_step(cb, q, k, with_selection=True, kernel=kernel)
    overlaps = []
    for i, u in enumerate(units):
        c = O.prefill(u.keys, u.values, sink_count=64)
        got = res.selection[i, : int(res.counts[i])].cpu().numpy()
        ok, ndiff, gap, bound = R.certified_selection_check(c, u.queries[:gq].astype(np.float32), k, got)
        overlaps.append(1.0 - ndiff / (2 * len(got)))
        assert ok, (i, ndiff, gap, bound)
    print(f"[certified] L={L} k={k} gq={gq}: overlap with float64 sets {min(overlaps):.6f} (min over units)")
