"""GPU parity of the batched fast path (encoder planes, scores, top-k sets, attention).

Checked against the CPU oracle (oracle/sikv_oracle.py, pinned to the reference's golden
vectors) and the float32 scoring restatement (oracle/restate32.py):
  * encoder planes, mu, alpha: bit-exact; float32 centroids == fl32(oracle float64);
  * fast-path scores: bit-exact vs restate32;
  * selections: exact index sets vs restate32 + the reference's top_k_select rule;
  * attention: rel-L2 and cosine vs the float64 oracle on the same selection within the bars
    of tests/tolerances.py (set from the measured maxima; fp16 mma operands, fp32 accumulation).
"""

import numpy as np
import pytest
import torch

from oracle import restate32 as R
from oracle import sikv_oracle as O
from paper_2603_14224_b200 import batch as B
from paper_2603_14224_b200.synth import gen_unit

from .fastlayout import records_to_reference, unrotate_signs

pytestmark = pytest.mark.gpu

from .tolerances import ATT_COS, att_rel_l2


def make(L, seeds, gq=4, sinks=64, appends=0, dtype=torch.bfloat16):
    units = [gen_unit(L, 128, gq + appends, s) for s in seeds]
    K = torch.tensor(np.stack([u.keys for u in units]), dtype=dtype, device="cuda")
    V = torch.tensor(np.stack([u.values for u in units]), dtype=dtype, device="cuda")
    cb = B.prefill_batch(K, V, sink_count=sinks, recent_capacity=max(appends, 1), keep_reference=True)
    oc = [O.prefill(u.keys, u.values, sink_count=sinks) for u in units]
    for a in range(appends):
        kk = np.stack([u.queries[gq + a] * 0.5 for u in units])
        vv = np.stack([u.queries[gq + a][::-1].copy() for u in units])
        B.append_batch(cb, torch.tensor(kk, device="cuda"), torch.tensor(vv, device="cuda"))
        for i, c in enumerate(oc):
            O.append(c, kk[i], vv[i])
    q = torch.tensor(np.stack([u.queries[:gq] for u in units]), dtype=torch.float32, device="cuda")
    return units, cb, oc, q


@pytest.fixture(scope="module")
def c1():
    return make(4096, [100, 101, 102, 103])


def test_encoder_planes_bit_exact(c1, golden):
    units, cb, oc, _ = c1
    meta, arr = golden
    torch.cuda.synchronize()
    for i, c in enumerate(oc):
        np.testing.assert_array_equal(cb.mu64[i].cpu().numpy(), c.mu)
        np.testing.assert_array_equal(cb.alpha64[i].cpu().numpy(), c.alpha)
        np.testing.assert_array_equal(cb.ref["codes"][i].cpu().numpy(), c.packed_codes)
        np.testing.assert_array_equal(cb.ref["kq"][i].cpu().numpy(), c.kmag.packed)
        np.testing.assert_array_equal(cb.ref["ks"][i].cpu().numpy(), c.kmag.scales)
        np.testing.assert_array_equal(cb.ref["kz"][i].cpu().numpy(), c.kmag.zeros)
        np.testing.assert_array_equal(cb.ref["vq"][i].cpu().numpy(), c.vq.packed)
        np.testing.assert_array_equal(cb.ref["vs"][i].cpu().numpy(), c.vq.scales)
        np.testing.assert_array_equal(cb.ref["vz"][i].cpu().numpy(), c.vq.zeros)
        np.testing.assert_array_equal(cb.cent32[i].cpu().numpy(), c.centroids.astype(np.float32))
        np.testing.assert_allclose(cb.cent64[i].cpu().numpy(), c.centroids, rtol=1e-12, atol=1e-15)
        # golden (reference itself) for the first unit
    np.testing.assert_array_equal(cb.mu64[0].cpu().numpy(), arr["c1_u0/mu"])


def test_fast_layout_matches_reference_planes(c1):
    units, cb, oc, _ = c1
    for i, c in enumerate(oc):
        np.testing.assert_array_equal(unrotate_signs(cb.signs[i].cpu().numpy()), c.packed_codes)
        kc, vc, kpar, vpar, neg = records_to_reference(cb.recs[i].cpu().numpy())
        np.testing.assert_array_equal(kc, c.kmag.codes())
        np.testing.assert_array_equal(vc, c.vq.codes())
        np.testing.assert_array_equal(kpar[:, :, 0], c.kmag.scales.view(np.uint16))
        np.testing.assert_array_equal(kpar[:, :, 1], c.kmag.zeros.view(np.uint16))
        np.testing.assert_array_equal(vpar[:, :, 0], c.vq.scales.view(np.uint16))
        np.testing.assert_array_equal(vpar[:, :, 1], c.vq.zeros.view(np.uint16))
        np.testing.assert_array_equal(neg, O.sign_plane(c.codes) < 0)


def test_sink_rows(c1):
    units, cb, oc, _ = c1
    for i, c in enumerate(oc):
        np.testing.assert_array_equal(cb.sink_idx[i].cpu().numpy(), c.sinks)
        np.testing.assert_array_equal(cb.sink_k[i].cpu().numpy(), c.sink_k.astype(np.float32))
        np.testing.assert_array_equal(cb.sink_v[i].cpu().numpy(), c.sink_v.astype(np.float32))


def test_fast_scores_bit_exact(c1):
    units, cb, oc, q = c1
    s = B.score_fast(cb, q).cpu().numpy()
    for i, c in enumerate(oc):
        qbar = R.group_query(q[i].cpu().numpy())
        ref = R.scores32(R.lut32(qbar, c.centroids), c.packed_codes)
        np.testing.assert_array_equal(s[i], ref)


def _check_decode(units, cb, oc, q, k, **kw):
    res = B.decode_step(cb, q, k, with_selection=True, with_lse=True, with_diag=True, **kw)
    torch.cuda.synchronize()
    sel = res.selection.cpu().numpy()
    cnt = res.counts.cpu().numpy()
    out = res.out.cpu().numpy()
    for i, c in enumerate(oc):
        qs = q[i].cpu().numpy().astype(np.float64)
        idx, ns, nr, nd = R.select32(c, q[i].cpu().numpy(), k)
        assert cnt[i] == len(idx)
        np.testing.assert_array_equal(sel[i, :cnt[i]], idx)
        tol = att_rel_l2(c.L)
        for h in range(qs.shape[0]):
            ref = O.sparse_attention(qs[h], idx, c)
            assert O.rel_l2(out[i, h], ref) <= tol, (i, h, O.rel_l2(out[i, h], ref))
            assert O.cosine(out[i, h], ref) >= ATT_COS
    return res


KERNELS = [1, 3, 4]  # one CTA per unit / split across a cluster / two kernels


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("k", [256, 0, 1, 4032, 5000])
def test_decode_selection_and_attention(c1, k, kernel):
    units, cb, oc, q = c1
    _check_decode(units, cb, oc, q, k, kernel=kernel)


def test_decode_matches_reference_selection(c1, golden):
    """Against the real reference's float64 select_tokens(cache, sum q, k) (golden)."""
    units, cb, oc, q = c1
    meta, arr = golden
    res = B.decode_step(cb, q, 256, with_selection=True)
    sel = res.selection[0, :res.counts[0]].cpu().numpy()
    ref = arr["c1_u0/sel"]
    np.testing.assert_array_equal(sel, ref)          # measured: identical to the reference's set


@pytest.mark.parametrize("kernel", KERNELS)
def test_decode_fallback_path(c1, kernel):
    """A tiny candidate buffer forces the exact multi-pass rescoring path."""
    units, cb, oc, q = c1
    # the split kernel's buffer is per CTA: ask for more than one CTA's share can hold
    k, cap = (3500, 40) if kernel == 3 else (256, 300)
    res = _check_decode(units, cb, oc, q, k, cap=cap, kernel=kernel)
    assert (res.diag.cpu().numpy() & 4).all()


@pytest.fixture(scope="module")
def c32k():
    return make(32768, [200, 201, 202])


@pytest.mark.parametrize("kernel", KERNELS)
def test_decode_sampled_threshold_32k(c32k, kernel):
    units, cb, oc, q = c32k
    res = _check_decode(units, cb, oc, q, 2048, kernel=kernel)
    d = res.diag.cpu().numpy()
    assert ((d & 3) == 3).all() and not (d & 4).any()


def _assert_order_close(a, b, lse_a=None, lse_b=None):
    """Same selection, attention split over a different number of warps: the outputs agree to
    the fp16 rounding of P against each warp's own running max."""
    rel = (a - b).norm(dim=-1) / b.norm(dim=-1)
    assert rel.max().item() <= 1e-3, rel.max().item()
    if lse_a is not None:
        torch.testing.assert_close(lse_a, lse_b, rtol=1e-5, atol=1e-4)


def test_kernels_agree(c32k):
    """The two-kernel path selects bit-identically to the one-CTA path; its attention CTAs have
    4 warps instead of 8, so its outputs agree to fp16 P rounding."""
    units, cb, oc, q = c32k
    kernel = 4
    r1 = B.decode_step(cb, q, 2048, with_selection=True, with_lse=True, kernel=1)
    r2 = B.decode_step(cb, q, 2048, with_selection=True, with_lse=True, kernel=kernel)
    assert torch.equal(r1.selection, r2.selection) and torch.equal(r1.counts, r2.counts)
    _assert_order_close(r2.out, r1.out, r2.lse, r1.lse)
    # without the sorted selection the dynamic rows come straight from the candidate segments,
    # in the same order
    r3 = B.decode_step(cb, q, 2048, with_lse=True, kernel=kernel)
    assert torch.equal(r2.out, r3.out) and torch.equal(r2.lse, r3.lse)


def test_split_kernel_matches_single_cta(c32k):
    """The cluster-split kernel selects exactly what the one-CTA kernel selects."""
    units, cb, oc, q = c32k
    r1 = B.decode_step(cb, q, 2048, with_selection=True, with_lse=True, with_diag=True, kernel=1)
    r3 = B.decode_step(cb, q, 2048, with_selection=True, with_lse=True, with_diag=True, kernel=3)
    assert torch.equal(r1.selection, r3.selection) and torch.equal(r1.counts, r3.counts)
    assert (r3.diag.cpu().numpy() & 8).all()
    # P is rounded to fp16 against each CTA's own running max, so outputs agree to the fp16
    # probability rounding (both are also checked against the float64 oracle above)
    rel = (r3.out - r1.out).norm(dim=-1) / r1.out.norm(dim=-1)
    assert rel.max().item() <= 1e-3, rel.max().item()
    torch.testing.assert_close(r3.lse, r1.lse, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("kernel", KERNELS)
def test_decode_with_appends_and_gq7(kernel):
    units, cb, oc, q = make(2048, [11, 12], gq=7, appends=3)
    _check_decode(units, cb, oc, q, 128, kernel=kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_decode_no_sinks_fp32_inputs(kernel):
    units, cb, oc, q = make(1000, [5, 6, 7], gq=2, sinks=0, dtype=torch.float32)
    _check_decode(units, cb, oc, q, 100, kernel=kernel)


def test_two_kernel_path_many_units():
    """More units than CTAs: every persistent CTA loops over several units."""
    units = [gen_unit(1024, 128, 4, 500 + i) for i in range(2)]
    K = torch.tensor(np.stack([u.keys for u in units]), dtype=torch.bfloat16, device="cuda")
    V = torch.tensor(np.stack([u.values for u in units]), dtype=torch.bfloat16, device="cuda")
    reps = 400
    cb = B.prefill_batch(K.repeat(reps, 1, 1), V.repeat(reps, 1, 1), sink_count=64)
    q = torch.tensor(np.stack([u.queries[:4] for u in units]), dtype=torch.float32, device="cuda").repeat(reps, 1, 1)
    r1 = B.decode_step(cb, q, 100, with_selection=True, kernel=1)
    r2 = B.decode_step(cb, q, 100, with_selection=True, kernel=4)
    assert torch.equal(r1.selection, r2.selection)
    _assert_order_close(r2.out, r1.out)
    assert torch.equal(r2.out[0::2], r2.out[0:1].expand(reps, -1, -1))
    r0 = B.decode_step(cb, q, 100, with_selection=True)        # auto: two kernels at 800 units
    assert torch.equal(r2.selection, r0.selection) and torch.equal(r2.out, r0.out)


def test_decode_ties_lowest_index_first():
    """Repeated key rows give exactly tied scores; the k boundary must keep the lowest
    indices (stable argsort, retrieval.py:149), in both the sampled and the exact path."""
    rng = np.random.default_rng(3)
    L = 9000
    base = gen_unit(97, 128, 4, 31)
    reps = np.concatenate([base.keys] * (L // 97 + 1))[:L]
    V = rng.standard_normal((L, 128))
    from paper_2603_14224_b200.synth import bf16_round
    V = bf16_round(V)
    K_t = torch.tensor(reps[None], dtype=torch.bfloat16, device="cuda")
    V_t = torch.tensor(V[None], dtype=torch.bfloat16, device="cuda")
    cb = B.prefill_batch(K_t, V_t, sink_count=64)
    c = O.prefill(reps, V, sink_count=64)
    q = torch.tensor(base.queries[None, :4], dtype=torch.float32, device="cuda")
    for k, cap, kern in ((500, 0, 1), (500, 200, 1), (333, 0, 1), (500, 0, 3),
                         (500, 200, 3), (333, 0, 3), (500, 0, 4), (500, 200, 4), (333, 0, 4)):
        res = B.decode_step(cb, q, k, cap=cap, with_selection=True, kernel=kern)
        idx = R.select32(c, base.queries[:4].astype(np.float32), k)[0]
        got = res.selection[0, : res.counts[0]].cpu().numpy()
        np.testing.assert_array_equal(got, idx)


@pytest.mark.parametrize("gq", [1, 8])
@pytest.mark.parametrize("kernel", [1, 4])
def test_decode_gqa_extremes(gq, kernel):
    """GQA group sizes 1 and 8: the two-kernel path stages Gq x 128 queries per unit and the
    attention packs Gq heads into the mma N dimension (8 = no padding)."""
    units, cb, oc, q = make(4096, [300, 301], gq=gq)
    _check_decode(units, cb, oc, q, 512, kernel=kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_recent_ring_growth_per_unit_counts(kernel):
    """cache.py:274-287 / 302: hundreds of appends through the batched ring, growing it by
    doubling from 0 rows, with per-unit counts (each append goes to a different subset of
    units); every recent row is force-included and the selection / attention match the oracle
    replaying the same appends per unit."""
    rng = np.random.default_rng(7)
    units, cb, oc, q = make(2048, [40, 41, 42], gq=4, appends=0)
    U = len(units)
    counts = np.zeros(U, dtype=int)
    for step in range(300):
        ids = np.flatnonzero(rng.random(U) < 0.7)
        if step % 50 == 0:
            ids = np.arange(U)
        if ids.size == 0:
            continue
        kk = rng.standard_normal((ids.size, 128)) * 2.0
        vv = rng.standard_normal((ids.size, 128))
        B.append_batch(cb, torch.tensor(kk, device="cuda"), torch.tensor(vv, device="cuda"),
                       units=torch.tensor(ids), check=(step % 100 == 0))
        for j, i in enumerate(ids):
            O.append(oc[i], kk[j], vv[j])
        counts[ids] += 1
    assert cb.recent_capacity >= counts.max()
    np.testing.assert_array_equal(cb.recent_n.cpu().numpy(), counts)
    res = _check_decode(units, cb, oc, q, 128, kernel=kernel)
    for i in range(U):
        got = res.selection[i, : res.counts[i]].cpu().numpy()
        assert np.array_equal(got[-counts[i]:], 2048 + np.arange(counts[i]))


@pytest.mark.parametrize("kernel", KERNELS)
def test_recent_rows_beyond_prefill_alpha(kernel):
    """A recent key far outside the prefill range (|K'| / alpha ~ 1e6 in a near-constant
    channel) stays finite and exact to tolerance: its fragment row carries a power-of-two
    scale instead of overflowing fp16."""
    units = [gen_unit(1024, 128, 4, s) for s in (60, 61)]
    K = np.stack([u.keys for u in units])
    K[:, :, 5] = 0.25                                   # constant channel: alpha = 0
    K[:, :, 9] = 0.25 + 1e-3 * np.sign(np.random.default_rng(1).standard_normal(K.shape[:2]))
    V = np.stack([u.values for u in units])
    cb = B.prefill_batch(torch.tensor(K, device="cuda"), torch.tensor(V, device="cuda"), sink_count=64)
    oc = [O.prefill(K[i], V[i], sink_count=64) for i in range(2)]
    kk = np.stack([u.queries[0] for u in units])
    kk[:, 9] += 500.0                                   # |K'| / alpha ~ 5e5 in channel 9
    vv = np.stack([u.values[3] for u in units])
    B.append_batch(cb, torch.tensor(kk, device="cuda"), torch.tensor(vv, device="cuda"))
    for i in range(2):
        O.append(oc[i], kk[i], vv[i])
    q = torch.tensor(np.stack([u.queries[:4] for u in units]) * 1e-3, dtype=torch.float32, device="cuda")
    res = _check_decode(units, cb, oc, q, 100, kernel=kernel)
    assert bool(torch.isfinite(res.out).all())


def test_append_rejects_non_finite_and_checks_buffers(c1):
    units, cb, oc, q = make(1024, [70], gq=4)
    bad = torch.zeros(1, 128, dtype=torch.float64, device="cuda")
    bad[0, 3] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        B.append_batch(cb, bad, torch.zeros(1, 128, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="sel_buf"):
        B.decode_step(cb, q, 16, with_selection=True, sel_buf=torch.empty(1, 8, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="out must"):
        B.decode_step(cb, q, 16, out=torch.empty(1, 4, 128, dtype=torch.float64, device="cuda"))


# ---------------------------------------------------------------- SnapKV window sinks
def make_window(L, seeds, gq=4, sinks=64, wn=32, pool=7):
    units = [gen_unit(L, 128, gq, s, window=wn) for s in seeds]
    K = torch.tensor(np.stack([u.keys for u in units]), dtype=torch.bfloat16, device="cuda")
    V = torch.tensor(np.stack([u.values for u in units]), dtype=torch.bfloat16, device="cuda")
    W = torch.tensor(np.stack([u.window for u in units]), device="cuda")
    cb = B.prefill_batch(K, V, sink_count=sinks, window=W, pool_width=pool)
    oc = []
    for u in units:
        c = O.prefill(u.keys, u.values, sink_count=sinks)
        if sinks < L:
            c.sinks = O.window_sinks(u.keys - c.mu, u.window, sinks, pool)
            c.sink_k = (u.keys - c.mu)[c.sinks].copy()
            c.sink_v = u.values[c.sinks].copy()
        oc.append(c)
    q = torch.tensor(np.stack([u.queries[:gq] for u in units]), dtype=torch.float32, device="cuda")
    return units, cb, oc, q


def test_window_sinks_golden_win_1k(golden):
    """The batched GPU window sinks equal the real reference's select_sink_tokens (golden
    win_1k: L = 1024, 32 window queries, 64 sinks, pool 7)."""
    meta, _ = golden
    rec = meta["win_1k"]
    units, cb, oc, q = make_window(rec["L"], [rec["seed"]])
    assert cb.sink_idx[0].cpu().tolist() == rec["sink_indices"]


@pytest.mark.parametrize("L,sinks,wn,pool", [(4096, 64, 32, 7), (3001, 100, 8, 6), (20000, 64, 40, 1), (700, 650, 32, 7)])
def test_window_sinks_match_oracle(L, sinks, wn, pool):
    units, cb, oc, q = make_window(L, [300, 301, 302], sinks=sinks, wn=wn, pool=pool)
    for i, c in enumerate(oc):
        np.testing.assert_array_equal(cb.sink_idx[i].cpu().numpy(), c.sinks)
        np.testing.assert_array_equal(cb.sink_k[i].cpu().numpy(), c.sink_k.astype(np.float32))


@pytest.mark.parametrize("kernel", KERNELS)
def test_decode_with_window_sinks(kernel):
    """Non-prefix sinks (SnapKV) through every fused decode kernel: forced-bit exclusion
    beyond the first block, forced fragments of scattered rows, sorted selection."""
    units, cb, oc, q = make_window(32768 if kernel == 3 else 8192, [310, 311], sinks=64)
    assert int(cb.sink_idx[:, -1].min()) > 64                   # scattered, not a prefix
    _check_decode(units, cb, oc, q, 512, kernel=kernel)


# ---------------------------------------------------------------- fast-path variants (§8f3)
def make_variant(L, seeds, bits, siq, gq=4, sinks=64):
    units = [gen_unit(L, 128, gq, s) for s in seeds]
    K = torch.tensor(np.stack([u.keys for u in units]), dtype=torch.bfloat16, device="cuda")
    V = torch.tensor(np.stack([u.values for u in units]), dtype=torch.bfloat16, device="cuda")
    cb = B.prefill_batch(K, V, sink_count=sinks, keep_reference=True, bits=bits, sign_in_quant=siq)
    oc = [O.prefill(u.keys, u.values, bits=bits, sink_count=sinks, sign_in_quant=siq) for u in units]
    q = torch.tensor(np.stack([u.queries[:gq] for u in units]), dtype=torch.float32, device="cuda")
    return units, cb, oc, q


@pytest.mark.parametrize("bits,siq", [(2, False), (1, True), (1, False)])
@pytest.mark.parametrize("kernel", KERNELS)
def test_fast_path_variants(bits, siq, kernel):
    """bits 1 / 2 x sign-in-quant / direct keys (cache.py:236-244) on the fused path: reference
    planes bit-exact, fast records decode to them, selections exact, attention in tolerance."""
    L = 32768 if kernel == 3 else 4096
    units, cb, oc, q = make_variant(L, [500, 501], bits, siq)
    for i, c in enumerate(oc):
        plane = c.kmag if siq else c.kdirect
        np.testing.assert_array_equal(cb.ref["kq"][i].cpu().numpy(), plane.packed)
        np.testing.assert_array_equal(cb.ref["ks"][i].cpu().numpy(), plane.scales)
        np.testing.assert_array_equal(cb.ref["kz"][i].cpu().numpy(), plane.zeros)
        np.testing.assert_array_equal(cb.ref["vq"][i].cpu().numpy(), c.vq.packed)
        kc, vc, kpar, vpar, neg = records_to_reference(cb.recs[i].cpu().numpy())
        np.testing.assert_array_equal(kc, plane.codes())
        np.testing.assert_array_equal(vc, c.vq.codes())
        np.testing.assert_array_equal(kpar[:, :, 1], plane.zeros.view(np.uint16))
        np.testing.assert_array_equal(neg, (O.sign_plane(c.codes) < 0) if siq else np.zeros_like(neg))
    _check_decode(units, cb, oc, q, 256, kernel=kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_sign_only_lut(kernel, golden):
    """select_tokens(..., sign_only=True) (retrieval.py:54-62) on the fused path: exact vs the
    float32 sign-LUT restatement, certified vs the float64 reference sets, and the golden
    sparsity-0.05 sign-only selection of c1_u0 (k = 205 - 64 = 141)."""
    L = 32768 if kernel == 3 else 4096
    seeds = [100, 101] if L == 4096 else [610, 611]
    units, cb, oc, q = make_variant(L, seeds, 2, True)
    res = B.decode_step(cb, q, 141, with_selection=True, kernel=kernel, sign_only=True)
    for i, c in enumerate(oc):
        got = res.selection[i, : int(res.counts[i])].cpu().numpy()
        np.testing.assert_array_equal(got, R.select32(c, q[i].cpu().numpy(), 141, sign_only=True)[0])
        ok, nd, gap, bound = R.certified_selection_check(c, q[i].cpu().numpy(), 141, got, sign_only=True)
        assert ok, (nd, gap, bound)
        for h in range(4):
            ref = O.sparse_attention(q[i, h].cpu().numpy().astype(np.float64), got, c)
            assert O.rel_l2(res.out[i, h].cpu().numpy(), ref) <= att_rel_l2(L)
    if L == 4096:
        meta, _ = golden
        np.testing.assert_array_equal(res.selection[0, : int(res.counts[0])].cpu().numpy(),
                                      meta["c1_u0"]["sparsity_signonly_sel"])
    s = B.score_fast(cb, q, sign_only=True).cpu().numpy()
    for i, c in enumerate(oc):
        qbar = R.group_query(q[i].cpu().numpy())
        np.testing.assert_array_equal(s[i], R.scores32(R.sign_lut32(qbar, 32), c.packed_codes))


@pytest.mark.parametrize("kernel", KERNELS)
def test_per_q_head_policy(kernel):
    """Per-q-head policy: each query head's own select_tokens(cache, q_h, k) (cache.py:290-309)
    and attention, through unit_map (query unit -> cache unit) on every fused kernel."""
    L = 32768 if kernel == 3 else 4096
    units, cb, oc, q = make_variant(L, [700, 701], 2, True, gq=4)
    res = B.decode_step_per_head(cb, q, 200, with_selection=True, kernel=kernel)
    for i, c in enumerate(oc):
        for h in range(4):
            r = i * 4 + h
            idx = R.select32(c, q[i, h:h + 1].cpu().numpy(), 200)[0]
            np.testing.assert_array_equal(res.selection[r, : int(res.counts[r])].cpu().numpy(), idx)
            ref = O.sparse_attention(q[i, h].cpu().numpy().astype(np.float64), idx, c)
            assert O.rel_l2(res.out[i, h].cpu().numpy(), ref) <= att_rel_l2(L)


def test_sixteen_bit_records():
    """bits = 16 on the fast path ("Ours (16 bits)", cache.py:236-238 at model precision):
    sign plane and codebook as the 2-bit path, records = fp16 K' / alpha-hat and V in fragment
    order (bit-exact to the float64 values rounded once), selections exact vs restate32,
    attention vs the float64 lossless oracle; the two-kernel path runs it (1 / 3 refuse)."""
    from .fastlayout import records16_to_arrays
    units = [gen_unit(L, 128, 4, s) for L, s in ((4096, 800), (4096, 801))]
    K = torch.tensor(np.stack([u.keys for u in units]), dtype=torch.bfloat16, device="cuda")
    V = torch.tensor(np.stack([u.values for u in units]), dtype=torch.bfloat16, device="cuda")
    cb = B.prefill_batch(K, V, sink_count=64, bits=16)
    oc = [O.prefill(u.keys, u.values, bits=16, sink_count=64) for u in units]
    q = torch.tensor(np.stack([u.queries[:4] for u in units]), dtype=torch.float32, device="cuda")
    for i, (u, c) in enumerate(zip(units, oc)):
        np.testing.assert_array_equal(unrotate_signs(cb.signs[i].cpu().numpy()), c.packed_codes)
        kh, vh = records16_to_arrays(cb.recs[i].cpu().numpy())
        ahat = cb.alpha32[i].cpu().numpy().astype(np.float64)
        ahat[ahat == 0] = 1.0
        np.testing.assert_array_equal(kh, ((u.keys - c.mu) / ahat).astype(np.float16))
        np.testing.assert_array_equal(vh, u.values.astype(np.float16))
    for kern in (0, 4):
        _check_decode(units, cb, oc, q, 256, kernel=kern)
    for kern in (1, 3):
        with pytest.raises(NotImplementedError):
            B.decode_step(cb, q, 256, kernel=kern)


@pytest.mark.parametrize("bits,siq", [(4, True), (8, True), (4, False), (8, False)])
def test_wide_bit_records(bits, siq):
    """bits 4 / 8 on the fast path (cache.py:52-75, QuantConfig(bits=4|8)): the reference-layout
    planes bit-exact vs the oracle, the sign plane equal to its codes, the fp16 records equal
    to the oracle's dequantised rows (cache.gather, cache.py:118-158) divided by alpha-hat and
    rounded once, selections exact vs restate32, attention vs the float64 oracle on the same
    b-bit cache; the two-kernel path runs it (1 / 3 refuse, as at bits 16)."""
    from .fastlayout import records16_to_arrays
    units, cb, oc, q = make_variant(4096, [820, 821], bits, siq)
    torch.cuda.synchronize()
    for i, c in enumerate(oc):
        plane = c.kmag if siq else c.kdirect
        np.testing.assert_array_equal(cb.mu64[i].cpu().numpy(), c.mu)
        np.testing.assert_array_equal(cb.alpha64[i].cpu().numpy(), c.alpha)
        np.testing.assert_array_equal(cb.ref["codes"][i].cpu().numpy(), c.packed_codes)
        np.testing.assert_array_equal(cb.ref["kq"][i].cpu().numpy(), plane.packed)
        np.testing.assert_array_equal(cb.ref["ks"][i].cpu().numpy(), plane.scales)
        np.testing.assert_array_equal(cb.ref["kz"][i].cpu().numpy(), plane.zeros)
        np.testing.assert_array_equal(cb.ref["vq"][i].cpu().numpy(), c.vq.packed)
        np.testing.assert_array_equal(cb.ref["vs"][i].cpu().numpy(), c.vq.scales)
        np.testing.assert_array_equal(cb.ref["vz"][i].cpu().numpy(), c.vq.zeros)
        np.testing.assert_array_equal(unrotate_signs(cb.signs[i].cpu().numpy()), c.packed_codes)
        kh, vh = records16_to_arrays(cb.recs[i].cpu().numpy())
        kd = O.dequantize_keys(c.kmag, c.alpha, c.codes) if siq else O.dequantize(c.kdirect)
        ahat = cb.alpha32[i].cpu().numpy().astype(np.float64)
        if siq:
            ahat[ahat == 0] = 1.0
        else:
            assert np.all(ahat == 1.0)
        np.testing.assert_array_equal(kh, (kd / ahat).astype(np.float16))
        np.testing.assert_array_equal(vh, O.dequantize(c.vq).astype(np.float16))
    for kern in (0, 4):
        _check_decode(units, cb, oc, q, 256, kernel=kern)
    for kern in (1, 3):
        with pytest.raises(NotImplementedError):
            B.decode_step(cb, q, 256, kernel=kern)


def test_wide_bits_with_window_sinks_and_appends():
    """bits 4 with SnapKV window sinks and decode-time appends (the recent ring) through the
    16-bit-record decode: the same sinks as the oracle, selections exact vs restate32 and the
    attention vs the float64 4-bit oracle cache with its appended rows."""
    L, seeds, gq, appends = 4096, [830, 831], 4, 3
    units = [gen_unit(L, 128, gq + appends, s, window=32) for s in seeds]
    K = torch.tensor(np.stack([u.keys for u in units]), dtype=torch.bfloat16, device="cuda")
    V = torch.tensor(np.stack([u.values for u in units]), dtype=torch.bfloat16, device="cuda")
    W = torch.tensor(np.stack([u.window for u in units]), device="cuda")
    cb = B.prefill_batch(K, V, sink_count=64, window=W, bits=4, recent_capacity=1)
    oc = []
    for u in units:
        c = O.prefill(u.keys, u.values, bits=4, sink_count=64)
        c.sinks = O.window_sinks(u.keys - c.mu, u.window, 64, 7)
        c.sink_k = (u.keys - c.mu)[c.sinks].copy()
        c.sink_v = u.values[c.sinks].copy()
        oc.append(c)
    for i, c in enumerate(oc):
        np.testing.assert_array_equal(cb.sink_idx[i].cpu().numpy(), c.sinks)
    for a in range(appends):
        kk = np.stack([u.queries[gq + a] * 0.5 for u in units])
        vv = np.stack([u.queries[gq + a][::-1].copy() for u in units])
        B.append_batch(cb, torch.tensor(kk, device="cuda"), torch.tensor(vv, device="cuda"))
        for i, c in enumerate(oc):
            O.append(c, kk[i], vv[i])
    q = torch.tensor(np.stack([u.queries[:gq] for u in units]), dtype=torch.float32, device="cuda")
    _check_decode(units, cb, oc, q, 300, kernel=0)


@pytest.mark.parametrize("name,bits,siq", [("direct_d128", 2, False), ("b1_sinks_d128", 1, True),
                                           ("lossless_d128", 16, True), ("c1_u0", 2, True)])
def test_fast_variants_match_reference_golden(golden, name, bits, siq):
    """Fast-path variants against the real reference's outputs (tests/golden, made by running
    sikv.prefill / select_tokens / sparse_attention): the group-sum selection equals the
    reference's set (certified float32 check, measured: identical) and the attention is within
    the bars of the reference's float64 outputs on that selection."""
    meta, arr = golden
    rec = meta[name]
    u = gen_unit(rec["L"], 128, rec["gq"], rec["seed"])
    K = torch.tensor(u.keys[None], dtype=torch.bfloat16, device="cuda")
    V = torch.tensor(u.values[None], dtype=torch.bfloat16, device="cuda")
    cb = B.prefill_batch(K, V, sink_count=rec["sinks"], bits=bits, sign_in_quant=siq)
    q = torch.tensor(u.queries[None, : rec["gq"]], dtype=torch.float32, device="cuda")
    res = B.decode_step(cb, q, rec["k"], with_selection=True)
    got = res.selection[0, : int(res.counts[0])].cpu().numpy()
    np.testing.assert_array_equal(got, arr[f"{name}/sel"])
    ref_out = arr[f"{name}/attn"]
    for h in range(rec["gq"]):
        assert O.rel_l2(res.out[0, h].cpu().numpy(), ref_out[h]) <= att_rel_l2(rec["L"]), h


@pytest.mark.parametrize("kernel", [0, 1, 3, 4])
def test_decode_step_in_cuda_graph(c1, kernel):
    """The hot path is stream-ordered and allocation-free once its output and workspace exist
    (no host syncs, PDL launches capture as programmatic edges): one decode step captured in a
    CUDA graph and replayed with new queries gives the eager step's outputs bit for bit."""
    units, cb, oc, q = c1
    k = 256
    q_static = q.clone()
    out_static = torch.empty(q.shape[0], q.shape[1], 128, device="cuda")
    B.decode_step(cb, q_static, k, out=out_static, kernel=kernel)          # warm-up: workspace, attributes
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        B.decode_step(cb, q_static, k, out=out_static, kernel=kernel)      # the capture stream's workspace
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        B.decode_step(cb, q_static, k, out=out_static, kernel=kernel)
    rng = np.random.default_rng(11)
    for _ in range(3):
        qn = torch.tensor(rng.standard_normal(tuple(q.shape)), dtype=torch.float32, device="cuda")
        q_static.copy_(qn)
        g.replay()
        torch.cuda.synchronize()
        ref = B.decode_step(cb, qn, k, kernel=kernel).out
        torch.cuda.synchronize()
        assert torch.equal(out_static, ref)


def test_long_units_extra_sample_passes_and_retries():
    """Units of >= 64K tokens take extra sample passes (decode_select_kernel<true>); a candidate
    buffer too small for the sampled threshold forces the rescan path, whose sample rank is
    converted to the first pass's keys.  The selections stay exact (restate32) either way."""
    from paper_2603_14224_b200 import _lib
    units, cb, oc, q = make(65536, [300, 301], gq=4)
    k = 2048
    _check_decode(units, cb, oc, q, k, kernel=4)                  # default buffer: no rescan
    clk = torch.zeros(len(units), 16, dtype=torch.int64, device="cuda")
    _lib.call("sikv_debug_set_decode_profile", _lib.ptr(clk))
    try:
        res = _check_decode(units, cb, oc, q, k, kernel=4, cap=2400)
    finally:
        _lib.call("sikv_debug_set_decode_profile", None)
    attempts = clk[:, 9].cpu().numpy()
    fallback = (res.diag.cpu().numpy() & 4) != 0
    assert ((attempts >= 1) | fallback).all(), (attempts, fallback)


_FIRST_CALL_IN_CAPTURE = r"""
import sys
sys.path.insert(0, sys.argv[1])
import torch
from paper_2603_14224_b200 import _lib as L_
L = 1000
sc = torch.randn(L, dtype=torch.float64, device="cuda")
ws = torch.empty(L_.lib().sikv_topk_workspace_bytes(1, L), dtype=torch.uint8, device="cuda")
out = torch.empty(8, dtype=torch.int32, device="cuda")
cnt = torch.zeros(2, dtype=torch.int32, device="cuda")
s, g = torch.cuda.Stream(), torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):      # the library's first runtime call is captured
        L_.call("sikv_topk", L_.ptr(sc), 0, 1, L, None, 0, 8, L_.ptr(ws), L_.ptr(out), 8, L_.ptr(cnt),
                L_.stream())
g.replay()
torch.cuda.synchronize()
assert torch.equal(out.sort().values, torch.topk(sc, 8).indices.int().sort().values)
print("ok")
"""


def test_first_library_call_inside_graph_capture():
    """The C ABI binds the thread's context before its first launch (capi.cu rt_bind) in a
    capture-safe way: a fresh process whose first library call is captured into a CUDA graph."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _FIRST_CALL_IN_CAPTURE, root], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
