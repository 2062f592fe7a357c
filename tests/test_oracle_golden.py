"""Pin the CPU oracle against the real reference's outputs and known answers (CPU only)."""

import hashlib

import numpy as np
import pytest

from oracle import restate32 as R
from oracle import sikv_oracle as O
from paper_2603_14224_b200.synth import gen_unit

FAST_CASES = ["c1_u0", "c1_u1", "win_1k", "append_2k", "gq7_2k", "b4_d64", "direct_d32",
              "b8_d32", "b1_d128", "lossless_d64", "direct_d128", "b1_sinks_d128", "lossless_d128"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def build(rec):
    u = gen_unit(rec["L"], rec["D"], rec["gq"] + rec["appends"], rec["seed"])
    cache = O.prefill(u.keys, u.values, bits=rec["bits"], group=rec["group"],
                      sink_count=rec["sinks"], sign_in_quant=rec["sign_in_quant"],
                      window=u.window if rec["window"] else None)
    for a in range(rec["appends"]):
        q = u.queries[rec["gq"] + a]
        O.append(cache, q * 0.5, q[::-1].copy())
    return u, cache


@pytest.mark.parametrize("name", FAST_CASES + [pytest.param("c2_1unit", marks=pytest.mark.slow)])
def test_oracle_matches_reference(golden, name):
    meta, arr = golden
    rec = meta[name]
    u, c = build(rec)
    assert rec["inputs_sha"] == sha(np.stack([u.keys.sum(0), u.values.sum(0)])) + sha(u.keys) + sha(u.values)
    assert sha(c.packed_codes) == rec["codes_sha"]
    np.testing.assert_array_equal(c.mu, arr[f"{name}/mu"])
    np.testing.assert_array_equal(c.alpha, arr[f"{name}/alpha"])
    np.testing.assert_array_equal(c.centroids, arr[f"{name}/centroids"])
    for tag, q in (("kmag", c.kmag), ("kdirect", c.kdirect), ("values", c.vq)):
        if tag in rec["planes"]:
            p = rec["planes"][tag]
            assert (sha(q.packed), sha(q.scales), sha(q.zeros)) == (p["packed"], p["scales"], p["zeros"])
        else:
            assert q is None
    assert c.sinks.tolist() == rec["sink_indices"]
    qh = u.queries[: rec["gq"]]
    qbar = qh.sum(axis=0)
    table = O.lut(qbar, c.centroids)
    np.testing.assert_array_equal(table, arr[f"{name}/lut"])
    assert sha(O.score(table, c.codes)) == rec["scores_sha"]
    idx, ns, nr, nd = O.select(c, qbar, k=rec["k"])
    np.testing.assert_array_equal(idx, arr[f"{name}/sel"])
    assert [ns, nr, nd] == rec["sel_counts"]
    for h, q in enumerate(qh):
        assert O.select(c, q, k=rec["k"])[0].tolist() == rec["per_head_sel"][h]
        out = O.sparse_attention(q, idx, c)
        np.testing.assert_allclose(out, arr[f"{name}/attn"][h], rtol=1e-12, atol=1e-14)
    if "budget_sel" in rec:
        assert O.select(c, qbar, budget=rec["k"] + 10)[0].tolist() == rec["budget_sel"]
        assert O.select(c, qbar, sparsity=0.05, sign_only=True)[0].tolist() == rec["sparsity_signonly_sel"]


def test_restate32_overlaps_reference(golden):
    """fp32 pair-LUT scoring picks (nearly) the same set as the fp64 reference."""
    meta, arr = golden
    for name in ("c1_u0", "c1_u1", "gq7_2k"):
        rec = meta[name]
        u, c = build(rec)
        idx = R.select32(c, u.queries[: rec["gq"]], rec["k"])[0]
        ref = arr[f"{name}/sel"]
        assert len(np.intersect1d(idx, ref)) >= len(ref) - 1


# ---- known answers from the reference's own unit tests -------------------------------
def test_sign_code_known_answers():
    # test_codebook.py:19-30, 49-51, 61-63
    assert O.sign_codes(np.array([[0.5, -0.3, 1.2, -0.1]]))[0, 0] == 10
    assert O.sign_codes(np.zeros((1, 4)))[0, 0] == 15
    assert O.sign_codes(np.array([[0.0, -1.0, 0.0, -1.0]]))[0, 0] == 10
    assert O.sign_codes(-np.ones((1, 4)))[0, 0] == 0
    assert O.sign_codes(np.array([[0.5, -0.3, 1.2, -0.1, 1, 1, 1, 1]])).tolist() == [[10, 15]]


def test_pack_known_answers():
    # test_quantizer.py:26-31
    assert O.pack(np.array([[1, 0, 3, 2]]), 2).tolist() == [[1 | (3 << 4) | (2 << 6)]]
    assert O.pack(np.array([[0xA, 0x5]]), 4).tolist() == [[0x5A]]
    rng = np.random.default_rng(0)
    for bits in (1, 2, 4, 8):
        c = rng.integers(0, 1 << bits, size=(7, 37))
        np.testing.assert_array_equal(O.unpack(O.pack(c, bits), bits, 37), c)


def test_quant_known_answers():
    # test_quantizer.py:48-73
    q = O.quantize(np.array([[0.0, 1.0, 2.0, 3.0]]), 2, 4)
    assert q.scales.tolist() == [[1.0]] and q.zeros.tolist() == [[0.0]]
    assert q.codes().tolist() == [[0, 1, 2, 3]]
    q = O.quantize(np.array([[5.0] * 4]), 2, 4)
    assert q.scales.tolist() == [[0.0]] and q.codes().tolist() == [[0, 0, 0, 0]]
    assert O.quantize(np.array([[0.0, 0.4, 2.6, 3.0]]), 2, 4).codes().tolist() == [[0, 0, 3, 3]]
    assert O.quantize(np.array([[0.0, 0.5, 1.5, 3.0]]), 2, 4).codes().tolist() == [[0, 1, 2, 3]]
    # exact recompose of a degenerate key group (test_quantizer.py:154-162)
    K = np.array([[0.5, -0.25, 1.0, -1.0]])
    a = np.array([0.5, 0.25, 1.0, 1.0])
    km = O.quantize_key_mags(K, a, 2, 4)
    np.testing.assert_array_equal(O.dequantize_keys(km, a, O.sign_codes(K)), K)


def test_retrieval_known_answers():
    # test_retrieval.py:19-29, 122-148, 181-192
    K = np.array([[0.5, -0.3, 1.2, -0.1]])
    cb = O.codebook(K, O.sign_codes(K))
    assert O.lut(np.array([1.0, 0, 0, 0]), cb)[0, 10] == pytest.approx(0.5)
    assert O.top_k([0.1, 5.0, 3.0, 2.0], 2)[0].tolist() == [1, 2]
    assert O.top_k([0.1, 5.0, 3.0, 2.0], 2, sink={0})[0].tolist() == [0, 1, 2]
    assert O.top_k([1.0, 1.0, 0.0], 1)[0].tolist() == [0]
    assert O.top_k([1.0, 2.0, 3.0, 4.0], 1, sink={0, 1}, recent={1, 2})[1:] == (2, 1, 1)
    assert O.top_k([3.0, 1.0, 2.0], 10, sink={0})[3] == 2
    assert O.resolve_k(4096, 64, budget=160) == 96
    assert O.resolve_k(4096, 0, sparsity=0.075) == 307
    assert O.resolve_k(1000, 0, sparsity=0.0755) == 76
    assert O.resolve_k(1000, 64, sparsity=0.01) == 1
    with pytest.raises(ValueError, match="exactly one"):
        O.resolve_k(100, 0)


def test_codebook_known_answers():
    # test_codebook.py:115-130
    K = np.array([[1, -1, 1, -1], [3, -3, 3, -3]], dtype=float)
    np.testing.assert_array_equal(O.codebook(K, O.sign_codes(K))[0, 10], [2, -2, 2, -2])
    K = np.array([[1.0, 1.0, 1.0, 1.0]])
    np.testing.assert_array_equal(O.codebook(K, O.sign_codes(K))[0, 7], np.zeros(4))


def test_stats_known_answers():
    # test_normalize.py:11-14
    mu, alpha = O.channel_stats(np.array([[1.0, 3.0], [3.0, 5.0]]))
    assert mu.tolist() == [2.0, 4.0] and alpha.tolist() == [1.0, 1.0]
