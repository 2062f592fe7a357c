"""Full-size checks of the benchmarked workloads on the decode path bench.py times:
C2 (BASELINE.json configs[1], the headline: 4096 units x 32K tokens, top-k 2048, auto ->
the two-kernel path), C4 (Qwen2.5-7B: 7168 units x 8K, top-k 1024, GQA 7, two kernels) and
C3 (Llama-3.1-8B: 256 units x 128K, top-k 4096, one CTA per unit).

  * every unit: size-independent properties of the selection (exactly 64 + k sorted,
    unique indices, the 64 sinks first, no exact-fallback) and finite outputs;
  * a spread of units: the selection equals the float32 scoring restatement + the
    reference's top_k_select rule (oracle/restate32.py) on the same regenerated inputs,
    and the attention matches the float64 oracle within the stated tolerance.
"""

import numpy as np
import pytest
import torch

import bench
from oracle import restate32 as R
from oracle import sikv_oracle as O
from paper_2603_14224_b200 import _lib
from paper_2603_14224_b200 import batch as B
from paper_2603_14224_b200.synth import gen_units_torch

pytestmark = pytest.mark.gpu

SEED = 1234


@pytest.mark.parametrize("config,path", [("c2", 4), ("c4", 4), ("c3", 1)])
def test_full_scale(config, path):
    layers, batch, kvh, gq, L, k, _ = bench.CONFIGS[config]
    units = layers * batch * kvh
    dev = torch.device("cuda", 0)
    cb, q = bench.build_cache(units, 0, L, gq, SEED, dev)
    res = B.decode_step(cb, q, k, with_selection=True, with_lse=True, with_diag=True)
    torch.cuda.synchronize()
    assert _lib.lib().sikv_decode_last_kernel() == path
    S = bench.SINKS
    sel, cnt = res.selection, res.counts
    assert bool((cnt == S + k).all())
    assert bool((sel[:, 1:] > sel[:, :-1]).all())                      # sorted, unique
    assert bool((sel[:, :S] == torch.arange(S, device=dev, dtype=sel.dtype)).all())
    assert bool((sel[:, -1] < L).all())
    assert not bool(((res.diag & 4) != 0).any())                        # no exact fallback
    assert bool(torch.isfinite(res.out).all()) and bool(torch.isfinite(res.lse).all())

    chunk = max(1, min(units, (1 << 31) // (L * 128 * 2)))              # bench.build_cache's chunks
    for u in (0, units // 5, units // 2, units - 1):
        u0 = (u // chunk) * chunk
        K, V = gen_units_torch(min(chunk, units - u0), L, 128, SEED + u0, dev)
        keys = K[u - u0].double().cpu().numpy()
        values = V[u - u0].double().cpu().numpy()
        del K, V
        c = O.prefill(keys, values, sink_count=S)
        qu = q[u].cpu().numpy()
        idx = R.select32(c, qu, k)[0]
        got = sel[u, : int(cnt[u])].cpu().numpy()
        np.testing.assert_array_equal(got, idx)
        # and the float64 reference selection on the group-summed query (cache.py:290-309):
        # the float32 order may only move boundary ties (>= k - 1 of k)
        ref64 = O.select(c, qu.astype(np.float64).sum(axis=0), k)[0]
        assert len(np.intersect1d(ref64, idx)) >= len(idx) - 1
        out = res.out[u].cpu().numpy()
        for h in range(gq):
            ref = O.sparse_attention(qu[h].astype(np.float64), idx, c)
            assert O.rel_l2(out[h], ref) <= 3e-3, (u, h, O.rel_l2(out[h], ref))
            assert O.cosine(out[h], ref) >= 0.99999
