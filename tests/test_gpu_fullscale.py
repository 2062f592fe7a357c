"""Full-size checks of the benchmarked workloads on the decode path bench.py times:
C2 (BASELINE.json configs[1], the headline: 4096 units x 32K tokens, top-k 2048, auto ->
the two-kernel path), C4 (Qwen2.5-7B: 7168 units x 8K, top-k 1024, GQA 7, two kernels) and
C3 (Llama-3.1-8B: 256 units x 128K, top-k 4096, two kernels with split attention).

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
from .tolerances import ATT_COS, att_rel_l2
from oracle import restate32 as R
from oracle import sikv_oracle as O
from paper_2603_14224_b200 import _lib
from paper_2603_14224_b200 import batch as B
from paper_2603_14224_b200.synth import gen_units_by_id

pytestmark = pytest.mark.gpu

SEED = 1234


_FULL = {}


def full_run(config):
    """The config's whole cache (every unit, as bench.py builds it) and one decode step of
    it, built once per session and shared by the tests below."""
    if config not in _FULL:
        layers, batch, kvh, gq, L, k, _ = bench.CONFIGS[config]
        units = layers * batch * kvh
        cb, q = bench.build_cache(range(units), L, gq, SEED, torch.device("cuda", 0))
        res = B.decode_step(cb, q, k, with_selection=True, with_lse=True, with_diag=True)
        torch.cuda.synchronize()
        _FULL[config] = (cb, q, res, _lib.lib().sikv_decode_last_kernel())
    return _FULL[config]


@pytest.mark.parametrize("config,path", [("c2", 4), ("c4", 4), ("c3", 4)])
def test_full_scale(config, path):
    layers, batch, kvh, gq, L, k, _ = bench.CONFIGS[config]
    units = layers * batch * kvh
    dev = torch.device("cuda", 0)
    cb, q, res, used = full_run(config)
    assert used == path
    S = bench.SINKS
    sel, cnt = res.selection, res.counts
    assert bool((cnt == S + k).all())
    assert bool((sel[:, 1:] > sel[:, :-1]).all())                      # sorted, unique
    assert bool((sel[:, :S] == torch.arange(S, device=dev, dtype=sel.dtype)).all())
    assert bool((sel[:, -1] < L).all())
    assert not bool(((res.diag & 4) != 0).any())                        # no exact fallback
    assert bool(torch.isfinite(res.out).all()) and bool(torch.isfinite(res.lse).all())

    for u in (0, units // 5, units // 2, units - 1):
        K, V = gen_units_by_id([u], L, 128, SEED, dev)                  # bench.build_cache's unit u
        keys = K[0].double().cpu().numpy()
        values = V[0].double().cpu().numpy()
        del K, V
        c = O.prefill(keys, values, sink_count=S)
        qu = q[u].cpu().numpy()
        idx = R.select32(c, qu, k)[0]
        got = sel[u, : int(cnt[u])].cpu().numpy()
        np.testing.assert_array_equal(got, idx)
        # and the float64 reference selection on the group-summed query (cache.py:290-309):
        # equal sets unless the float64 boundary gap is within the certified float32 bound
        ok, ndiff, gap, bound = R.certified_selection_check(c, qu, k, idx)
        assert ok, (u, ndiff, gap, bound)
        out = res.out[u].cpu().numpy()
        for h in range(gq):
            ref = O.sparse_attention(qu[h].astype(np.float64), idx, c)
            assert O.rel_l2(out[h], ref) <= att_rel_l2(L), (u, h, O.rel_l2(out[h], ref))
            assert O.cosine(out[h], ref) >= ATT_COS


# the auto path each rank's shard runs at N GPUs (units per rank decide it, capi.cu)
SHARD_PATHS = {("c2", 2): 4, ("c2", 4): 4, ("c2", 8): 1, ("c4", 2): 4, ("c4", 4): 4, ("c4", 8): 4,
               ("c3", 2): 1, ("c3", 4): 3, ("c3", 8): 3}


@pytest.mark.parametrize("config", ["c2", "c4", "c3"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_shard_slices_match_full_run(config, world):
    """every rank's shard (ShardPlan, head x batch), decoded on its own at its
    own size and auto path, reproduces the single-GPU run: selections identical, outputs
    equal to the full run within the cross-path fp16-P rounding (rel-L2 <= 1e-3) and to the
    float64 oracle on one unit per rank; the assembled model output equals the full run's."""
    from paper_2603_14224_b200.shard import ShardPlan, assemble
    layers, batch, kvh, gq, L, k, _ = bench.CONFIGS[config]
    cb, q, full, _ = full_run(config)
    plan = ShardPlan(layers, batch, kvh, world)
    outs = []
    for rank in range(world):
        ids = plan.local_units(rank).to("cuda")
        sub = B.subset(cb, ids)
        res = B.decode_step(sub, q.index_select(0, ids), k, with_selection=True)
        torch.cuda.synchronize()
        assert _lib.lib().sikv_decode_last_kernel() == SHARD_PATHS[(config, world)]
        assert torch.equal(res.counts, full.counts.index_select(0, ids))
        assert torch.equal(res.selection, full.selection.index_select(0, ids))
        ref = full.out.index_select(0, ids)
        err = ((res.out - ref).norm(dim=-1) / ref.norm(dim=-1)).max().item()
        assert err <= 1e-3, (rank, err)
        outs.append(res.out)
        del sub
        if rank in (0, world - 1):
            u = int(ids[len(ids) // 2])
            K, V = gen_units_by_id([u], L, 128, SEED, torch.device("cuda", 0))
            c = O.prefill(K[0].double().cpu().numpy(), V[0].double().cpu().numpy(), sink_count=bench.SINKS)
            qu = q[u].cpu().numpy()
            i = len(ids) // 2
            got = res.selection[i, : int(res.counts[i])].cpu().numpy()
            np.testing.assert_array_equal(got, R.select32(c, qu, k)[0])
            for h in range(gq):
                r64 = O.sparse_attention(qu[h].astype(np.float64), got, c)
                assert O.rel_l2(res.out[i, h].cpu().numpy(), r64) <= att_rel_l2(L)
    model = assemble(torch.cat(outs), plan)
    ref_model = full.out.view(layers, batch, kvh * gq, 128)
    err = ((model - ref_model).norm(dim=-1) / ref_model.norm(dim=-1)).max().item()
    assert err <= 1e-3
