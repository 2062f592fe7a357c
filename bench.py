"""Decode-step benchmark of the self-indexing KV-cache path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One *step* = one decode step of the whole model configuration: for every decode unit
(layer x batch x KV head) the fused kernel scores all L sign records, selects the exact
top-k, and runs sparse attention for the unit's GQA query heads.  Metric:
decode steps/s (BASELINE.json), plus the HBM roofline fraction of the decode kernel.

Default workload = BASELINE.json configs[1] (C2): Llama-3-8B geometry, 32 layers x batch 16
x 8 KV heads = 4096 units, 32K context, top-k 2048, 64 sinks, GQA group 4, bf16 synthetic
K/V compressed by our encoder (layer by layer, raw K/V discarded).  The compressed planes
(~19 GB) are far larger than L2, so no flush is needed between steps.

Multi-GPU (torchrun): units are sharded by KV head across ranks (no data-path collective);
the per-step bf16 outputs are all-gathered over NCCL inside the timed region.

``--impl reference`` times the CPU oracle (oracle/, the float64 restatement of the
reference, the only CPU implementation of this path that can run on the GPU box) on a
bounded sample of units with every host core, and prints the same JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (layers, batch, kv_heads, gq, L, k, label)
    "c1": (1, 1, 8, 4, 4096, 256, "Llama-3-8B head geometry, 1 layer, batch 1, 4K ctx, top-k 256"),
    "c2": (32, 16, 8, 4, 32768, 2048, "Llama-3-8B, 32 layers, batch 16, 32K ctx, top-k 2048"),
    "c3": (32, 1, 8, 4, 131072, 4096, "Llama-3.1-8B, 32 layers, batch 1, 128K ctx, top-k 4096"),
    "c4": (28, 64, 4, 7, 8192, 1024, "Qwen2.5-7B, 28 layers, batch 64, 8K ctx, top-k 1024"),
    # prefill-side compression throughput (BASELINE.json configs[4])
    "c5": (32, 1, 8, 4, 131072, 0, "key/value compression of 128K tokens x 32 layers, Llama-3-8B geometry"),
}
SINKS = 64


# bytes of one selected token's K/V: 2-bit (payloads 2 x 32 B + fp16 params 2 x 16 B), 1-bit
# (2 x 16 B + 2 x 16 B), 16-bit (2 x 256 B)
SEL_BYTES = {2: 96, 1: 64, 16: 512, 4: 512, 8: 512}   # bits 4 / 8: stored as the 16-bit records


def algo_bytes_per_unit(L: int, k: int, gq: int, S: int = SINKS, bits: int = 2) -> int:
    """16 L (sign index) + 96 k (2-bit K/V payload + fp16 params of the
    selected tokens; 512 k at bits 16) + 512 S (bf16 sink K, V) + 2 Gq 256 (q, out) + 8 KiB
    centroids + 512 B alpha."""
    return 16 * L + SEL_BYTES[bits] * min(k, L - S) + 512 * S + 2 * gq * 256 + 8192 + 512


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every 10 ms during the timed
    region (nvidia-smi fallback when pynvml is missing)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def __enter__(self):
        def run_nvml(pynvml, h):
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = [0x8, 0x40, 0x20, 0x4]   # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while True:
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append([sm, mx] + ["active" if r & b else "" for b in bits])
                except Exception:
                    pass
                if self._stop.wait(0.002):
                    break

        def run_smi():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.05)

        try:   # NVML is initialised (and its first, slow queries made) before the timed region
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self._nvml = (pynvml, h)
            target = lambda: run_nvml(pynvml, h)  # noqa: E731
        except Exception:
            self._nvml = None
            target = run_smi
        self._t = threading.Thread(target=target, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        # one more sample taken here, as the timed region's final synchronize returns
        if self._nvml is not None:
            pynvml, h = self._nvml
            try:
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([sm, mx] + ["active" if r & b else "" for b in (0x8, 0x40, 0x20, 0x4)])
            except Exception:
                pass
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(int(float(s[0])) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if str(s[2 + i]).lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(float(self.samples[0][1])),
                "reasons": reasons, "samples": len(sm)}


def ncu_traffic(config: str):
    """DRAM bytes (read + write) per launch of the decode kernel from the committed ncu
    capture of this configuration (profiles/*/ncu_<config>_summary.json), or None."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", f"ncu_{config}_summary.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
            best = {"bytes": int(d["dram_bytes_read"]) + int(d["dram_bytes_write"]), "kernel": d.get("kernel"),
                    "source": os.path.relpath(path, ROOT)}
        except Exception:
            pass
    return best


def scaled_config(name: str, n: int, scaling: str):
    """The workload at N GPUs.  Weak scaling (default; the decode units are independent, so
    the path partitions): the model's batch grows with N, every GPU keeps the N = 1 config's
    unit count (KV-head x batch shard), and `value` counts N = 1-sized steps (units processed
    / units per N = 1 step / time).  Strong: the N = 1 model split over N GPUs."""
    layers, batch, kvh, gq, L, k, label = CONFIGS[name]
    if scaling == "weak" and n > 1:
        return (layers, batch * n, kvh, gq, L, k, f"{label}; batch x{n} over {n} GPUs (weak scaling)"), n
    return CONFIGS[name], 1


def decode_config(name: str, world: int, cfg=None, rep: int = 1) -> dict:
    """The workload description both arms print (identical for the same config and N)."""
    from paper_2603_14224_b200.shard import ShardPlan
    layers, batch, kvh, gq, L, k, label = cfg or CONFIGS[name]
    plan = ShardPlan(layers, batch, kvh, world)
    planes = (16 + 128) * L * plan.units_per_rank / 1e9
    return {"workload": name, "label": label, "layers": layers, "batch": batch, "kv_heads": kvh,
            "q_heads_per_kv": gq, "context": L, "top_k": k, "sinks": SINKS, "units": layers * batch * kvh,
            "units_per_gpu": plan.units_per_rank,
            "parallelism": f"kv-head x batch shard {plan.head_parts}x{plan.batch_parts}",
            "global_batch": batch,
            "value_counts": (f"steps of the N = 1 model ({layers * batch * kvh // rep} units) per second, "
                             f"all GPUs: {rep} per step of this {rep}x-batch model" if rep > 1
                             else "decode steps of this model per second"),
            "l2": (f"inputs > L2: {planes:.1f} GB of compressed planes per GPU, every step reads them afresh"
                   if planes > 0.5 else f"inputs {planes * 1e3:.0f} MB, smaller than L2 (CPU-reference config)")}


# ------------------------------------------------------------------------------- GPU arm
def build_cache(gids, L: int, gq: int, seed: int, device, bits: int = 2, sign_in_quant: bool = True):
    """Compressed caches of the decode units with global ids `gids` (unit content depends
    only on its id: synth.gen_units_by_id), plus their queries [n, gq, 128] float32."""
    import torch

    from paper_2603_14224_b200 import _lib
    from paper_2603_14224_b200 import batch as B
    from paper_2603_14224_b200.synth import gen_queries_by_id, gen_units_by_id

    gids = [int(x) for x in gids]
    n_units = len(gids)
    cb = B.empty_batch(n_units, L, sink_count=SINKS, device=device, bits=bits, sign_in_quant=sign_in_quant)
    q = torch.empty(n_units, gq, 128, device=device, dtype=torch.float32)
    chunk = max(1, min(n_units, (1 << 31) // (L * 128 * 2)))   # <= 2 GiB of raw K per chunk
    ws = None
    for u0 in range(0, n_units, chunk):
        ids = gids[u0:u0 + chunk]
        K, V = gen_units_by_id(ids, L, 128, seed, device)
        need = _lib.lib().sikv_encode_workspace_bytes(len(ids), L, 128)
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=device)
        B.prefill_into(cb, u0, K, V, workspace=ws, check=False)
        q[u0:u0 + len(ids)] = gen_queries_by_id(K, ids, gq, seed + 7919).float()
        del K, V
    torch.cuda.synchronize()
    return cb, q


def run_ours(args, rank, world, cfg):
    import torch
    import torch.distributed as dist

    from paper_2603_14224_b200 import batch as B
    from paper_2603_14224_b200.shard import OutputExchange, ShardPlan, gather_outputs

    layers, batch, kvh, gq, L, k, label = cfg
    units = layers * batch * kvh
    plan = ShardPlan(layers, batch, kvh, world)
    ul = plan.units_per_rank
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cb, q = build_cache(plan.local_units(rank).tolist(), L, gq, 1234, dev, bits=args.bits,
                        sign_in_quant=not args.direct_keys)

    out = torch.empty(ul, gq, 128, device=dev, dtype=torch.float32)
    out16 = torch.empty(ul, gq, 128, device=dev, dtype=torch.bfloat16)
    flat = torch.empty(world * ul, gq, 128, device=dev, dtype=torch.bfloat16) if world > 1 else None
    model_out = torch.empty(layers, batch, kvh * gq, 128, device=dev, dtype=torch.bfloat16) if world > 1 else None

    per_head = args.policy == "per-head"
    decode = B.decode_step_per_head if per_head else B.decode_step
    # the output all-gather (north_star: "NCCL over NVLink only for the final output
    # all-gather"): fused into the decode's attention epilogue over NVLink peer memory
    # (OutputExchange, CUDA IPC) by default, or NCCL all_gather_into_tensor + reassembly
    xch = OutputExchange(plan, gq, rank, dev) if world > 1 and args.gather == "fused" else None

    def step(qq, o=out):
        if xch is not None:
            decode(cb, qq, k, out=o, exchange=xch)
            xch.wait()
        else:
            decode(cb, qq, k, out=o)
            if world > 1:   # sharded outputs -> [layers, batch, H_q, D] on every rank (NCCL all-gather)
                out16.copy_(o)
                gather_outputs(out16, layers, batch, kvh, world, out=model_out, flat=flat)

    # correctness spot check on this rank (selection of unit 0 vs float32 restatement is in tests)
    for _ in range(args.warmup):
        step(q)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            step(q)
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # kernel-only time of the decode launches (same stream) for the roofline: at N = 1 the
    # timed step is exactly those launches; at N > 1 it also holds the all-gather, so the
    # decode launches are timed again on their own
    if world == 1:
        kern_ms = ms
    else:
        ek0, ek1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ek0.record(st)
        for _ in range(args.steps):
            decode(cb, q, k, out=out)
        ek1.record(st)
        torch.cuda.synchronize()
        kern_ms = ek0.elapsed_time(ek1) / args.steps

    # end to end through the public API: every step copies its queries from pinned host
    # memory and its outputs back to pinned host memory; copies run on a side stream and
    # overlap the neighbouring steps' decode (double-buffered device q / out)
    cs_in, cs_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    qh = q.cpu().pin_memory()
    oh = [torch.empty(ul, gq, 128, dtype=torch.float32).pin_memory() for _ in range(2)]
    qd = [torch.empty_like(q) for _ in range(2)]
    od = [torch.empty_like(out) for _ in range(2)]
    ev = lambda: torch.cuda.Event()  # noqa: E731
    h2d, comp, d2h = [ev(), ev()], [ev(), ev()], [ev(), ev()]

    def e2e_steps(n):
        for i in range(n):
            b = i & 1
            with torch.cuda.stream(cs_in):
                if i >= 2:
                    cs_in.wait_event(comp[b])         # qd[b] was read by step i-2
                qd[b].copy_(qh, non_blocking=True)
                h2d[b].record(cs_in)
            st.wait_event(h2d[b])
            if i >= 2:
                st.wait_event(d2h[b])                 # od[b] was copied out by step i-2
            step(qd[b], od[b])
            comp[b].record(st)
            with torch.cuda.stream(cs_out):
                cs_out.wait_event(comp[b])
                oh[b].copy_(od[b], non_blocking=True)
                d2h[b].record(cs_out)
        st.wait_stream(cs_in)
        st.wait_stream(cs_out)

    e2e_steps(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record(st)
    cs_in.wait_stream(st)
    cs_out.wait_stream(st)
    e2e_steps(args.steps)
    ee1.record(st)
    torch.cuda.synchronize()
    e2e_ms = ee0.elapsed_time(ee1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    res = decode(cb, q, k, with_diag=True)
    torch.cuda.synchronize()
    fallbacks = int(((res.diag & 4) != 0).sum().item())
    from paper_2603_14224_b200 import _lib as L_
    path = int(L_.lib().sikv_decode_last_kernel())
    launches_per_step = (2 if path == 4 else 1) + (0 if xch is None else (1 if path == 4 else 2))
    if world > 1:
        dist.barrier()         # no rank frees its exchange buffers while a peer still writes them

    if rank != 0:
        return None
    peak, peak_kind = peaks()
    # per-q-head policy: every query head scans its KV head's sign plane and gathers its own k
    bpu = (algo_bytes_per_unit(L, k, 1, bits=args.bits) * gq if per_head
           else algo_bytes_per_unit(L, k, gq, bits=args.bits))
    bytes_step = bpu * ul
    achieved = bytes_step / (kern_ms * 1e-3) / 1e9
    traffic = ncu_traffic(args.config) if world == 1 else None
    line = {
        "metric": "decode steps/sec + HBM roofline fraction, Llama-3-8B geometry, 32K ctx",
        "value": round(args.rep * 1000.0 / ms, 3),
        "unit": "decode steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 5),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "u2 K/V payload, f32 scores, f16 mma operands / f32 accumulate",
        "data": "synthetic (gen_synthetic distribution, Philox on GPU), random-init caches",
        "config": dict(decode_config(args.config, world, cfg, args.rep), policy=args.policy, bits=args.bits,
                       keys="direct" if args.direct_keys else "sign-in-quant",
                       **({"output_gather": "fused into the attention epilogue (NVLink peer stores, CUDA IPC)"
                           if xch is not None else "NCCL all_gather_into_tensor + reassembly"}
                          if world > 1 else {})),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_source": traffic["source"] if traffic else None,
                     "algo_bytes_per_launch": bytes_step,
                     "kernel_ms": round(kern_ms, 5)},
        "e2e": {"value": round(args.rep * 1000.0 / e2e_ms, 3), "unit": "decode steps/s",
                "h2d_bytes_per_step": int(qh.numel() * qh.element_size()),
                "d2h_bytes_per_step": int(oh[0].numel() * oh[0].element_size()),
                "overlap": "H2D and D2H on two side streams, double-buffered device q / out"},
        "gpu_launches": args.steps * launches_per_step,
        "decode_path": {1: "one CTA per unit", 2: "persistent warp-specialised", 3: "cluster split",
                        4: "two kernels: decode_select_kernel + decode_attend_kernel"}.get(path),
        "clocks": clk.summary(),
        "selection_fallbacks_last_step": fallbacks,
    }
    return line


def run_prefill(args, rank, world, cfg):
    """C5: compressed token-heads per second of the encoder (stats + sign codes + codebook
    + 2-bit K/V payloads + fp16 params, both layouts' fast planes), units head-sharded."""
    import torch
    import torch.distributed as dist

    from paper_2603_14224_b200 import _lib
    from paper_2603_14224_b200 import batch as B
    from paper_2603_14224_b200.synth import gen_units_torch

    layers, batch, kvh, gq, L, _, label = cfg
    units = layers * batch * kvh
    ul = units // world
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    chunk = min(64, ul)           # heads per prefill call (8: 1.57 G token-heads/s, 32: 1.75 G, 64: 1.78 G)
    cb = B.empty_batch(chunk, L, sink_count=SINKS, device=dev)
    ws = torch.empty(_lib.lib().sikv_encode_workspace_bytes(chunk, L, 128), dtype=torch.uint8, device=dev)
    K, V = gen_units_torch(chunk, L, 128, 77 + rank, dev)
    st = torch.cuda.current_stream()
    for _ in range(max(1, args.warmup)):
        B.prefill_into(cb, 0, K, V, workspace=ws, check=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    reps = max(1, ul // chunk)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        e0.record(st)
        for _ in range(args.steps):
            for _r in range(reps):       # every step encodes this rank's ul units (chunk at a time)
                B.prefill_into(cb, 0, K, V, workspace=ws, check=False)
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank != 0:
        return None
    th = units * L / (ms * 1e-3)            # token-heads per second, whole job
    peak, peak_kind = peaks()
    per_th = 512 + 112                      # read bf16 K,V; write 896-bit compressed record
    achieved = (reps * chunk * L * per_th) / (ms * 1e-3) / 1e9
    return {
        "metric": "prefill key/value compression throughput, Llama-3-8B geometry, 128K tokens x 32 layers",
        "value": round(th, 1), "unit": "token-heads/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64 math on bf16 inputs -> u2 payloads, f16 params",
        "data": "synthetic (gen_synthetic distribution, Philox on GPU)",
        "config": {"workload": "c5", "label": label, "units": units, "tokens": L,
                   "parallelism": f"kv-head shard x{world}"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind, "traffic": None,
                     "algo_bytes_per_token_head": per_th},
        "gpu_launches": args.steps * reps * 6, "clocks": clk.summary(),
    }


# ------------------------------------------------------------------------------- CPU arm
def _cpu_worker(conn, jobs, per_head=False):
    """One host core: prefills its sample units once (untimed), then on every 'step' runs the
    reference decode path of each of them (group-sum select_tokens + Gq x sparse_attention,
    cache.py:290-309, attention.py:52-62) on the CPU oracle and reports the seconds taken."""
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import sikv_oracle as O
    from paper_2603_14224_b200.synth import gen_unit
    units = []
    for (L, gq, k, seed) in jobs:
        u = gen_unit(L, 128, gq, seed)
        units.append((O.prefill(u.keys, u.values, sink_count=SINKS), u.queries[:gq], k))
    conn.send("ready")
    while conn.recv() == "step":
        t0 = time.perf_counter()
        for c, qs, k in units:
            if per_head:              # every query head selects for itself
                for h in range(qs.shape[0]):
                    O.sparse_attention(qs[h], O.select(c, qs[h], k=k)[0], c)
            else:
                idx = O.select(c, qs.sum(axis=0), k=k)[0]
                for h in range(qs.shape[0]):
                    O.sparse_attention(qs[h], idx, c)
        conn.send(time.perf_counter() - t0)
    conn.close()


class CpuArm:
    """The reference's CPU decode path on every host core, over a bounded sample of the
    workload's units (prefilled once, outside the timing).  One step = every core decodes its
    share of the sample; steps/s of the whole workload = (sample / units) / step seconds."""

    def __init__(self, cfg, sample_units: int, cores: int, per_head: bool = False):
        import multiprocessing as mp
        layers, batch, kvh, gq, L, k, _ = cfg
        self.units = layers * batch * kvh
        self.sample = sample_units
        self.cores = min(cores, sample_units)
        ctx = mp.get_context("fork")
        self.procs, self.conns = [], []
        for w in range(self.cores):
            jobs = [(L, gq, k, 9000 + i) for i in range(w, sample_units, self.cores)]
            a, b = ctx.Pipe()
            p = ctx.Process(target=_cpu_worker, args=(b, jobs, per_head), daemon=True)
            p.start()
            self.procs.append(p)
            self.conns.append(a)
        for c in self.conns:
            assert c.recv() == "ready"

    def step(self) -> float:
        t0 = time.perf_counter()
        for c in self.conns:
            c.send("step")
        busy = [c.recv() for c in self.conns]
        self.last_busy = busy
        return time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            c.send("stop")
        for p in self.procs:
            p.join(timeout=30)

    def line(self, seconds: float) -> dict:
        v = (self.sample / self.units) / seconds
        return {"value": round(v, 6), "unit": "decode steps/s", "cores": self.cores, "kind": "port",
                "unit_ms_1core": round(1e3 * sum(self.last_busy) / self.sample, 2),
                "sample": f"{self.sample} of the {self.units} units of one decode step per timed step "
                          f"(decode only: prefill once, untimed), steps/s = (sample / units) / step seconds",
                "cpu": _cpu_model()}


def cpu_baseline(cfg, sample_units: int, workers: int, steps: int = 3, warmup: int = 1, per_head: bool = False):
    arm = CpuArm(cfg, sample_units, workers, per_head)
    try:
        for _ in range(warmup):
            arm.step()
        t = sorted(arm.step() for _ in range(steps))
        res = arm.line(t[len(t) // 2])
    finally:
        arm.close()
    return res


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--bits", type=int, default=2, choices=[1, 2, 4, 8, 16], help="payload bits of the fast path")
    ap.add_argument("--direct-keys", action="store_true", help="keys quantised directly (no sign-in-quant)")
    ap.add_argument("--policy", default="group-sum", choices=["group-sum", "per-head"],
                    help="GQA selection policy: one selection per KV head from the summed queries "
                         "(default), or one per query head (SURVEY.md 8d)")
    ap.add_argument("--gather", default="fused", choices=["fused", "nccl"],
                    help="N > 1: output all-gather fused into the decode (peer stores) or NCCL")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=0, help="units in the CPU-baseline sample (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = batch x N, fixed units per GPU (default); strong = the N = 1 model split")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # not launched by torchrun: become the launcher of N ranks (one process per GPU)
        import socket
        with socket.socket() as s_:
            s_.bind(("127.0.0.1", 0))
            port = s_.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    cfg, args.rep = scaled_config(args.config, world if world > 1 else args.gpus, args.scaling)

    if args.impl == "reference":
        if rank != 0:
            return
        cores = os.cpu_count() or 1
        sample = args.cpu_sample or 2 * cores
        # every step = the sample's decode on every host core; --warmup / --steps as given
        arm = CpuArm(cfg, sample, cores, args.policy == "per-head")
        try:
            for _ in range(args.warmup):
                arm.step()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                arm.step()
            secs = (time.perf_counter() - t0) / args.steps
            v = arm.line(secs)
            v["value"] = v["value"] * args.rep      # weak scaling: in steps of the N = 1 model
        finally:
            arm.close()
        layers, batch, kvh, gq, L, k, label = cfg
        print(json.dumps({
            "metric": "decode steps/sec + HBM roofline fraction, Llama-3-8B geometry, 32K ctx",
            "value": v["value"], "unit": "decode steps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1000.0 / v["value"], 3),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gen_synthetic distribution)", "impl": "reference",
            "config": dict(decode_config(args.config, world if world > 1 else args.gpus, cfg, args.rep),
                           policy=args.policy,
                           bits=args.bits, keys="direct" if args.direct_keys else "sign-in-quant"),
            "cpu_baseline": v,
            "e2e": {"value": v["value"], "unit": "decode steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        # NCCL's init log (transport / NVLS choice) to a per-rank file, stdout stays one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH,NVLS")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(os.environ.get("SIKV_NCCL_LOG_DIR", "/tmp"),
                                                              "sikv_nccl.%h.%p.log"))
        if os.environ.get("SIKV_BENCH_SHARE_GPU"):
            # code-path check on a one-GPU box: every rank on cuda:0, gloo for the host-side
            # collectives (NCCL refuses two ranks on one device); timings are not meaningful
            os.environ["LOCAL_RANK"] = "0"
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
            dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    line = run_prefill(args, rank, world, cfg) if args.config == "c5" else run_ours(args, rank, world, cfg)
    if rank == 0 and line is not None:
        if world == 1 and not args.no_cpu_baseline and args.config != "c5":   # rank 0 at N = 1 only
            cores = os.cpu_count() or 1
            sample = args.cpu_sample or 2 * cores
            try:
                line["cpu_baseline"] = cpu_baseline(cfg, sample, cores, per_head=args.policy == "per-head")
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "error": repr(e)}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
