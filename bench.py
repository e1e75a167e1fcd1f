#!/usr/bin/env python3
"""Hybrid-batch attention bench (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_b64] [--impl pod|reference]

A "step" is one hybrid-batch attention layer: the fused POD launch (SM-aware
prefill + decode CTAs, then the split merge) over one synthetic Llama-3-8B
batch resident in HBM.  At N > 1 (torchrun, one rank per GPU) the layer is
sharded by KV-head group (TP = N, each rank owns Hkv/N whole KV heads) and the
per-rank outputs are assembled with one NCCL all-gather inside the step.

Rank 0 prints ONE JSON line.  `value` is the fused layer latency in us
(lower is better, max over ranks); the line also carries serial / prefill-alone
/ decode-alone latencies, the speedup over serial, the combined-roofline
fraction, e2e through the C ABI with host buffers, the roofline object for the
fused kernel and the CPU reference baseline (oracle/_ref, test infrastructure,
timed on a bounded sample on this host's cores).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "hybrid-batch attention µs/layer, speedup vs serial, % of combined roofline"

# name -> (Hq, Hkv, chunk, offset, decode batch, decode ctx)
CONFIGS = {
    "c1": (32, 8, 512, 1536, 8, 2048),
    "c2_b8": (32, 8, 1024, 15360, 8, 16384),
    "c2_b16": (32, 8, 1024, 15360, 16, 16384),
    "c2_b32": (32, 8, 1024, 15360, 32, 16384),
    "c2_b64": (32, 8, 1024, 15360, 64, 16384),
    "c4": (32, 32, 2048, 2048, 128, 4096),
    # one rank's share of C2 B=64 under KV-head-group TP (what each GPU runs at T = 2/4/8)
    "c3_tp2_rank": (16, 4, 1024, 15360, 64, 16384),
    "c3_tp4_rank": (8, 2, 1024, 15360, 64, 16384),
    "c3_tp8_rank": (4, 1, 1024, 15360, 64, 16384),
}
DEFAULT_CONFIG = "c2_b64"


def peaks():
    p = {"hbm_gbs": 6538.9, "bf16_tflops": 1665.7, "bf16_tflops_sustained": 1381.4, "source": "measured"}
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        j = json.loads(f.read_text())
        for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained"):
            if k in j:
                p[k] = float(j[k])
    else:
        p.update(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0, source="fallback")
    return p


def work(hq, hkv, chunk, off, b, ctx, d=128):
    """Algorithmic work of one layer: prefill FLOPs (QK^T + PV,
    causal, masked work excluded) and decode bytes (bf16 K+V + Q + fp32 O + LSE)."""
    flops = 4.0 * d * hq * (chunk * off + chunk * (chunk + 1) / 2.0)
    dbytes = b * (2.0 * ctx * hkv * d * 2) + b * hq * d * 2 + b * hq * d * 4 + b * hq * 4
    return flops, dbytes


class ClockSampler:
    """SM clocks + throttle reasons sampled every 2 ms (NVML) while the timed
    phases run; falls back to nvidia-smi polling when NVML is unavailable."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self._stop = threading.Event()

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for n, bit in bits.items():
                            if r & bit:
                                self.reasons.add(n)
                    except Exception:
                        pass
                    self._stop.wait(0.002)

            self._thread = threading.Thread(target=loop, daemon=True)
            self._thread.start()
        except Exception:
            self._stop = None
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


# ----------------------------------------------------------- CPU baseline --
_CPU_INPUTS = {}


def _cpu_layer_inputs(hq, hkv, chunk, off, b, ctx, threads, seed=7, rows_per_block=64):
    """Full-layer inputs for the reference's CPU path, built once per process (the step
    times only the reference's attention, not input generation):
      prefill: one shard per (KV head, block of `rows_per_block` chunk rows) --
               tiled_prefill_attention on QueryChunk(rows, group, d, off + r0) against
               that KV head's cache prefix, an exact restriction of the full call by GQA
               consistency (test_attention.cpp:252-270) and row independence
               (attention.hpp:183-212);
      decode:  one shard per (request, KV head) -- decode_attention over ctx keys.
    Decode caches are drawn from a pool of min(B*Hkv, 4*threads) distinct [ctx][1][d]
    arrays (each 2*ctx*d*8 bytes, far beyond the CPU caches), so the 16 GB of distinct
    fp64 caches of C2 B=64 need not be materialised."""
    import numpy as np

    key = (hq, hkv, chunk, off, b, ctx, threads)
    if key in _CPU_INPUTS:
        return _CPU_INPUTS[key]
    d, G = 128, hq // hkv
    rng = np.random.default_rng(seed)
    pf, dc, keep = [], [], []
    if chunk:
        kvlen = off + chunk
        for h in range(hkv):
            k = rng.uniform(-1, 1, (kvlen, 1, d))
            v = rng.uniform(-1, 1, (kvlen, 1, d))
            keep += [k, v]
            for r0 in range(0, chunk, rows_per_block):
                rows = min(rows_per_block, chunk - r0)
                q = rng.uniform(-1, 1, (rows, G, d))
                o = np.zeros((rows, G * d))
                n = off + r0 + rows
                pf.append(dict(kind=0, group=G, rows=rows, offset=off + r0, q=q, k=k[:n], v=v[:n], out=o))
    if b:
        npool = min(b * hkv, 4 * threads)
        pool = [(rng.uniform(-1, 1, (ctx, 1, d)), rng.uniform(-1, 1, (ctx, 1, d))) for _ in range(npool)]
        keep += pool
        for i in range(b * hkv):
            k, v = pool[i % npool]
            dc.append(dict(kind=1, group=G, rows=1, offset=0, q=rng.uniform(-1, 1, (G, d)), k=k, v=v,
                           out=np.zeros((G, d))))
    _CPU_INPUTS[key] = (pf, dc, keep)
    return _CPU_INPUTS[key]


def cpu_reference_layer(hq, hkv, chunk, off, b, ctx, threads=None, max_core_s=900.0):
    """Times ONE FULL layer of the reference's own tiled_prefill_attention /
    decode_attention (oracle/_ref, compiled from /root/reference; its parallel_for over
    all host threads, tile_q = tile_kv = 64) -- no sampling, no extrapolation.
    Layers estimated above `max_core_s` core-seconds (C5 extremes) fall back to
    `cpu_reference_sample`.  Returns (us_per_layer, threads, description, wall_s)."""
    import numpy as np

    from oracle import pyoracle as O

    if not O.ref_available():
        raise RuntimeError("oracle/_ref missing")
    threads = threads or os.cpu_count() or 1
    d, G = 128, hq // hkv
    # single-core rate of the reference's inner loops (one small decode shard)
    rng = np.random.default_rng(1)
    kcal = rng.uniform(-1, 1, (4096, 1, d))
    t = O.run_shards([dict(kind=1, group=G, rows=1, offset=0, q=rng.uniform(-1, 1, (G, d)), k=kcal, v=kcal,
                           out=np.zeros((G, d)))], d, math.sqrt(d), 64, 64, 1)
    rate1 = G * 4096 / max(t, 1e-6)
    pairs = hkv * G * (chunk * off + chunk * (chunk + 1) / 2.0) + b * hkv * G * float(ctx)
    if pairs / rate1 > max_core_s:
        us, thr, desc, wall = cpu_reference_sample(hq, hkv, chunk, off, b, ctx, target_s=max_core_s / 4,
                                                   threads=threads)
        return us, thr, desc + f" (full layer ~{pairs / rate1:.0f} core-s > {max_core_s:.0f}: sampled)", wall
    pf, dc, _ = _cpu_layer_inputs(hq, hkv, chunk, off, b, ctx, threads)
    t_pf = O.run_shards(pf, d, math.sqrt(d), 64, 64, threads) if pf else 0.0
    t_dc = O.run_shards(dc, d, math.sqrt(d), 64, 64, threads) if dc else 0.0
    desc = (f"full layer, no extrapolation: {len(pf)} prefill shards (KV head x 64-row block, "
            f"{G} q heads each) + {len(dc)} decode (request, KV head) shards at {ctx} keys; "
            f"prefill {t_pf:.2f} s + decode {t_dc:.2f} s wall on {threads} threads (the reference's parallel_for; "
            f"each shard builds its KVCache, as the reference API requires)")
    return (t_pf + t_dc) * 1e6, threads, desc, t_pf + t_dc


def cpu_reference_sample(hq, hkv, chunk, off, b, ctx, target_s=12.0, threads=None, seed=7):
    """Times the reference's own tiled_prefill_attention / decode_attention
    (oracle/_ref, built from /root/reference) on a bounded, representative sample
    of the layer and extrapolates linearly in (q-head row, key) pairs.  Only used
    for layers too large to time whole (cpu_reference_layer).
    Returns (us_per_layer, threads, sample_description, wall_s)."""
    import numpy as np

    from oracle import pyoracle as O

    if not O.ref_available():
        raise RuntimeError("oracle/_ref missing")
    threads = threads or os.cpu_count() or 1
    d = 128
    G = hq // hkv
    scale = math.sqrt(d)
    rng = np.random.default_rng(seed)
    pf_pairs = hkv * G * (chunk * off + chunk * (chunk + 1) / 2.0)
    dec_pairs = b * hkv * G * float(ctx)
    total_pairs = pf_pairs + dec_pairs
    kcal = rng.uniform(-1, 1, (4096, 1, d)).round(3)
    qcal = rng.uniform(-1, 1, (G, d))
    out = np.zeros((G, d))
    t = O.run_shards([dict(kind=1, group=G, rows=1, offset=0, q=qcal, k=kcal, v=kcal, out=out)], d, scale, 64, 64, 1)
    rate1 = G * 4096 / max(t, 1e-6)
    budget_pairs = target_s * rate1
    n_shards = max(2 * threads, 8)
    pf_share = pf_pairs / total_pairs
    shards = []
    keep = []
    pf_budget = budget_pairs * pf_share
    dec_budget = budget_pairs - pf_budget
    sample_pairs = 0.0
    npf = n_shards if chunk > 0 else 0
    if npf:
        rows_per = max(1, int(pf_budget / npf / (G * (off + chunk / 2.0))))
        rows_per = min(rows_per, chunk)
        for i in range(npf):
            r0 = int((chunk - rows_per) * i / max(1, npf - 1))
            kv = off + r0 + rows_per
            k = rng.uniform(-1, 1, (kv, 1, d))
            v = rng.uniform(-1, 1, (kv, 1, d))
            q = rng.uniform(-1, 1, (rows_per, G, d))
            o = np.zeros((rows_per, G * d))
            shards.append(dict(kind=0, group=G, rows=rows_per, offset=off + r0, q=q, k=k, v=v, out=o))
            keep += [k, v, q, o]
            sample_pairs += G * sum(off + r0 + r + 1 for r in range(rows_per))
    ndec = n_shards if b > 0 else 0
    if ndec:
        dctx = int(min(ctx, max(16, dec_budget / ndec / G)))
        for i in range(ndec):
            k = rng.uniform(-1, 1, (dctx, 1, d))
            v = rng.uniform(-1, 1, (dctx, 1, d))
            q = rng.uniform(-1, 1, (G, d))
            o = np.zeros((G, d))
            shards.append(dict(kind=1, group=G, rows=1, offset=0, q=q, k=k, v=v, out=o))
            keep += [k, v, q, o]
    else:
        dctx = 0
    pf = [s for s in shards if s["kind"] == 0]
    dc = [s for s in shards if s["kind"] == 1]
    t_pf = O.run_shards(pf, d, scale, 64, 64, threads) if pf else 0.0
    t_dc = O.run_shards(dc, d, scale, 64, 64, threads) if dc else 0.0
    us = 0.0
    if pf:
        us += t_pf * (pf_pairs / sample_pairs) * 1e6
    if dc:
        us += t_dc * (dec_pairs / (len(dc) * G * dctx)) * 1e6
    desc = (f"{len(pf)} prefill row-blocks x {pf[0]['rows'] if pf else 0} rows (1 KV head, {G} q heads) + "
            f"{len(dc)} decode (request, KV head) shards at {dctx} keys; {t_pf + t_dc:.1f} s wall on {threads} "
            f"threads; extrapolated linearly in (q-head row, key) pairs to the full layer")
    return us, threads, desc, t_pf + t_dc


# --------------------------------------------------------------- GPU arm ---
def _max_over_ranks(t, dev):
    import torch
    import torch.distributed as dist

    x = torch.tensor([t], device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return float(x.item())


def _timer(dev, flush, world):
    import torch
    import torch.distributed as dist

    def timed(step, steps, warmup):
        """Mean device time of `steps` calls of step() (CUDA events on the launching
        stream, L2 flushed before each), max over ranks."""
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        # the device first spins while the host enqueues every timed step: a step shorter
        # than its own host launch path (C1: ~56 us on the device) then still runs back to
        # back, and the events time the device, not the Python / ctypes enqueue (host
        # overhead is what the e2e number carries)
        if not os.environ.get("BENCH_NO_PRESLEEP"):  # (A/B switch for the timing method itself)
            torch.cuda._sleep(int(min(steps, 200) * 4e5))  # ~0.2 ms of GPU clock per step
        for i in range(steps):
            flush.zero_()  # L2 flush (512 MB > 126 MB L2), outside the timed events
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
        ms = [a.elapsed_time(e) for a, e in ev]
        t = sum(ms) / len(ms)
        if world > 1:
            t = _max_over_ranks(t, dev)
            dist.barrier()
        return t, ms

    return timed


def serial_candidates(batch):
    """Every way the repo can run the prefill alone and the decode alone: both POD
    kernels, both pair-engine tile widths, prefill split caps 1..8 (gpu_sim.hpp:496-506
    defines serial as prefill-then-decode with the same kernels; the honest comparator
    takes the fastest of each)."""
    import paper_2410_18038_b200 as pkg
    from paper_2410_18038_b200._abi import POD_POLICY_COMPLEMENT, POD_POLICY_WARPSPEC

    pf, dc = [], []
    if batch.prefill is not None:
        for tk in (32, 64):
            for cap in (1, 2):
                pf.append((f"warpspec/{tk}-key/cap{cap}",
                           pkg.PlanOptions(policy=POD_POLICY_WARPSPEC, prefill_tile_keys=tk, split_wave_cap=cap)))
        for cap in (1, 2, 4, 8):
            pf.append((f"complement/cap{cap}", pkg.PlanOptions(policy=POD_POLICY_COMPLEMENT, split_wave_cap=cap)))
    if batch.decodes:
        dc = [("warpspec", pkg.PlanOptions(policy=POD_POLICY_WARPSPEC)),
              ("complement", pkg.PlanOptions(policy=POD_POLICY_COMPLEMENT))]
    return pf, dc


def bench_oproj(wl, gb, world, rank, dev, timed, hq, d=128, seed=7):
    """The o_proj consumer on this rank's attention output: a row-
    parallel GEMM Y += O_rank W_rank with the reduce-scatter fused into its epilogue
    (tp.oproj -> pod_oproj_run), timed like the layer.  N = 1: the plain GEMM, beside
    torch.matmul (cuBLAS).  N > 1: every rank reduces into the row owners' Y through
    peer-mapped symmetric memory (no all-gather of O at all); rank 0 checks its rows."""
    import torch
    import torch.distributed as dist

    from paper_2410_18038_b200.tp import oproj

    hidden = hq * d
    o = torch.cat([t for t in (gb.outputs.o_prefill, gb.outputs.o_decode) if t is not None]).reshape(gb.tokens, -1)
    o = o.to(torch.bfloat16).contiguous()
    kr = o.shape[1]
    g = torch.Generator(device=dev).manual_seed(seed)
    w_full = ((torch.rand(hidden, hidden, generator=g, device=dev) * 2 - 1) / 64).to(torch.bfloat16)
    w = w_full[rank * kr:(rank + 1) * kr].contiguous()
    flops = 2.0 * gb.tokens * kr * hidden
    if world == 1:
        y = torch.empty(gb.tokens, hidden, device=dev)
        t, _ = timed(lambda: oproj(o, w, [y]), 10, 3)
        t_ref, _ = timed(lambda: torch.matmul(o, w), 10, 3)
        torch.cuda.synchronize()
        err = float((y - o.float() @ w.float()).abs().max() / (o.float() @ w.float()).abs().max())
        return {"us": round(t * 1000, 2), "tflops": round(flops / (t * 1e-3) / 1e12, 1),
                "torch_matmul_us": round(t_ref * 1000, 2), "rel_err_vs_torch_fp32": err,
                "shape": f"[{gb.tokens}][{kr}] x [{kr}][{hidden}] bf16 -> fp32", "fused_reduce_scatter": False}
    if dist.get_backend() != "nccl":
        return {"skipped": "peer-mapped symmetric memory needs the NCCL / CUDA backend"}
    import torch.distributed._symmetric_memory as symm_mem

    rows = (gb.tokens + world - 1) // world
    y = symm_mem.empty(rows, hidden, dtype=torch.float32, device=dev)
    hdl = symm_mem.rendezvous(y, dist.group.WORLD)
    ptrs = [int(hdl.buffer_ptrs[r]) for r in range(world)]

    def step():
        oproj(o, w, ptrs, rows_per_rank=rows, accumulate=True)

    y.zero_()
    dist.barrier()
    step()
    torch.cuda.synchronize()
    dist.barrier()
    check = None
    o_all = torch.empty(world * gb.tokens * kr, dtype=torch.bfloat16, device=dev)  # (the check only)
    dist.all_gather_into_tensor(o_all, o.reshape(-1))
    o_full = o_all.view(world, gb.tokens, kr).permute(1, 0, 2).reshape(gb.tokens, world * kr)
    if rank == 0:
        ref = (o_full.float() @ w_full.float())[:rows]
        check = float((y[:min(rows, gb.tokens)] - ref).abs().max() / ref.abs().max())
    t, _ = timed(step, 10, 3)  # (the reductions accumulate across steps: timing only)
    return {"us": round(t * 1000, 2), "tflops_per_rank": round(flops / (t * 1e-3) / 1e12, 1),
            "shape": f"[{gb.tokens}][{kr}] x [{kr}][{hidden}] per rank, fused reduce-scatter over {world} ranks",
            "fused_reduce_scatter": True, "rank0_rel_err": check}


def run_pod(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2410_18038_b200 as pkg
    from paper_2410_18038_b200.hybrid import PodAttention
    from paper_2410_18038_b200.tp import (all_gather_bytes, assemble_layer, gather_buffers, layer_error,
                                          shard_heads, shard_workload)
    from paper_2410_18038_b200.workload import build_workload, make_batch

    hq, hkv, chunk, off, b, ctx = CONFIGS[args.config]
    if hkv % world:
        raise SystemExit(f"Hkv={hkv} not divisible by {world} GPUs")
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    full_shape = pkg.ModelShape(hq, hkv, 128, math.sqrt(128))
    shard = shard_heads(full_shape, rank, world)
    hq_r, hkv_r = shard.shape.num_q_heads, shard.shape.num_kv_heads
    # every rank draws the SAME seeded full layer and keeps its KV-head group
    full_batch = make_batch(full_shape, chunk=chunk, offset=off, decode_ctx=[ctx] * b)
    full_wl = build_workload(full_batch, device=dev)
    wl = shard_workload(full_wl, shard) if world > 1 else full_wl
    if world > 1 and rank != 0:
        del full_wl
        full_wl = None
        torch.cuda.empty_cache()
    batch = wl.batch
    odt = {"f32": torch.float32, "bf16": torch.bfloat16}[args.out_dtype]
    opts = pkg.PlanOptions(policy=args.policy, tile_mode=args.tile_mode, precision=args.precision,
                           decode_splits=args.decode_splits, split_wave_cap=args.split_wave_cap,
                           out_dtype={"f32": 0, "bf16": 1}[args.out_dtype],
                           prefill_tile_keys=args.prefill_tile_keys, prefill_s_buffers=args.prefill_s_buffers)
    op = PodAttention(batch, options=opts, device=local_rank)
    # the kernel writes straight into the all-gather send buffer (two, for the pipelined e2e)
    gbs = [gather_buffers(batch, world, odt, dev) for _ in range(2)]
    out = gbs[0].outputs
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    timed = _timer(dev, flush, world)

    def layer(mode, o=None, gb=None, stream=None):
        op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices,
               out=o or out, mode=mode, stream=stream)
        if world > 1:  # assemble the layer output: one all-gather of [tokens][Hq/T][d] + LSE over NVLink
            g = gb or gbs[0]
            all_gather_bytes(g.send, g.recv, world)

    # KV append (the write step before attention): the batch's new
    # K/V rows (chunk tokens + one per decode, read back from their slots) scattered
    # into the paged pools.  Reported beside the attention metric, not part of it.
    ix = wl.page_indices.cpu().tolist()
    ip = wl.page_indptr.cpu().tolist()
    slots = [(ix[ip[0] + t // 16], t % 16) for t in range(off, off + chunk)] if chunk else []
    slots += [(ix[ip[(1 if chunk else 0) + i] + (ctx - 1) // 16], (ctx - 1) % 16) for i in range(b)]
    pg = torch.tensor([p_ for p_, _ in slots], device=dev)
    sl = torch.tensor([s_ for _, s_ in slots], device=dev)
    k_rows = wl.k_pool[pg, :, sl, :].contiguous()
    v_rows = wl.v_pool[pg, :, sl, :].contiguous()

    def append():
        op.append_kv(k_rows[:chunk] if chunk else None, v_rows[:chunk] if chunk else None,
                     k_rows[chunk:] if b else None, v_rows[chunk:] if b else None,
                     wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices)

    t_append, _ = timed(append, args.steps, args.warmup)
    append_bytes = 2 * 2 * k_rows.numel() * k_rows.element_size()  # K + V, read + write

    sampler = ClockSampler(local_rank)
    with sampler:
        t_fused, ms_fused = timed(lambda: layer("fused"), args.steps, args.warmup)
        t_serial, _ = timed(lambda: layer("serial"), args.steps, args.warmup)
        t_pf, _ = timed(lambda: layer("prefill"), args.steps, args.warmup) if chunk else (0.0, [])
        t_dec, _ = timed(lambda: layer("decode"), args.steps, args.warmup) if b else (0.0, [])
        t_attn = timed(lambda: op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr,
                                      wl.page_indices, out=out), args.steps, args.warmup)[0] if world > 1 else t_fused
        # honest serial comparator: the fastest prefill-alone and decode-alone over every
        # kernel / tile width / split cap the repo has (no all-gather: attention only)
        best = {}
        if not args.no_serial_search:
            pf_c, dc_c = serial_candidates(batch)
            for role, cands, mode in (("prefill", pf_c, "prefill"), ("decode", dc_c, "decode")):
                for name, o in cands:
                    c_op = PodAttention(batch, options=o, device=local_rank)
                    c_out = c_op.alloc_outputs()
                    t, _ = timed(lambda: c_op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr,
                                                  wl.page_indices, out=c_out, mode=mode), args.steps, args.warmup)
                    if role not in best or t < best[role][0]:
                        best[role] = (t, name)
                    del c_op, c_out
    clocks = sampler.summary()

    # e2e through the C ABI with HOST buffers (pinned): every step copies its queries
    # H2D, runs the fused layer (+ the all-gather at N > 1) and copies its outputs
    # (O + LSE) D2H.  Steps are pipelined the way a serving loop runs them:
    # double-buffered device Q / O, the H2D of step i+1 and the D2H of step i-1 on their
    # own copy streams (separate copy engines) overlap the kernel of step i.  The paged
    # KV cache is device state.
    qp_h = wl.q_prefill.cpu().pin_memory() if chunk else None
    qd_h = wl.q_decode.cpu().pin_memory() if b else None
    q_dev = [(wl.q_prefill, wl.q_decode),
             (wl.q_prefill.clone() if chunk else None, wl.q_decode.clone() if b else None)]

    def _dev_out(g):  # what the step hands back to the host: this rank's O + LSE, or the gathered layer
        return [g.send] if world == 1 else [g.recv]

    host_out = [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in _dev_out(g)] for g in gbs]
    h2d = (qp_h.numel() * 2 if qp_h is not None else 0) + (qd_h.numel() * 2 if qd_h is not None else 0)
    d2h = sum(t.numel() * t.element_size() for t in _dev_out(gbs[0]))
    s_c = torch.cuda.current_stream(dev)
    s_h, s_d = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_h = [torch.cuda.Event() for _ in range(2)]
    ev_c = [torch.cuda.Event() for _ in range(2)]
    ev_d = [torch.cuda.Event() for _ in range(2)]
    for e in ev_c + ev_d:
        e.record(s_c)

    def e2e_step(i):
        j = i % 2
        qp, qd = q_dev[j]
        with torch.cuda.stream(s_h):  # H2D of this step's queries (buffer free once kernel i-2 is done)
            s_h.wait_event(ev_c[j])
            if qp_h is not None:
                qp.copy_(qp_h, non_blocking=True)
            if qd_h is not None:
                qd.copy_(qd_h, non_blocking=True)
            ev_h[j].record(s_h)
        s_c.wait_event(ev_h[j])
        s_c.wait_event(ev_d[j])  # O buffer j drained by the D2H of step i-2
        op.run(qp, qd, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, out=gbs[j].outputs, mode="fused",
               stream=s_c)
        if world > 1:
            all_gather_bytes(gbs[j].send, gbs[j].recv, world)
        ev_c[j].record(s_c)
        with torch.cuda.stream(s_d):  # D2H of this step's outputs
            s_d.wait_event(ev_c[j])
            for hsrc, dsrc in zip(host_out[j], _dev_out(gbs[j])):
                hsrc.copy_(dsrc, non_blocking=True)
            ev_d[j].record(s_d)

    for i in range(args.warmup):
        e2e_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(s_c)
    s_h.wait_event(t0)
    for i in range(args.steps):
        e2e_step(args.warmup + i)
    for e in ev_d:
        s_c.wait_event(e)  # the last step's D2H is inside the timed region
    t1.record(s_c)
    torch.cuda.synchronize()
    t_e2e = t0.elapsed_time(t1) / args.steps
    if world > 1:
        t_e2e = _max_over_ranks(t_e2e, dev)

    oproj_res = None
    if world > 1 and not args.oproj_tp:
        oproj_res = {"skipped": "the multi-rank reduce-scatter run is opt-in (--oproj-tp): symmetric-memory "
                                "peers are unvalidated on this one-GPU development setup"}
    elif not args.no_oproj:
        try:
            oproj_res = bench_oproj(wl, gbs[0], world, rank, dev, timed, hq)
        except Exception as e:  # reported, never fatal for the attention number
            oproj_res = {"error": f"{type(e).__name__}: {e}"[:300]}

    # TP self-check: the assembled layer (every rank's kernel + the all-gather) against a
    # TP1 run of the same seeded layer on rank 0 (north-star tolerance, 2e-3)
    tp_check = None
    if world > 1:
        layer("fused")
        torch.cuda.synchronize()
        if rank == 0:
            o_tp, lse_tp = assemble_layer(gbs[0])
            ref_op = PodAttention(full_batch, options=pkg.PlanOptions(out_dtype=opts.out_dtype), device=local_rank)
            ro = ref_op.run(full_wl.q_prefill, full_wl.q_decode, full_wl.k_pool, full_wl.v_pool,
                            full_wl.page_indptr, full_wl.page_indices)
            torch.cuda.synchronize()
            o_ref = torch.cat([t for t in (ro.o_prefill, ro.o_decode) if t is not None])
            lse_ref = torch.cat([t for t in (ro.lse_prefill, ro.lse_decode) if t is not None])
            eo, el = layer_error(o_tp, lse_tp, o_ref, lse_ref, hq // hkv)
            tp_check = {"vs": "tp1 fused run of the same layer on rank 0", "o_rel_err": eo, "lse_abs_err": el,
                        "tol": 2e-3, "ok": bool(eo <= 2e-3 and el <= 2e-3)}
        dist.barrier()

    info = op.info
    launches_per_step = 1 + (1 if (info.num_merge_rows_prefill or info.num_merge_rows_decode) else 0)  # one merge launch
    # + the fp16 V shadow's conversion kernel (pod_plan.cpp: bf16 data, F16PV, a prefill on the
    # two-CTA kernel or the 64-key pair engine)
    if (chunk and args.precision == 2 and (info.policy == 3 or (info.policy == 7 and info.prefill_tile_keys == 64))):
        launches_per_step += 1
    res = dict(t_fused=t_fused, ms_fused=ms_fused, t_serial=t_serial, t_pf=t_pf, t_dec=t_dec, t_e2e=t_e2e,
               t_attn=t_attn, t_append=t_append, append_bytes=append_bytes, best=best, tp_check=tp_check,
               oproj=oproj_res,
               clocks=clocks, info=info, launches=launches_per_step, h2d=h2d, d2h=d2h, hq_r=hq_r, hkv_r=hkv_r)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="pod", choices=["pod", "reference"])
    ap.add_argument("--policy", type=int, default=8, help="POD_POLICY_*: 8 = AUTO (default), 7 = WARPSPEC, 3 = COMPLEMENT")
    ap.add_argument("--tile-mode", type=int, default=1)
    ap.add_argument("--precision", type=int, default=2, help="POD_PRECISION_*: 0 prefill P as bf16 hi+lo, 1 single bf16, 2 fp16 P x fp16 V")
    ap.add_argument("--out-dtype", default="f32", choices=["f32", "bf16"],
                    help="element type of the attention outputs (LSE stays fp32); f32 = the reference's")
    ap.add_argument("--decode-splits", type=int, default=0)
    ap.add_argument("--prefill-tile-keys", type=int, default=0, help="warp-specialised pair engine: 0 auto, 32 or 64")
    ap.add_argument("--prefill-s-buffers", type=int, default=0,
                    help="64-key pair engine: 0 auto, 1 single S (Q in TMEM), 2 double S (Q in smem)")
    ap.add_argument("--split-wave-cap", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-oproj", action="store_true", help="skip the o_proj consumer measurement")
    ap.add_argument("--oproj-tp", action="store_true",
                    help="at N > 1 also run the o_proj consumer's fused reduce-scatter over symmetric-memory peers")
    ap.add_argument("--no-serial-search", action="store_true",
                    help="skip the search for the fastest prefill-alone / decode-alone (serial_best_us)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    hq, hkv, chunk, off, b, ctx = CONFIGS[args.config]
    flops, dbytes = work(hq, hkv, chunk, off, b, ctx)
    pk = peaks()
    config = {"workload": f"{args.config}: Llama-3-8B-shaped layer ({hq} Q / {hkv} KV heads, d=128, bf16), "
                          f"prefill chunk {chunk} at offset {off} (context {off + chunk}) + {b} decodes at "
                          f"context {ctx}, paged KV (page 16, HND, random block tables)",
              "tp": args.gpus, "parallelism": f"kv-head-group tp{args.gpus}", "l2": "flushed between steps "
              "(512 MB write); KV working set also exceeds L2", "page_size": 16}

    if args.impl == "reference":
        if rank != 0:
            return
        steps = max(1, args.steps)
        vals = []
        for i in range(args.warmup + steps):
            us, thr, desc, wall = cpu_reference_layer(hq, hkv, chunk, off, b, ctx)
            if i >= args.warmup:
                vals.append(us)
        v = sum(vals) / len(vals)
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "us/layer", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": round(v / 1000.0, 3), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (uniform[-1,1))",
            "config": config,
            "cpu_baseline": {"value": round(v, 1), "unit": "us/layer", "cores": thr, "kind": "reference",
                             "sample": desc},
            "e2e": {"value": round(v, 1), "unit": "us/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # one rank per GPU; --dist-backend gloo with more ranks than GPUs is a plumbing
        # check of the TP path on a 1-GPU box (ranks share the device), never a number
        local_rank = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(args.dist_backend)
    r = run_pod(args, rank, world, local_rank)
    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # per-rank roofline (each rank owns 1/world of the heads)
    flops_r, dbytes_r = flops / world, dbytes / world
    t_pf_roof = flops_r / (pk["bf16_tflops"] * 1e12) * 1e6
    t_dec_roof = dbytes_r / (pk["hbm_gbs"] * 1e9) * 1e6
    roof_us = max(t_pf_roof, t_dec_roof)
    us = r["t_fused"] * 1000.0
    bound = "hbm" if t_dec_roof >= t_pf_roof else "tensor"
    if bound == "hbm":
        achieved = dbytes_r / (us * 1e-6) / 1e9
        peak, unit = pk["hbm_gbs"], "GB/s"
    else:
        achieved = flops_r / (us * 1e-6) / 1e12
        peak, unit = pk["bf16_tflops"], "TFLOP/s"
    traffic = None  # DRAM bytes of one fused launch from the committed ncu capture of this config
    if args.config == DEFAULT_CONFIG and world == 1:
        caps = sorted((ROOT / "profiles").glob("round*/fused_traffic.json"))
        if caps:
            traffic = json.loads(caps[-1].read_text()).get("dram_bytes_per_launch")
    cpu = None
    if not args.no_cpu_baseline and world == 1:  # the CPU baseline runs on rank 0 at N = 1 only
        try:
            cus, thr, desc, _ = cpu_reference_layer(hq, hkv, chunk, off, b, ctx)
            cpu = {"value": round(cus, 1), "unit": "us/layer", "cores": thr, "kind": "reference", "sample": desc}
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": "us/layer", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    info = r["info"]
    serial_best = sum(v[0] for v in r["best"].values()) if r["best"] else None
    line = {
        "metric": METRIC, "value": round(us, 2), "unit": "us/layer", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(r["t_fused"], 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (splitmix64 uniform[-1,1) -> bf16)",
        "config": config,
        "serial_us": round(r["t_serial"] * 1000, 2),
        "speedup_vs_serial": round(r["t_serial"] / r["t_fused"], 3),
        "prefill_alone_us": round(r["t_pf"] * 1000, 2), "decode_alone_us": round(r["t_dec"] * 1000, 2),
        "fused_vs_max_alone": round(r["t_fused"] / max(r["t_pf"], r["t_dec"], 1e-9), 3),
        "serial_best_us": round(serial_best * 1000, 2) if serial_best else None,
        "speedup_vs_best_serial": round(serial_best / r["t_fused"], 3) if serial_best else None,
        "serial_best": {k: {"us": round(v[0] * 1000, 2), "kernel": v[1]} for k, v in r["best"].items()},
        "combined_roofline_us": round(roof_us, 2), "combined_roofline_frac": round(roof_us / us, 4),
        "prefill_tensor_frac_alone": round(t_pf_roof / max(r["t_pf"] * 1000, 1e-9), 4) if chunk else None,
        # the same against the fastest prefill-alone of any kernel (serial_best.prefill)
        "prefill_tensor_frac_best": (round(t_pf_roof / (r["best"]["prefill"][0] * 1000), 4)
                                     if chunk and "prefill" in r["best"] else None),
        "decode_hbm_frac_alone": round(t_dec_roof / max(r["t_dec"] * 1000, 1e-9), 4) if b else None,
        "tokens_per_s": round((chunk + b) / (us * 1e-6), 1),
        "plan": {"prefill_ctas": info.num_prefill_ctas, "decode_ctas": info.num_decode_ctas,
                 "prefill_splits": info.prefill_splits, "decode_splits": info.decode_splits,
                 "ratio": f"{info.prefill_ratio}:{info.decode_ratio}", "smem_per_cta": info.smem_bytes,
                 "policy": {3: "complement", 7: "warpspec"}.get(info.policy, info.policy), "split_wave_cap": info.config.split_wave_cap, "prefill_tile_keys": info.prefill_tile_keys, "prefill_s_buffers": info.prefill_s_buffers, "prefill_p": {0: "bf16 hi+lo", 1: "bf16", 2: "fp16 (V -> fp16: " + ("one shadow pass per launch)" if r["launches"] > 1 + (1 if (info.num_merge_rows_prefill or info.num_merge_rows_decode) else 0) else "per tile in smem)")}[args.precision], "out_dtype": args.out_dtype},
        "roofline": {"bound": bound, "achieved": round(achieved, 1), "peak": peak, "unit": unit,
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": {7: "pod_sm_kernel (+merge)"}.get(r["info"].policy, "pod_fused_kernel (+merge)"),
                     "peak_source": pk["source"]},
        "cpu_baseline": cpu,
        "kv_append": {"us": round(r["t_append"] * 1000, 2), "bytes": r["append_bytes"],
                      "gb_s": round(r["append_bytes"] / (r["t_append"] * 1e-3) / 1e9, 1),
                      "note": "pod_attn_append_kv of the batch's new K/V tokens into the paged pools (not in value)"},
        "e2e": {"value": round(r["t_e2e"] * 1000, 2), "unit": "us/layer", "h2d_bytes_per_step": r["h2d"],
                "d2h_bytes_per_step": r["d2h"]},
        "gpu_launches": r["launches"] * args.steps,
        "tp_check": r["tp_check"],
        "oproj": r["oproj"],
        "attention_only_us": round(r["t_attn"] * 1000, 2),
        "clocks": r["clocks"],
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
