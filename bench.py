#!/usr/bin/env python3
"""bench.py -- 2-bit-KV decode throughput of the AKVQ-VL hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl akvq|reference]

One "step" = one decode step of the whole model for the whole batch: for every
layer, append the new token's K/V (flushing a G-block to 2 bits when it leaves the
window) and run single-query decode attention over that layer's packed cache
(SURVEY 8(a) rows a2-a7), plus the all-gather of outputs across ranks (a8).
Prompts are quantized (rows a2-a5, incl. saliency) before timing; that prefill is
timed separately and reported under "prefill".

Default workload: BJ:9's batch sweep at LLaVA-1.5-7B shape, batch 64 ("sweep@b64":
32 layers, 32 MHA heads, d 128, 3-image prompt of 1848 tokens), the largest
configuration BASELINE.json's metric is quoted on that fits one GPU.  Synthetic
inputs (paper_2501_15021_b200/synth.py) stand in for MileBench prompts.

Multi-GPU: launched by torchrun; rank r owns a contiguous slice of the global
units (batch x kv-head, BJ:5).  Units are independent (no data-path collective),
so by default every rank runs the full per-GPU workload on its own batch rows
("weak" scaling: global batch = N x 64); --scaling strong splits a fixed batch.
Outputs are all-gathered with NCCL once per step (shard.OutputGather, row a8).  Timing: CUDA events on the
launching stream with a barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2501_15021_b200 import shard, synth  # noqa: E402

METRIC = "2-bit-KV decode tokens/s and attention HBM GB/s vs peak at 1/2/4/8 B200"


def _peaks():
    p = {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md: 6.65 TB/s)"}
    f = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(f):
        with open(f) as fh:
            j = json.load(fh)
        p = {"hbm_gbs": float(j["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)",
             "sm_max_mhz": j.get("sm_max_mhz")}
    return p


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


# ----------------------------------------------------------------- byte model
def decode_bytes_per_unit(w, kind, L, n_q, side):
    """Algorithmic bytes one decode reads/writes for one unit:
    2-bit codes + K meta (8 B/channel/block) + V meta (8 B/group/token) + bitmask
    for [0, n_q); 16-bit ring rows; side rows; q in, fp32 out."""
    d, G = w.d, w.G
    ng = d // G
    b = n_q * (2 * d / 4 + 8 * d / G + 8 * ng + 1 / 8)
    b += (L - n_q) * 4 * d
    b += side * (4 * d if kind == 1 else d + 16 * ng)
    b += w.g * d * (2 + 4)
    return b


def prefill_bytes_per_unit(w, kind, L0):
    """Prefill quantize: read K,V rows (16-bit) + types/colsum; write packed pages,
    ring rows and side rows."""
    d, G = w.d, w.G
    ng = d // G
    n_q = (L0 - w.R) // G * G if L0 > w.R else 0
    rd = L0 * 4 * d + (L0 * 4 * w.g if kind == 1 else L0)
    wr = n_q * (2 * d / 4 + 8 * d / G + 8 * ng) + (L0 - n_q) * 4 * d
    return rd + wr


# ----------------------------------------------------------------- CPU oracle leg
class OracleSample:
    """The oracle (as it stands, never tuned) on the host cores, on a bounded sample
    of the workload: `n_units` units of one PSA layer, prefilled once; each step is
    one decode step (append + attention) of those units, extrapolated to the whole
    batch and all layers (tokens/s)."""

    def __init__(self, w, n_units=16, layer=2):
        import oracle
        oracle.build()
        self.oracle, self.w, self.layer = oracle, w, layer
        U = w.U
        self.units = sorted(set(int(round(i * (U - 1) / max(1, n_units - 1)))
                                for i in range(n_units)))
        kind = w.kind(layer)
        ocfg = oracle.OracleConfig(len(self.units), w.g, w.d, w.G, w.R, w.capacity, w.top_k,
                                   kind, oracle.BF16 if w.dtype == "bf16" else oracle.FP16,
                                   w.clip2, w.clip4)
        self.oc = oracle.OracleCache(ocfg)
        inp = synth.layer_inputs(w, layer, units=self.units, device="cpu")
        self.oc.prefill(synth.to_u16(inp["K"]), synth.to_u16(inp["V"]), inp["types"].numpy(),
                        inp["colsum"].numpy())
        self.steps, self.t_tot = 0, 0.0

    def step(self) -> float:
        """One timed oracle decode step; returns the extrapolated tokens/s."""
        w = self.w
        if self.oc.L >= w.capacity:
            raise RuntimeError("oracle sample ran out of capacity")
        di = synth.decode_inputs(w, self.layer, self.steps, units=self.units, device="cpu")
        k, v, q = synth.to_u16(di["k"]), synth.to_u16(di["v"]), synth.to_u16(di["q"])
        t0 = time.perf_counter()
        self.oc.append(k, v, di["types"].numpy())
        self.oc.decode(q)
        dt = time.perf_counter() - t0
        self.steps += 1
        self.t_tot += dt
        return w.batch / (dt / len(self.units) * w.U * w.n_layers)

    def describe(self) -> str:
        w = self.w
        return (f"oracle decode steps (append + attention) of {len(self.units)} of {w.U} "
                f"units of layer {self.layer}, {self.steps} steps in {self.t_tot:.3f} s; "
                f"extrapolated x{w.U}/{len(self.units)} units x{w.n_layers} layers")

    @property
    def cores(self) -> int:
        return self.oracle.nthreads()


def oracle_baseline(w, seconds=10.0, max_steps=250):
    """cpu_baseline leg of the GPU run: ~10-30 s of oracle work (prefill of the
    sampled units plus up to `seconds` of timed decode steps)."""
    smp = OracleSample(w, n_units=128)
    vals = []
    while smp.steps < max_steps and smp.t_tot < seconds and smp.oc.L < w.capacity:
        vals.append(smp.step())
    val = len(vals) / sum(1.0 / v for v in vals)
    return {"value": val, "unit": "tokens/s", "cores": smp.cores, "kind": "oracle",
            "sample": smp.describe()}


def workload_config(args, w, w1, world, n_layers):
    """The `config` object of both arms' JSON lines (the workload, no model keys)."""
    return {"workload": w1.name, "source": "BJ:9 batch sweep at LLaVA-1.5-7B shape"
            if w1.name.startswith("sweep") else f"synth.{w1.name}",
            "layers": n_layers, "global_batch": w.batch,
            "per_gpu_batch": w.batch // world if args.scaling == "weak" else None,
            "heads": w.hq, "kv_heads": w.hkv, "head_dim": w.d, "prompt_tokens": w.L0,
            "group": w.G, "residual": w.R, "top_k": w.top_k,
            "tsa_layers": list(w.tsa_layers), "kv_bits": 2,
            "k_axis": "per-" + args.k_axis, "pivots": args.pivots,
            "parallelism": f"units (batch x kv-head) sharded over {world} GPU(s)"}


def run_reference(args, w, rank):
    """--impl reference: the oracle as the reference arm, rank 0 only."""
    if rank != 0:
        return
    smp = OracleSample(w, n_units=32)
    n = min(args.warmup + args.steps, w.capacity - smp.oc.L)
    times = []
    for i in range(n):
        v = smp.step()
        if i >= args.warmup:
            times.append(1.0 / v)
    val = len(times) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
            "ms_per_step": 1000.0 * w.batch / val, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(args, w, w, max(1, args.gpus), w.n_layers),
                           l2="n/a (CPU oracle)"),
            "extrapolated": True,
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": smp.cores,
                             "kind": "oracle", "sample": smp.describe(), "extrapolated": True},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU leg
def emulate_rank_shape(ak, synth, wr, n_layers, dt, args, dev, steps=10, warmup=3):
    """Decode-step time of one rank's share of a strong-scaled batch, on this GPU:
    prefill every layer for the smaller batch, then time `steps` fused steps
    issued through the C ABI, and `steps` replays of the same step captured once
    in a CUDA graph (AKVQ_OPT_DEVICE_L caches, inputs copied into the captured
    buffers outside the timed replays)."""
    cap = wr.L0 + warmup + 2 * steps + 4
    caches = []
    for layer in range(n_layers):
        cfg = ak.make_config(wr.U, wr.g, wr.d, wr.G, wr.R, cap, wr.top_k, wr.kind(layer), dt,
                             wr.clip2, wr.clip4, 1 if args.k_axis == "token" else 0)
        lc = ak.LayerCache(cfg, device=dev, options=ak.AKVQ_OPT_DEVICE_L)
        inp = synth.layer_inputs(wr, layer, device=dev)
        lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
        del inp
        caches.append(lc)
    ins = []
    for s in range(warmup + steps):
        per = [synth.decode_inputs(wr, layer, s, device=dev) for layer in range(n_layers)]
        ins.append(per)
    outs = [torch.empty((wr.U, wr.g, wr.d), dtype=torch.float32, device=dev) for _ in range(n_layers)]
    for s in range(warmup):
        for layer, lc in enumerate(caches):
            di = ins[s][layer]
            lc.step(di["k"], di["v"], di["q"], di["types"], out=outs[layer])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(warmup, warmup + steps):
        for layer, lc in enumerate(caches):
            di = ins[s][layer]
            lc.step(di["k"], di["v"], di["q"], di["types"], out=outs[layer])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    # one step captured in a CUDA graph, replayed (no block flush inside the window)
    gms = None
    if all(lc.L - wr.R - lc.n_q + steps + 1 < wr.G for lc in caches):
        bufs = [{k_: v_.clone() for k_, v_ in ins[warmup][layer].items()} for layer in range(n_layers)]
        s_ = torch.cuda.Stream(device=dev)
        s_.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s_):
            with torch.cuda.graph(graph, stream=s_):
                for layer, lc in enumerate(caches):
                    b_ = bufs[layer]
                    lc.step(b_["k"], b_["v"], b_["q"], b_["types"], out=outs[layer])
        torch.cuda.current_stream().wait_stream(s_)
        graph.replay()                                     # warm replay
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        gms = e0.elapsed_time(e1) / steps
        for lc in caches:                                  # host mirrors: capture counted 1
            ak.akvq_cache_advance(lc.handle, steps)
    del caches
    torch.cuda.empty_cache()
    return {"workload": wr.name, "ms_per_step": ms, "tokens_per_s": wr.batch / (ms * 1e-3),
            "ms_per_layer": ms / n_layers, "graph_ms_per_step": gms,
            "graph_tokens_per_s": wr.batch / (gms * 1e-3) if gms else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="sweep@b64")
    ap.add_argument("--impl", default="akvq", choices=["akvq", "reference"])
    ap.add_argument("--layers", type=int, default=0, help="override layer count (debug only)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank runs the full per-GPU workload on its own batch "
                         "rows (units are independent, task rule 5); strong: the global "
                         "batch is fixed and split")
    ap.add_argument("--pivots", default="colsum", choices=["colsum", "massive"],
                    help="PSA saliency: column-sum top-k (BJ:5, graded) or massive-activation "
                         "pivots from a synthetic residual stream (P:209-213, NEXT-2)")
    ap.add_argument("--k-axis", default="channel", choices=["channel", "token", "token-exact"],
                    help="K quantization axis: per channel (R1, graded), per token (P:246), or "
                         "per token with the exact residual window (R26, NEXT-1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-strong-emulation", action="store_true",
                    help="skip the 1-GPU emulation of the strong-scaling per-rank shapes")
    ap.add_argument("--stream-only", action="store_true",
                    help="profiling: kernels stream their bytes but skip the math (invalid outputs)")
    ap.add_argument("--skip-rows", action="store_true", help="profiling: no row kernel (invalid)")
    ap.add_argument("--skip-pages", action="store_true", help="profiling: no page kernel (invalid)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    w = synth.get(args.workload)

    if args.impl == "reference":
        run_reference(args, w, rank)
        return
    w1 = w                                              # per-GPU workload (the N = 1 config)
    if args.scaling == "weak" and world > 1:
        w = w1.with_batch(w1.batch * world)             # global: N x the batch rows

    from paper_2501_15021_b200 import akvq as ak

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    n_layers = args.layers or w.n_layers
    U = w.U
    lo, hi = shard.unit_range(U, world, rank)        # contiguous b-major unit slice
    Ul = hi - lo
    units = list(range(lo, hi))
    dt = ak.AKVQ_BF16 if w.dtype == "bf16" else ak.AKVQ_FP16
    need_steps = args.warmup + 2 * args.steps
    nq0 = (w.L0 - w.R) // w.G * w.G if w.L0 > w.R else 0
    first_flush = w.R + nq0 + w.G - w.L0              # decode steps until the first flush
    cap = w.L0 + max(w.decode_steps, need_steps, first_flush + 2)
    stream = torch.cuda.current_stream()

    # ---------------- prefill every layer (timed separately)
    caches, pre_ms, pre_bytes = [], 0.0, 0.0
    piv = None
    if args.pivots == "massive":      # one pivot set per batch row, for every PSA layer (R22)
        rows = sorted({u // w.hkv for u in units})
        res = synth.residual_inputs(w, rows=rows, device=dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        piv, cnt = ak.akvq_detect_pivots(res, dt, 50.0, w.top_k)
        e1.record()
        torch.cuda.synchronize()
        pre_ms += e0.elapsed_time(e1)
        pre_bytes += res.numel() * res.element_size()
        del res
        # per local unit (its batch row's list), so any unit slicing works
        sel = torch.tensor([u // w.hkv - rows[0] for u in units], device=dev)
        piv, cnt = piv.index_select(0, sel).contiguous(), cnt.index_select(0, sel).contiguous()
    for layer in range(n_layers):
        kind = w.kind(layer)
        cfg = ak.make_config(Ul, w.g, w.d, w.G, w.R, cap, w.top_k, kind, dt, w.clip2, w.clip4,
                             1 if args.k_axis.startswith("token") else 0,
                             exact_r=1 if args.k_axis == "token-exact" else 0)
        lc = ak.LayerCache(cfg, device=dev)
        lc.handle.options = ((ak.AKVQ_OPT_STREAM_ONLY if args.stream_only else 0) |
                             (ak.AKVQ_OPT_SKIP_ROWS if args.skip_rows else 0) |
                             (ak.AKVQ_OPT_SKIP_PAGES if args.skip_pages else 0))
        inp = synth.layer_inputs(w, layer, units=units, device=dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if piv is not None and kind == 1:
            lc.prefill_pivots(inp["K"], inp["V"], piv, cnt, 1)
        else:
            lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
        e1.record()
        torch.cuda.synchronize()
        pre_ms += e0.elapsed_time(e1)
        pre_bytes += Ul * prefill_bytes_per_unit(w, kind, w.L0)
        del inp
        caches.append(lc)
    torch.cuda.empty_cache()

    # ---------------- decode-step inputs, resident in HBM before timing
    def step_inputs(step, device):
        qs, ks, vs = [], [], []
        for layer in range(n_layers):
            di = synth.decode_inputs(w, layer, step, units=units, device=device)
            qs.append(di["q"]); ks.append(di["k"]); vs.append(di["v"])
        return torch.stack(qs), torch.stack(ks), torch.stack(vs), di["types"]

    inputs = [step_inputs(s, dev) for s in range(args.warmup + args.steps)]
    # Outputs of a whole step ([layers, U_local, g, d]); with N > 1 they are
    # all-gathered once per step (row a8) on NCCL's stream, double-buffered so
    # the gather of step s overlaps the attention of step s + 1 (legitimate in
    # this attention-only benchmark: synthetic queries do not depend on the
    # gathered outputs).
    gathers = [shard.OutputGather(U, world, rank, w.g, w.d, lead=(n_layers,), device=dev)
               for _ in range(2 if world > 1 else 1)]
    pending = [None] * len(gathers)
    n_step = [0]
    launches = [0]

    def one_step(q, k, v, types):
        b = n_step[0] % len(gathers)
        if pending[b] is not None:
            pending[b].wait()                     # buffer b's previous gather is done
            pending[b] = None
        outs = gathers[b].local_view()
        for layer, lc in enumerate(caches):
            nq = lc.n_q
            # append + decode attention through the C ABI (one fused launch when
            # no block flush is due; append + quantize + decode when it is)
            lc.step(k[layer], v[layer], q[layer], types, out=outs[layer])
            launches[0] += lc.last_launches
        if world > 1:
            pending[b] = gathers[b].gather(async_op=True)
        n_step[0] += 1
        return b

    def drain():
        for i, wk in enumerate(pending):
            if wk is not None:
                wk.wait()
                pending[i] = None

    for s in range(args.warmup):
        one_step(*inputs[s])
    drain()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    # ---------------- timed region (device)
    # one event per step boundary (none between the PDL-chained layer launches)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    L_at = [caches[2 % n_layers].L]
    nq_at = [caches[2 % n_layers].n_q]
    sampler = ClockSampler(local)
    launches[0] = 0
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    with sampler:
        t0.record()
        evs[0].record()
        step_launches = []
        for s in range(args.steps):
            l0 = launches[0]
            one_step(*inputs[args.warmup + s])
            evs[s + 1].record()
            step_launches.append(launches[0] - l0)
            L_at.append(caches[2 % n_layers].L)
            nq_at.append(caches[2 % n_layers].n_q)
        drain()
        t1.record()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    n_launch = launches[0]
    ms = t0.elapsed_time(t1) / args.steps
    # mean k_decode_layer launch duration: steps whose launches are exactly the
    # n_layers decode launches (no block flush) -> step time / n_layers (includes
    # the inter-launch gaps, so it is a conservative per-launch time)
    plain = [s for s in range(args.steps) if step_launches[s] == n_layers]
    if world == 1 and plain:
        dec_ms = sum(evs[s].elapsed_time(evs[s + 1]) for s in plain) / (len(plain) * n_layers)
    else:
        dec_ms = ms / n_layers
    if dist:
        t = torch.tensor([ms, dec_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, dec_ms = float(t[0]), float(t[1])
    clocks = sampler.summary()

    # algorithmic bytes of one decode launch (per layer, this rank), averaged
    side_psa = w.top_k
    text_prefix = [0]
    for t in synth.token_types(w).tolist():
        text_prefix.append(text_prefix[-1] + (t == 1))
    bytes_layers = []
    for s in range(args.steps):
        L, nq = L_at[s + 1], nq_at[s + 1]
        for layer in range(n_layers):
            kind = w.kind(layer)
            if kind == 1:
                side = side_psa
            else:
                side = text_prefix[min(nq, w.L0)] + max(0, nq - w.L0)
            bytes_layers.append(Ul * decode_bytes_per_unit(w, kind, L, nq, side))
    dec_bytes = sum(bytes_layers) / len(bytes_layers)
    peaks = _peaks()
    traffic, traffic_commit = None, None   # dram bytes of one launch, committed ncu capture
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        with open(tf) as fh:
            tj = json.load(fh).get("k_decode_layer", {})
        # only for the exact configuration the capture was taken on
        if (tj.get("workload") == w.name and world == 1 and args.k_axis == "channel"
                and args.pivots == "colsum" and not (args.stream_only or args.skip_rows
                                                     or args.skip_pages)):
            traffic, traffic_commit = tj.get("traffic_bytes"), tj.get("commit")
    achieved = dec_bytes / (dec_ms * 1e-3) / 1e9
    tokens_per_s = w.batch / (ms * 1e-3)

    # ---------------- end to end through the C ABI with host buffers
    e2e_steps = args.steps
    host_in = []
    for s in range(e2e_steps):
        q, k, v, ty = step_inputs(args.warmup + args.steps + s, "cpu")
        host_in.append((q.pin_memory(), k.pin_memory(), v.pin_memory(), ty.pin_memory()))
    host_out = torch.empty((n_layers, U, w.g, w.d), dtype=torch.float32).pin_memory()
    dq = torch.empty_like(inputs[0][0]); dk = torch.empty_like(inputs[0][1])
    dv = torch.empty_like(inputs[0][2]); dty = torch.empty_like(inputs[0][3])
    h2d = sum(t.numel() * t.element_size() for t in host_in[0])
    d2h = host_out.numel() * host_out.element_size()
    # Step-level pipelining (world == 1): step s+1's inputs are copied host->device
    # on an H2D stream while step s computes (double-buffered), and step s's
    # outputs go device->host on a D2H stream while step s+1 computes.  Events
    # only at step boundaries, so the layer launches stay PDL-chained.
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    main_s = torch.cuda.current_stream()
    dbufs = [tuple(torch.empty_like(t) for t in inputs[0]) for _ in range(2)]
    obufs = [torch.empty((n_layers, Ul, w.g, w.d), dtype=torch.float32, device=dev) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    ev_read = [torch.cuda.Event() for _ in range(2)]

    def prefetch_inputs(s):
        b = s % 2
        h2d_s.wait_event(ev_used[b])                   # buffer b no longer read by step s-2
        with torch.cuda.stream(h2d_s):
            for dst, src in zip(dbufs[b], host_in[s]):
                dst.copy_(src, non_blocking=True)
            ev_in[b].record(h2d_s)

    def e2e_step_pipelined(s):
        b = s % 2
        dq, dk, dv, dty = dbufs[b]
        if s + 1 < e2e_steps:
            prefetch_inputs(s + 1)                     # the next step's inputs
        main_s.wait_event(ev_in[b])
        main_s.wait_event(ev_read[b])                  # obufs[b] copied out (step s-2)
        for l, lc in enumerate(caches):
            lc.step(dk[l], dv[l], dq[l], dty, out=obufs[b][l])
        ev_used[b].record(main_s)
        d2h_s.wait_event(ev_used[b])
        with torch.cuda.stream(d2h_s):
            host_out.copy_(obufs[b], non_blocking=True)
            ev_read[b].record(d2h_s)

    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if world == 1:
        prefetch_inputs(0)
    for s in range(e2e_steps):
        if world == 1:
            e2e_step_pipelined(s)
            continue
        q, k, v, ty = host_in[s]
        dq.copy_(q, non_blocking=True); dk.copy_(k, non_blocking=True)
        dv.copy_(v, non_blocking=True); dty.copy_(ty, non_blocking=True)
        b = one_step(dq, dk, dv, dty)
        if pending[b] is not None:                # the user reads the gathered result
            pending[b].wait()
            pending[b] = None
        res = gathers[b].result() if world > 1 else gathers[b].local_view()
        host_out.copy_(res, non_blocking=True)
    main_s.wait_stream(d2h_s)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
        dist.barrier()

    # ---------------- flush cost: a step that quantizes a G-block (every G steps)
    # is timed on its own (the timed region above may hold none) and amortized
    def sync_inputs(step):
        q, k, v, ty = step_inputs(step, dev)
        return q, k, v, ty

    flush = None
    st = args.warmup + 2 * args.steps
    # (exact residual window, R26: every step quantizes one token inside the timed
    # region, there is no block flush to time separately)
    while args.k_axis != "token-exact" and caches[0].L - w.R - caches[0].n_q < w.G - 1 \
            and caches[0].L < cap - 1:
        one_step(*sync_inputs(st)); st += 1             # plain steps up to the boundary
    drain()
    if args.k_axis != "token-exact" and caches[0].L - w.R - caches[0].n_q == w.G - 1 \
            and caches[0].L < cap:
        fin = sync_inputs(st)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        l0 = launches[0]
        one_step(*fin)
        drain()
        f1.record()
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1)
        if dist:
            t = torch.tensor([fms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            fms = float(t[0])
        amort = ((w.G - 1) * ms + fms) / w.G
        flush = {"ms_flush_step": fms, "ms_plain_step": ms, "flush_every_steps": w.G,
                 "launches_flush_step": launches[0] - l0,
                 "amortized_ms_per_step": amort, "amortized_tokens_per_s": w.batch / (amort * 1e-3)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(w)

    # ---------------- 1-GPU emulation of the per-rank shapes of strong scaling
    # (the BJ:9 global batch split over 2 / 4 / 8 GPUs = batch 32 / 16 / 8 per rank)
    emul = None
    if world == 1 and w1.name.startswith("sweep@b") and not args.no_strong_emulation \
            and args.k_axis != "token-exact":
        del caches
        inputs.clear()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        emul = {}
        for nshard in (2, 4, 8):
            if w1.batch % nshard:
                continue
            emul[f"n{nshard}"] = emulate_rank_shape(ak, synth, w1.with_batch(w1.batch // nshard),
                                                    n_layers, dt, args, dev)
            emul[f"n{nshard}"]["projected_speedup_vs_1"] = ms / emul[f"n{nshard}"]["ms_per_step"]

    if rank == 0:
        line = {
            "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "u8-imma+f32", "data": "synthetic",
            "config": dict(workload_config(args, w, w1, world, n_layers),
                           l2="no flush: per-step working set "
                              f"{sum(bytes_layers[:n_layers]) / 1e9:.2f} GB/rank >> 126 MB L2"),
            "attention_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                         "frac_nominal": achieved / 8000.0, "peak_nominal": 8000.0,
                         "traffic": traffic, "traffic_commit": traffic_commit,
                         "kernel": "k_decode_layer (append + all tiers + merge, one launch per layer)",
                         "bytes_per_launch": dec_bytes, "launch_ms": dec_ms,
                         "peak_src": peaks["src"]},
            "prefill": {"ms_all_layers": pre_ms, "quantize_gbs": pre_bytes / (pre_ms * 1e-3) / 1e9,
                        "frac": pre_bytes / (pre_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "e2e": {"value": w.batch / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "note": "pinned host inputs of step s+1 are copied while step s computes "
                            "(legitimate here: synthetic queries do not depend on outputs); "
                            "outputs of every step copied back"},
            "gpu_launches": n_launch,
            "clocks": clocks,
        }
        if flush:
            line["flush"] = flush
        if emul:
            line["strong_scaling_emulation"] = emul
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
