#!/usr/bin/env python
"""Throughput of the EMS prefill-compress path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

One step = the whole hot path over one synthetic batch of the workload:
score pass (O, LSE, GQA-mean glo/loc) -> select -> merge -> compact, for every
KV unit of the batch.  Default workload: BASELINE config 3 (B=1, H_q=32,
H_kv=8, d=128, L=32768, bf16, budget 256) -- the config the metric is quoted on.

* value: device-timed tokens/s with inputs resident in HBM (CUDA events,
  barrier + synchronize on both sides, max over ranks); inputs (>= 268 MB of Q)
  exceed the 126 MB L2, so no explicit flush is needed.
* e2e: the same metric through the public API (ems.Plan.run) from pinned HOST
  buffers: H2D of Q_rot/K_rot/K_raw/V and D2H of the compressed cache inside
  the timed region.
* roofline: the score pass (the dominant kernel pair) against the measured
  bf16 tensor peak; algorithmic FLOPs F_alg = 4*d*G*L(L+1)/2 per unit.
* cpu_baseline: the reference's own code (oracle/_ref) on a bounded sample,
  extrapolated (see _cpu_sample).
Multi-GPU (torchrun): weak scaling, each rank runs its own batch of units, no
collective on the data path.  --impl reference times the reference CPU path
(rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            p = json.load(f)
        p["source"] = "measured"
        return p
    except OSError:
        return dict(FALLBACK_PEAKS)


def traffic_bytes(w):
    """ncu-measured DRAM bytes per score pass (profiles/r1_traffic.json; config 3 only)."""
    if not w.name.startswith("cfg3") or w.seq_len != 32768 or w.batch != 1 or w.n_budget != 256:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            return json.load(f)["score_pass_bytes"]
    except (OSError, KeyError, ValueError):
        return None


def f_alg(w) -> float:
    """Algorithmic FLOPs of the score pass per step: QK^T + PV over the causal triangle."""
    L = w.seq_len
    return 4.0 * w.head_dim * w.heads_q * w.batch * L * (L + 1) / 2.0


def score_bytes(w) -> float:
    e = 4 if w.dtype == "f32" else 2
    L, d = w.seq_len, w.head_dim
    units = w.batch * w.heads_kv
    return (e * (w.batch * w.heads_q * L * d * 2 + units * 2 * L * d)
            + 4 * w.batch * w.heads_q * L + 8 * units * L)


class ClockSampler:
    """SM clock, throttle reasons and power sampled every 5 ms through NVML (the recipe's
    nvidia-smi clocks line without its 100 ms granularity).  The thread starts before the
    warm-up so NVML is initialised and sampling when the timed region begins; summary()
    keeps only the samples taken inside the window marked by begin()/end()."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.max_mhz = [], None  # (t, mhz, reasons_bits, watts)
        self.t0 = self.t1 = None
        self._thread = None

    def _run(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        self._ready.set()
        while not self._stop.is_set():
            t = time.perf_counter()
            mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            try:
                w = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
            except pynvml.NVMLError:
                w = None
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((t, mhz, r, w))
            time.sleep(self.period)

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
            if idx and idx[0].strip().isdigit():
                self.index = int(idx[self.index].strip()) if self.index < len(idx) else self.index
        except Exception:  # noqa: BLE001
            return self
        self._stop, self._ready = threading.Event(), threading.Event()
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        self._ready.wait(timeout=5.0)
        return self

    def _energy_mj(self):
        try:
            import pynvml
            return pynvml.nvmlDeviceGetTotalEnergyConsumption(pynvml.nvmlDeviceGetHandleByIndex(self.index))
        except Exception:  # noqa: BLE001
            return None

    def begin(self):
        self.e0 = self._energy_mj()
        self.t0 = time.perf_counter()

    def end(self):
        self.t1 = time.perf_counter()
        self.e1 = self._energy_mj()

    def energy_j(self):
        """Board energy over the timed window (NVML counter, J), or None."""
        e0, e1 = getattr(self, "e0", None), getattr(self, "e1", None)
        return None if e0 is None or e1 is None else (e1 - e0) / 1e3

    def stop(self):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self):
        import statistics
        win = [s for s in self.samples if self.t0 is not None and self.t0 <= s[0] <= (self.t1 or s[0])]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = sorted(n for n, bit in self.REASONS.items() if any(s[2] & bit for s in win))
        watts = [s[3] for s in win if s[3] is not None]
        return {"sm_mhz": statistics.median(s[1] for s in win), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(win), "sm_mhz_min": min(s[1] for s in win),
                "power_w_max": max(watts) if watts else None}


def unrope(x, base: float):
    """Inverse interleaved-pair RoPE (detail::rotate at -position, proj/src/rope.cpp:10-28), so
    the e2e arm can feed raw Q the way engine::prefill receives it."""
    import torch
    L, d = x.shape[-2], x.shape[-1]
    pos = -torch.arange(L, device=x.device, dtype=torch.float64)[:, None]
    freq = torch.pow(torch.tensor(base, dtype=torch.float64, device=x.device),
                     -torch.arange(0, d, 2, device=x.device, dtype=torch.float64) / d)[None, :]
    c, s = torch.cos(pos * freq), torch.sin(pos * freq)
    out = torch.empty_like(x)
    for p in range(x.shape[1]):  # plane by plane (fp64 temporaries stay small)
        a0, a1 = x[:, p, :, 0::2].double(), x[:, p, :, 1::2].double()
        out[:, p, :, 0::2] = (a0 * c - a1 * s).to(x.dtype)
        out[:, p, :, 1::2] = (a0 * s + a1 * c).to(x.dtype)
    return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cpu_sample(w, seconds_budget: float = 20.0, fixed_lp: int | None = None):
    """Reference CPU path (oracle/_ref = the reference's own sources) on a bounded sample.

    Sample: unit 0's G query heads through prefill_attention (parallel over heads as
    engine.cpp:65 does) + GQA mean + compress_prefill, on the first L' tokens of the
    workload's recipe, L' chosen so the sample runs ~10-30 s.  Extrapolation to the
    full step: score cost scales as (L/L')^2 (causal L^2 d), compress as L/L'; both
    scale linearly in the number of units.  Returns (tokens/s, description, cores)."""
    import numpy as np

    from oracle.oracle import Config, RefLib
    from paper_2412_08521_b200.inputs import make_unit_np

    ref = RefLib()
    cores = ref.max_threads()
    cfg = Config(n_budget=w.n_budget, l_win=w.l_win, tau=w.tau, gamma=w.gamma, kernel_size=w.kernel_size)
    Lp = fixed_lp or min(w.seq_len, 1024)
    un = make_unit_np(w, seed=1, seq_len=Lp, unit=0)
    t0 = time.perf_counter()
    ref.prefill_unit(un.q_rot, un.k_rot, un.k_raw, un.v, cfg, dump=False)
    t_small = time.perf_counter() - t0
    # grow L' while the projected sample stays inside the budget
    while fixed_lp is None and Lp * 2 <= w.seq_len and t_small * 4 <= seconds_budget:
        Lp *= 2
        un = make_unit_np(w, seed=1, seq_len=Lp, unit=0)
        t0 = time.perf_counter()
        ref.prefill_unit(un.q_rot, un.k_rot, un.k_raw, un.v, cfg, dump=False)
        t_small = time.perf_counter() - t0
    scale = (w.seq_len / Lp) ** 2
    t_full = t_small * scale * w.units
    tok = w.batch * w.seq_len / t_full
    desc = (f"reference prefill_attention x{w.group} heads + GQA mean + compress_prefill on 1 unit at "
            f"L'={Lp} ({t_small:.2f}s, {cores} threads); extrapolated x(L/L')^2={scale:.0f} and x{w.units} units")
    return tok, desc, cores, Lp


def run_reference(args, w):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    os.environ.setdefault("OMP_WAIT_POLICY", "passive")
    times = []
    desc, cores, lp = "", 0, None
    for i in range(args.warmup + args.steps):
        # the first call sizes the sample (~cpu_seconds of work); later steps reuse L'
        tok, desc, cores, lp = _cpu_sample(w, seconds_budget=args.cpu_seconds, fixed_lp=lp)
        if i >= args.warmup:
            times.append(tok)
    import statistics
    v = statistics.median(times)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * w.batch * w.seq_len / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": config_dict(w, ws),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "reference",
                             "sample": desc},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "prefill+compress tokens/s per GPU at 32k ctx; % of attention roofline"


def config_dict(w, n):
    return {"workload": f"BASELINE config 3 ({w.name}): B={w.batch} H_q={w.heads_q} H_kv={w.heads_kv} "
                        f"d={w.head_dim} L={w.seq_len} {w.dtype} budget={w.n_budget} w={w.l_win} "
                        f"gamma={w.gamma} tau={w.tau} kernel={w.kernel_size}"
            if w.name.startswith("cfg3") else f"{w.name}",
            "global_batch": w.batch * n, "seq_len": w.seq_len, "layers": w.layers, "units_per_gpu": w.units,
            "parallelism": f"kv-unit sharding x{n} (weak, no collective)",
            "l2": _l2_note(w)}


def _l2_note(w) -> str:
    e = 2 if w.dtype == "bf16" else 4
    qb = w.batch * w.heads_q * w.seq_len * w.head_dim * e
    total = qb + 3 * w.batch * w.heads_kv * w.seq_len * w.head_dim * e  # Q, K_rot, K_raw, V
    if total > 126e6:
        return f"inputs > L2 (Q alone {qb / 1e6:.0f} MB per layer), no flush"
    return f"inputs fit in L2 ({total / 1e6:.0f} MB); not flushed (informational config, not the headline)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--seq-len", type=int, default=0, help="override L (debug / scaling sweeps)")
    ap.add_argument("--batch", type=int, default=0, help="override B (config 4 uses 1/8/32)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--score-impl", default="auto", choices=["auto", "simt", "tcgen05"])
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="CPU work budget per reference sample (ours arm uses 2.5x for cpu_baseline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="unit groups of the host copy/compute pipeline")
    args = ap.parse_args()

    from paper_2412_08521_b200.inputs import CONFIGS

    w = CONFIGS[args.config]
    if args.seq_len:
        w = w.with_(seq_len=args.seq_len)
    if args.batch:
        w = w.with_(batch=args.batch)
    if args.impl == "reference":
        run_reference(args, w)
        return

    import torch
    import torch.distributed as dist

    from paper_2412_08521_b200 import ems
    from paper_2412_08521_b200.inputs import make_batch_torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    # a step runs every layer of the workload (config 4: 32); layers alternate between two
    # distinct input sets (each layer's inputs are far larger than L2, so nothing is reused)
    n_layers = w.layers
    sets = [make_batch_torch(w, seed=1 + rank, device=dev, layer=l) for l in range(min(n_layers, 2))]
    q, kr, kw, v = sets[0]
    B, Hq, L, d = q.shape
    plan = ems.Plan(B, Hq, w.heads_kv, L, d, q.dtype, cfg, dev, args.score_impl, want_out=True)
    stream = torch.cuda.current_stream()

    def step(score_events=None):
        """One step through the staged C-ABI entry points (same kernels as ems_prefill_compress),
        all layers; score_events[l] = (start, end) bracket layer l's score pass for the roofline."""
        for li in range(n_layers):
            ql, krl, kwl, vl = sets[li % len(sets)]
            if score_events is not None:
                score_events[li][0].record(stream)
            plan.score(ql, krl, vl)
            if score_events is not None:
                score_events[li][1].record(stream)
            plan.select()
            plan.merge(kwl, vl)
            plan.compact(kwl, vl)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clk = ClockSampler(local).start()
    for _ in range(args.warmup):
        step()
    plan.sync_status()
    barrier()
    # timed region: per-step events bracket the score pass and the whole step
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_layers)]
           for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    barrier()
    clk.begin()
    t_start.record(stream)
    for i in range(args.steps):
        starts[i].record(stream)
        step(sev[i])
        ends[i].record(stream)
    t_end.record(stream)
    barrier()
    clk.end()
    plan.sync_status()
    total_ms = t_start.elapsed_time(t_end)
    score_ms = sum(a.elapsed_time(b) for i in range(args.steps) for a, b in sev[i]) / args.steps
    tail_ms = sum(starts[i].elapsed_time(ends[i]) for i in range(args.steps)) / args.steps - score_ms
    t = torch.tensor([total_ms], device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = t.item() / args.steps
    tokens_step = B * L * ws
    value = tokens_step / (ms_step / 1e3)

    # e2e through the public API the reference's callers use: engine::prefill on RAW host
    # matrices (ems_prefill_host): pinned host Q/K/V in, RoPE on the device, compressed cache
    # back to pinned host memory; copies pipelined with compute in --e2e-chunks unit groups.
    e2e = None
    if not args.no_e2e:
        base = w.rope_base or 0.0
        hsets = []
        for ql, _, kwl, vl in sets:
            q_raw = unrope(ql, base) if base else ql
            hsets.append(tuple(x.cpu().pin_memory() for x in (q_raw, kwl, vl)))
            del q_raw
        host_cache = plan.host_cache()
        h2d = n_layers * sum(x.numel() * x.element_size() for x in hsets[0])
        d2h = n_layers * sum(x.numel() * x.element_size() for x in host_cache.values())

        def e2e_step():  # every layer: its host inputs in, its compressed cache out
            for li in range(n_layers):
                hq, hk, hv = hsets[li % len(hsets)]
                plan.run_host(hq, hk, hv, base, h_k_raw=None if base else hk, chunks=args.e2e_chunks)

        for _ in range(2):
            e2e_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_e2e = max(2, min(args.steps, 5))
        for _ in range(n_e2e):
            e2e_step()
        e1.record(stream)
        barrier()
        te = torch.tensor([e0.elapsed_time(e1) / n_e2e], device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": tokens_step / (te.item() / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": te.item(),
               "api": f"ems.Plan.run_host (ems_prefill_host, raw Q/K + device RoPE, {args.e2e_chunks} chunks)"}

    pk = peaks()
    flops = f_alg(w) * n_layers  # every layer's score pass
    achieved = flops / (score_ms / 1e3) / 1e12
    peak_tf = pk.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
    roof_ms = max(flops / (peak_tf * 1e12), n_layers * score_bytes(w) / (pk.get("hbm_gbs", 6650.0) * 1e9)) * 1e3
    # the optional gather of every rank's fixed-size compressed caches, off the
    # timed path and reported on its own: one NCCL all_gather per cache tensor
    gather_ms = None
    if ws > 1:
        try:
            from paper_2412_08521_b200.shard import gather_caches, unit_shard
            shard = unit_shard(1, ws * plan.dims.units, ws, rank)
            gather_caches(plan.cache, shard, ws * plan.dims.units)  # warm-up (NCCL communicators)
            barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            gather_caches(plan.cache, shard, ws * plan.dims.units)
            g1.record(stream)
            barrier()
            tg = torch.tensor([g0.elapsed_time(g1)], device=dev)
            dist.all_reduce(tg, op=dist.ReduceOp.MAX)
            gather_ms = tg.item()
        except Exception as ex:  # noqa: BLE001 -- informational; never fails the bench line
            gather_ms = f"unavailable: {str(ex)[:120]}"
    # our kernel launches per step, counted by the CUDA profiler on one extra (untimed) step:
    # every kernel of libems_b200.so lives in namespace ems
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    kernels_per_step = sum(e.count for e in prof.key_averages() if e.device_time_total > 0 and "ems::" in e.key)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16" if w.dtype == "bf16" else "f32", "data": "synthetic",
            "config": config_dict(w, ws),
            "per_gpu_value": value / ws,
            "attention_roofline_frac": roof_ms / ms_step,
            "stage_ms": {"score": score_ms, "select+merge+compact": tail_ms},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic_bytes(w),
                         "frac_of_sustained_peak": achieved / pk.get("bf16_tflops_sustained", peak_tf),
                         "kernel": "score pass (O+LSE and glo/loc column sums)",
                         "peak_source": f"{pk['source']} bf16_tflops (burst)",
                         "algorithmic_flops_per_launch": f_alg(w)},
            "gpu_launches": kernels_per_step * args.steps,
            "clocks": clk.summary(),
            "step_ms": [round(starts[i].elapsed_time(ends[i]), 3) for i in range(args.steps)],
            "energy_j_per_step": (clk.energy_j() / args.steps) if clk.energy_j() is not None else None,
            "e2e": e2e,
        }
        if gather_ms is not None:
            line["cache_allgather_ms"] = gather_ms  # outside the timed region
        if not args.no_cpu_baseline and ws == 1:
            try:
                tok, desc, cores, _ = _cpu_sample(w, 2.5 * args.cpu_seconds)
                line["cpu_baseline"] = {"value": tok, "unit": "tokens/s", "cores": cores,
                                        "kind": "reference", "sample": desc}
            except Exception as ex:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
        print(json.dumps(line), flush=True)
    clk.stop()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
