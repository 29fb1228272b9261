#!/usr/bin/env python
"""Throughput of the EMS prefill-compress path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

One step = the whole hot path over one synthetic batch of the workload:
score pass (O, LSE, GQA-mean glo/loc) -> select -> merge -> compact, for every
KV unit of the batch.  Default workload: BASELINE config 3 (B=1, H_q=32,
H_kv=8, d=128, L=32768, bf16, budget 256) -- the config the metric is quoted on.

* value: device-timed tokens/s of the WHOLE workload with inputs resident in HBM
  (CUDA events, barrier + synchronize on both sides, max over ranks); inputs
  (>= 268 MB of Q) exceed the 126 MB L2, so no explicit flush is needed.
* e2e: the same metric through the public API (ems_prefill_host): pinned HOST raw
  Q/K/V in, RoPE on the device, compressed cache AND attention output O back to
  pinned host memory, all inside the timed region.
* roofline: the score pass (the dominant kernel pair) against the measured
  bf16 tensor peak; algorithmic FLOPs F_alg = 4*d*G*L(L+1)/2 per unit.
* cpu_baseline: the reference's own code (oracle/_ref) on all units of one layer at a
  fixed sample length L' (the same L' in both arms), every (unit, head) score pass in
  one OpenMP region over all host cores as engine.cpp:65 does; extrapolated to L
  (score pass x L(L+1)/L'(L'+1), compress x L/L') and to every layer / batch element,
  with the extrapolation stated in the line.
Multi-GPU: `--gpus N` (or torchrun with N ranks) shards the workload's units across the
ranks (shard.unit_shard: one KV head per GPU for configs 3 and 5 at N = 8), no
collective on the data path -> strong scaling.  --impl reference times the reference
CPU path (rank 0 only).
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
    """ncu-measured DRAM bytes per score pass (profiles/r2_traffic.json; config 3 only)."""
    if not w.name.startswith("cfg3") or w.seq_len != 32768 or w.batch != 1 or w.n_budget != 256:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
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

    def begin(self):
        self.t0 = time.perf_counter()

    def end(self):
        self.t1 = time.perf_counter()

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
                "power_w_max": max(watts) if watts else None,
                "power_w_median": statistics.median(watts) if watts else None}


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


# Reference sample lengths L' per workload: the same L' in both arms (the ours arm's
# cpu_baseline and --impl reference), sized so one sample (every unit of one layer of batch
# element 0, with O, all host cores) is a few seconds of CPU work.
SAMPLE_LEN = {"cfg1": 1024, "cfg2": 4096, "cfg3": 4096, "cfg3b": 4096, "cfg4": 2048, "cfg5": 2048,
              "cfgM": 4096}


def _cpu_sample(w, sample_len: int | None = None):
    """The reference CPU path (oracle/_ref = the reference's own sources) on a bounded sample.

    Sample: every KV unit of one layer of batch element 0 (config 3: all 8 units = 32 query
    heads) at the first L' tokens of the workload's recipe, through ems_ref_prefill_units:
    prefill_attention for every (unit, query head) in ONE OpenMP region over all host
    threads (engine.cpp:65 spreads heads the same way), GQA mean (D2), init_score_state,
    policy_prefill_compress -> compress_prefill per unit (parallel over units).  The library
    times the two phases separately; the full step is extrapolated as
        t = t_score * L(L+1) / L'(L'+1) + t_compress * L / L'     (causal pairs / tokens)
    times batch elements x layers (identical work per unit).  L' = L means no length
    extrapolation.  Returns (tokens/s, description, cores, extrapolation dict)."""
    import numpy as np

    from oracle.oracle import Config, RefLib
    from paper_2412_08521_b200.inputs import make_unit_np

    ref = RefLib()
    cores = ref.max_threads()
    cfg = Config(n_budget=w.n_budget, l_win=w.l_win, tau=w.tau, gamma=w.gamma, kernel_size=w.kernel_size)
    Lp = min(w.seq_len, sample_len or SAMPLE_LEN.get(w.name, 1024))
    units = [make_unit_np(w, seed=1, seq_len=Lp, unit=u) for u in range(w.heads_kv)]
    stack = lambda f: np.stack([getattr(u, f) for u in units])  # noqa: E731
    ref.prefill_units(stack("q_rot"), stack("k_rot"), stack("k_raw"), stack("v"), cfg, with_out=True, dump=False)
    t_score, t_comp = ref.last_seconds
    L = w.seq_len
    s_score = L * (L + 1) / (Lp * (Lp + 1))
    s_comp = L / Lp
    reps = w.batch * w.layers
    t_full = (t_score * s_score + t_comp * s_comp) * reps
    tok = w.batch * L / t_full
    ex = {"sample_len": Lp, "seq_len": L, "score_s": round(t_score, 3), "compress_s": round(t_comp, 3),
          "score_scale": round(s_score, 2), "compress_scale": round(s_comp, 2), "unit_scale": reps,
          "extrapolated": Lp != L or reps != 1}
    desc = (f"reference prefill_attention for all {w.heads_kv} units x {w.group} heads of one layer in one OpenMP "
            f"region + GQA mean + compress_prefill, at L'={Lp} ({t_score:.2f}s + {t_comp:.2f}s, {cores} threads)"
            + (f"; extrapolated: score x{s_score:.1f}, compress x{s_comp:.1f}, x{reps} (batch x layers)"
               if ex["extrapolated"] else "; no extrapolation"))
    return tok, desc, cores, ex


def run_reference(args, w):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    os.environ.setdefault("OMP_WAIT_POLICY", "passive")
    times = []
    desc, cores, ex = "", 0, {}
    for i in range(args.warmup + args.steps):
        # warm-up samples are short (thread pools, page faults); timed steps use the fixed L'
        lp = args.sample_len or SAMPLE_LEN.get(w.name, 1024)
        tok, desc, cores, ex = _cpu_sample(w, max(128, lp // 4) if i < args.warmup else lp)
        if i >= args.warmup:
            times.append(tok)
    import statistics
    v = statistics.median(times)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * w.batch * w.seq_len / v,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": config_dict(w, 1),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "reference",
                             "sample": desc, "extrapolation": ex},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "prefill+compress tokens/s per GPU at 32k ctx; % of attention roofline"


def config_dict(w, n):
    return {"workload": f"BASELINE config 3 ({w.name}): B={w.batch} H_q={w.heads_q} H_kv={w.heads_kv} "
                        f"d={w.head_dim} L={w.seq_len} {w.dtype} budget={w.n_budget} w={w.l_win} "
                        f"gamma={w.gamma} tau={w.tau} kernel={w.kernel_size}"
            if w.name.startswith("cfg3") else f"{w.name}",
            "global_batch": w.batch, "seq_len": w.seq_len, "layers": w.layers,
            "units": w.batch * w.heads_kv * w.layers,
            "parallelism": f"kv-unit sharding over {n} GPU(s) (shard.unit_shard; strong scaling, no collective)",
            "l2": _l2_note(w)}


def _l2_note(w) -> str:
    e = 2 if w.dtype == "bf16" else 4
    qb = w.batch * w.heads_q * w.seq_len * w.head_dim * e
    total = qb + 3 * w.batch * w.heads_kv * w.seq_len * w.head_dim * e  # Q, K_rot, K_raw, V
    if total > 126e6:
        return f"inputs > L2 (Q alone {qb / 1e6:.0f} MB per layer), no flush"
    return f"inputs fit in L2 ({total / 1e6:.0f} MB); not flushed (informational config, not the headline)"


def _relaunch(args) -> int:
    """`python bench.py --gpus N` outside torchrun: start N ranks the way the driver does
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1)."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


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
    ap.add_argument("--sample-len", type=int, default=0, help="reference sample length L' (default: SAMPLE_LEN)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="unit groups of the host copy/compute pipeline")
    ap.add_argument("--oversubscribe", action="store_true",
                    help="testing only: every rank on cuda:0 with gloo plumbing (ranks never wait on each "
                         "other's kernels); numbers from such a run are not scaling results")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args))

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
    from paper_2412_08521_b200.shard import slice_inputs, unit_shard

    ws, rank, local = dist_env()
    if ws > 1 and not args.oversubscribe and torch.cuda.device_count() < ws:
        raise SystemExit(f"bench.py: {ws} ranks but {torch.cuda.device_count()} visible GPU(s)")
    local = 0 if args.oversubscribe else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if args.oversubscribe:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    # this rank's units of every layer (strong scaling: the workload is fixed, the units are split)
    shard = unit_shard(w.batch, w.heads_kv, ws, rank)
    # a step runs every layer of the workload (config 4: 32); layers alternate between two
    # distinct input sets (each layer's inputs are far larger than L2, so nothing is reused)
    n_layers = w.layers
    sets = []
    for li in range(min(n_layers, 2)):
        full = make_batch_torch(w, seed=1, device=dev, layer=li)
        sets.append(tuple(x.contiguous() for x in slice_inputs(*full, shard)))
        del full
    torch.cuda.empty_cache()
    q, kr, kw, v = sets[0]
    B, Hq, L, d = q.shape
    plan = ems.Plan(B, Hq, kr.shape[1], L, d, q.dtype, cfg, dev, args.score_impl, want_out=True)
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
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if not args.oversubscribe else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

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
    ms_step = max_over_ranks(total_ms) / args.steps
    tokens_step = w.batch * L  # the whole workload's tokens (every rank holds a slice of its units)
    value = tokens_step / (ms_step / 1e3)

    # e2e through the public API the reference's callers use: engine::prefill on RAW host
    # matrices (ems_prefill_host): pinned host Q/K/V in, RoPE on the device, compressed cache and
    # the attention output O (PrefillResult.per_head) back to pinned host memory; copies
    # pipelined with compute in --e2e-chunks unit groups.
    e2e = None
    if not args.no_e2e:
        base = w.rope_base or 0.0
        hsets = []
        for ql, _, kwl, vl in sets:
            q_raw = unrope(ql, base) if base else ql
            hsets.append(tuple(x.cpu().pin_memory() for x in (q_raw, kwl, vl)))
            del q_raw
        host_cache = plan.host_cache()
        h_out = torch.empty(plan.out.shape, dtype=plan.out.dtype, pin_memory=True)
        h2d = n_layers * sum(x.numel() * x.element_size() for x in hsets[0])
        d2h = n_layers * (sum(x.numel() * x.element_size() for x in host_cache.values())
                          + h_out.numel() * h_out.element_size())

        def e2e_step():  # every layer: its host inputs in, its compressed cache and O out
            for li in range(n_layers):
                hq, hk, hv = hsets[li % len(hsets)]
                plan.run_host(hq, hk, hv, base, h_k_raw=None if base else hk, chunks=args.e2e_chunks, h_out=h_out)

        for _ in range(2):
            e2e_step()
        plan.sync_status()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n_e2e = max(2, min(args.steps, 5))
        for _ in range(n_e2e):
            e2e_step()
        e1.record(stream)
        barrier()
        te = max_over_ranks(e0.elapsed_time(e1) / n_e2e)
        sums = torch.tensor([h2d, d2h], dtype=torch.float64, device="cpu" if args.oversubscribe else dev)
        if ws > 1:  # whole-job bytes: every rank copies its own units
            dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        e2e = {"value": tokens_step / (te / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(sums[0].item()), "d2h_bytes_per_step": int(sums[1].item()),
               "ms_per_step": te,
               "api": f"ems.Plan.run_host (ems_prefill_host, raw Q/K + device RoPE, cache + O back, "
                      f"{args.e2e_chunks} chunks)"}

    pk = peaks()
    shard_w = w.with_(batch=1, heads_kv=plan.dims.units, heads_q=plan.dims.units * w.group)
    flops = f_alg(shard_w) * n_layers  # this rank's score passes
    achieved = flops / (score_ms / 1e3) / 1e12
    peak_tf = pk.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
    roof_ms = max(f_alg(w) * n_layers / ws / (peak_tf * 1e12),
                  n_layers * score_bytes(w) / ws / (pk.get("hbm_gbs", 6650.0) * 1e9)) * 1e3
    # the optional gather of every rank's fixed-size compressed caches, off the
    # timed path and reported on its own: one all_gather per cache tensor
    gather_ms = None
    if ws > 1:
        try:
            from paper_2412_08521_b200.shard import gather_caches
            total_units = w.batch * w.heads_kv
            gather_caches(plan.cache, shard, total_units)  # warm-up (communicators)
            barrier()
            g0 = time.perf_counter()
            gather_caches(plan.cache, shard, total_units)
            barrier()
            gather_ms = max_over_ranks((time.perf_counter() - g0) * 1e3)
        except Exception as ex:  # noqa: BLE001 -- informational; never fails the bench line
            gather_ms = f"unavailable: {str(ex)[:120]}"
    # our kernel launches per step, counted by the CUDA profiler on one extra (untimed) step:
    # every kernel of libems_b200.so lives in namespace ems
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    kernels_per_step = sum(e.count for e in prof.key_averages() if e.device_time_total > 0 and "ems::" in e.key)
    launches = int(max_over_ranks(kernels_per_step)) * ws
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16" if w.dtype == "bf16" else "f32", "data": "synthetic",
            "config": config_dict(w, ws),
            "per_gpu_value": value / ws,
            "units_per_gpu": plan.dims.units,
            "attention_roofline_frac": roof_ms / ms_step,
            "stage_ms": {"score": score_ms, "select+merge+compact": tail_ms},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic_bytes(w) if ws == 1 else None,
                         "frac_of_sustained_peak": achieved / pk.get("bf16_tflops_sustained", peak_tf),
                         "frac_of_spec_peak": achieved / 2250.0,  # nominal dense bf16
                         "kernel": "score pass (O+LSE and glo/loc column sums)",
                         "peak_source": f"{pk['source']} bf16_tflops (burst)",
                         "algorithmic_flops_per_launch": f_alg(shard_w)},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "step_ms": [round(starts[i].elapsed_time(ends[i]), 3) for i in range(args.steps)],
            "e2e": e2e,
        }
        if args.oversubscribe and ws > 1:
            line["oversubscribed"] = "all ranks on one GPU (plumbing test, not a scaling number)"
        if gather_ms is not None:
            line["cache_allgather_ms"] = gather_ms  # outside the timed region
        if not args.no_cpu_baseline and ws == 1:
            try:
                tok, desc, cores, ex = _cpu_sample(w, args.sample_len or None)
                line["cpu_baseline"] = {"value": tok, "unit": "tokens/s", "cores": cores,
                                        "kind": "reference", "sample": desc, "extrapolation": ex}
            except Exception as ex:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
        print(json.dumps(line), flush=True)
    clk.stop()
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
