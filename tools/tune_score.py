"""Times the score pass (P1 + P2) on config 3 for tuning knobs passed via env vars.

    python tools/tune_score.py [--config cfg3] [--reps 5]

Each variant runs in a fresh subprocess (knobs are read once per process)."""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(cfg: str, reps: int) -> dict:
    import torch

    from paper_2412_08521_b200 import ems
    from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch

    w = CONFIGS[cfg]
    dev = torch.device("cuda")
    q, kr, kw, v = make_batch_torch(w, seed=1, device=dev)
    B, Hq, L, d = q.shape
    plan = ems.Plan(B, Hq, w.heads_kv, L, d, q.dtype, ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma),
                    dev, "tcgen05", want_out=True)
    for _ in range(2):
        plan.score(q, kr, v)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.score(q, kr, v)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    glo = plan.glo.double()
    # per-kernel device times (CUPTI via torch.profiler)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            plan.score(q, kr, v)
        torch.cuda.synchronize()
    kern = {}
    for e in prof.key_averages():
        if e.device_time_total > 0 and ("tc_kernel" in e.key or "simt" in e.key):
            name = "fwd_tc" if "fwd_tc" in e.key else ("colsum_tc" if "colsum" in e.key else e.key[:40])
            kern[name] = round(e.device_time_total / e.count / 1e3, 3)
    return {"ms": sorted(ts)[len(ts) // 2], "min_ms": min(ts), "kernels_ms": kern,
            "glo_mass_err": float((glo.sum(-1) - L).abs().max().item() / L)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--var", action="append", default=[], help="ENV=V1,V2,... (cartesian product)")
    args = ap.parse_args()
    if args.child:
        print(json.dumps(child(args.config, args.reps)))
        return
    import itertools
    axes = [(kv.split("=")[0], kv.split("=")[1].split(",")) for kv in args.var] or [("NONE", [""])]
    for combo in itertools.product(*[[(k, v) for v in vs] for k, vs in axes]):
        env = dict(os.environ)
        env.update({k: v for k, v in combo if k != "NONE"})
        r = subprocess.run([sys.executable, __file__, "--child", "--config", args.config, "--reps",
                            str(args.reps)], env=env, capture_output=True, text=True)
        tag = " ".join(f"{k}={v}" for k, v in combo)
        print(tag, r.stdout.strip() or r.stderr.strip()[-400:], flush=True)


if __name__ == "__main__":
    main()
