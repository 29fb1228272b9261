"""Per-rank compute time of the N-way unit sharding, measured on ONE GPU: for N = 1, 2, 4, 8 every
rank's shard (shard.unit_shard) runs the device path (score + select + merge + compact) alone,
back to back for ~0.4 s after ~0.2 s of warm-up (both sides in the power-capped regime), and the
slowest rank's mean step time gives the strong-scaling speed-up the sharding itself allows
(T_1 / max_r T_N,r).  Not a multi-GPU measurement: no interconnect, no other GPUs' power or
clocks -- the path has no data-path collective, so this isolates the per-rank work.

    python tools/shard_scaling.py [--config cfg3]"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--seconds", type=float, default=0.4)
    args = ap.parse_args()
    import torch

    from paper_2412_08521_b200 import ems
    from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch
    from paper_2412_08521_b200.shard import slice_inputs, unit_shard

    w = CONFIGS[args.config]
    dev = torch.device("cuda")
    full = make_batch_torch(w, seed=1, device=dev)
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)

    def time_shard(q, kr, kw, v):
        B, Hq, L, d = q.shape
        plan = ems.Plan(B, Hq, kr.shape[1], L, d, q.dtype, cfg, dev, "auto", want_out=True)

        def step():
            plan.score(q, kr, v)
            plan.select()
            plan.merge(kw, v)
            plan.compact(kw, v)

        t_end = time.time() + args.seconds / 2
        while time.time() < t_end:  # warm-up into the sustained regime
            step()
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        e0.record()
        t_end = time.time() + args.seconds
        while time.time() < t_end:
            step()
            n += 1
        e1.record()
        torch.cuda.synchronize()
        plan.sync_status()
        return e0.elapsed_time(e1) / n

    res = {}
    for N in (1, 2, 4, 8):
        per_rank = []
        for r in range(N):
            sh = unit_shard(w.batch, w.heads_kv, N, r)
            part = tuple(x.contiguous() for x in slice_inputs(*full, sh))
            per_rank.append(time_shard(*part))
            del part
            torch.cuda.empty_cache()
        res[N] = max(per_rank)
        print(json.dumps({"config": args.config, "N": N, "units_per_rank": sh.n_units,
                          "max_rank_ms": round(res[N], 4), "min_rank_ms": round(min(per_rank), 4),
                          "speedup_vs_1": round(res[1] / res[N], 3)}), flush=True)


if __name__ == "__main__":
    main()
