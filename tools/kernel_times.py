"""Per-kernel device times of one full prefill step (score + select + merge + compact) on a
BASELINE config, via the CUDA profiler (CUPTI):  python tools/kernel_times.py [--config cfg2]"""
import argparse
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
w = CONFIGS[a.config]
q, kr, kw, v = make_batch_torch(w, seed=1, device="cuda")
B, Hq, L, d = q.shape
plan = ems.Plan(B, Hq, w.heads_kv, L, d, q.dtype, ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size),
                "cuda", "auto", want_out=True)
for _ in range(3):
    plan.run(q, kr, kw, v)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    for _ in range(a.reps):
        plan.run(q, kr, kw, v)
    torch.cuda.synchronize()
tot = 0.0
rows = []
for e in prof.key_averages():
    if e.device_time_total > 0 and "Memset" not in e.key and "cuda" not in e.key[:4]:
        t = e.device_time_total / a.reps / 1e3
        tot += t
        rows.append((t, e.count // a.reps, e.key[:80]))
for t, n, k in sorted(rows, reverse=True):
    print(f"{t:8.4f} ms  x{n}  {k}")
print(f"{tot:8.4f} ms  total kernel time per step ({a.config})")
