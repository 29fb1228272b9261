"""Timeline of one ems_prefill_host call (bench workload): copies and kernels per stream from
CUPTI (torch.profiler), to see the pipeline's fill and drain.

    python tools/e2e_timeline.py [--config cfg3] [--chunks 8]"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--chunks", type=int, default=8)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2412_08521_b200 import ems
    from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch

    w = CONFIGS[args.config]
    dev = torch.device("cuda")
    q, kr, kw, v = make_batch_torch(w, seed=1, device=dev)
    B, Hq, L, d = q.shape
    plan = ems.Plan(B, Hq, w.heads_kv, L, d, q.dtype, ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma),
                    dev, "tcgen05", want_out=True)
    base = w.rope_base or 0.0
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, kw, v))  # raw-vs-rotated content is irrelevant here
    h_out = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
    for _ in range(3):
        plan.run_host(hq, hk, hv, base, h_k_raw=None if base else hk, chunks=args.chunks, h_out=h_out)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        plan.run_host(hq, hk, hv, base, h_k_raw=None if base else hk, chunks=args.chunks, h_out=h_out)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    t0 = min(e.time_range.start for e in ev)
    rows = []
    for e in ev:
        s, t = (e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3
        name = e.name
        kind = "H2D" if "HtoD" in name else "D2H" if "DtoH" in name else "copy" if "Memcpy" in name else "kern"
        rows.append((s, t, kind, name[:60].replace("ems::(anonymous namespace)::", "")))
    rows.sort()
    end = max(r[1] for r in rows)
    first_kern = min(r[0] for r in rows if r[2] == "kern")
    h2d = [r for r in rows if r[2] == "H2D"]
    d2h = [r for r in rows if r[2] == "D2H"]
    print(f"call span {end:.3f} ms; first kernel at {first_kern:.3f} ms")
    print(f"H2D: {len(h2d)} copies, busy {sum(r[1]-r[0] for r in h2d):.3f} ms, last ends {max(r[1] for r in h2d):.3f} ms")
    print(f"D2H: {len(d2h)} copies, busy {sum(r[1]-r[0] for r in d2h):.3f} ms, first {min(r[0] for r in d2h):.3f}, "
          f"last ends {max(r[1] for r in d2h):.3f} ms")
    kb = sum(r[1] - r[0] for r in rows if r[2] == "kern")
    print(f"kernels busy (sum) {kb:.3f} ms")
    for r in rows:
        if r[2] == "kern" or r[1] - r[0] > 0.1 or r[0] > end - 1.0:
            print(f"{r[0]:8.3f} {r[1]:8.3f} {r[2]:4s} {r[3]}")


if __name__ == "__main__":
    main()
