"""Decode-step throughput of the device EMS decode loop (ems_decode_step), not the headline
metric: per-step latency for a prefilled batch (prefill itself untimed).

    python tools/bench_decode.py [--config cfg3] [--batch B] [--steps 200]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--seq-len", type=int, default=0)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    w = CONFIGS[a.config]
    if a.batch:
        w = w.with_(batch=a.batch)
    if a.seq_len:
        w = w.with_(seq_len=a.seq_len)
    dev = torch.device("cuda")
    q, kr, kw, v = make_batch_torch(w, seed=1, device=dev)
    B, Hq, L, d = q.shape
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    plan = ems.prefill_compress(q, kr, kw, v, cfg)
    base = w.rope_base or 1e4
    ds = ems.DecodeState(B, Hq, w.heads_kv, L, d, q.dtype, cfg, base, L + a.steps + 8)
    ds.init_from_plan(plan)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    xs = [(torch.randn((B, Hq, d), generator=g, device=dev).to(q.dtype),
           torch.randn((B, w.heads_kv, d), generator=g, device=dev).to(q.dtype),
           torch.randn((B, w.heads_kv, d), generator=g, device=dev).to(q.dtype)) for _ in range(a.steps + 5)]
    for x in xs[:5]:
        ds.step(*x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for x in xs[5:]:
        ds.step(*x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(json.dumps({"workload": f"{w.name} B={B} H_q={Hq} H_kv={w.heads_kv} d={d} prompt={L} budget={w.n_budget}",
                      "decode_ms_per_step": ms, "tokens_per_s": B / (ms / 1e3),
                      "units": B * w.heads_kv, "lut_capacity": ds.dims.lut}))


if __name__ == "__main__":
    main()
