"""Energy per score step (NVML total-energy counter) -- the chip is power-capped under
sustained load, so J/step bounds sustained throughput.  Variants via env knobs, each in a
fresh process:  python tools/energy.py [--steps 60] [--var ENV=V1,V2 ...]"""
import argparse
import itertools
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(steps, what):
    import pynvml
    import torch

    from paper_2412_08521_b200 import ems
    from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch
    w = CONFIGS["cfg3"]
    dev = torch.device("cuda")
    q, kr, kw, v = make_batch_torch(w, seed=1, device=dev)
    B, Hq, L, d = q.shape
    plan = ems.Plan(B, Hq, w.heads_kv, L, d, q.dtype, ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma), dev,
                    "tcgen05", want_out=True)
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
    step = (lambda: plan.score(q, kr, v)) if what == "score" else (lambda: (plan.score(q, kr, v), plan.select(),
                                                                            plan.merge(kw, v), plan.compact(kw, v)))
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    time.sleep(0.5)
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    j = (e1 - e0) / 1e3
    return {"ms_per_step": 1e3 * (t1 - t0) / steps, "J_per_step": j / steps, "avg_W": j / (t1 - t0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--what", default="score")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--var", action="append", default=[])
    a = ap.parse_args()
    if a.child:
        print(json.dumps(child(a.steps, a.what)))
        return
    axes = [(kv.split("=")[0], kv.split("=")[1].split(",")) for kv in a.var] or [("NONE", [""])]
    for combo in itertools.product(*[[(k, v) for v in vs] for k, vs in axes]):
        env = dict(os.environ)
        env.update({k: v for k, v in combo if k != "NONE"})
        r = subprocess.run([sys.executable, __file__, "--child", "--steps", str(a.steps), "--what", a.what], env=env,
                           capture_output=True, text=True)
        print(" ".join(f"{k}={v}" for k, v in combo), r.stdout.strip() or r.stderr.strip()[-300:], flush=True)


if __name__ == "__main__":
    main()
