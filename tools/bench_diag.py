"""Diagnostics timing at config 3 (8 units, L = 32768, bf16, d = 128): sparsity and the
tensor-core redundancy rate (CUDA events, warm-up first)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_08521_b200 import ems  # noqa: E402

U, L, d = 8, int(os.environ.get("L", 32768)), 128
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn(1, U, L, d, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(1, U, L, d, device="cuda", generator=g).to(torch.bfloat16)
glo = torch.rand(1, U, L, device="cuda", generator=g)
loc = torch.rand(1, U, L, device="cuda", generator=g)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {"L": L, "units": U,
       "sparsity_ms": timed(lambda: ems.sparsity_rate(glo, loc, 0.95)),
       "redundancy_tc_ms": timed(lambda: ems.redundancy_rate(k, v, 0.6))}
flops = 2 * 2 * d * L * (L - 1) / 2 * U  # two similarity GEMMs over the causal triangle
res["redundancy_tc_tflops"] = flops / res["redundancy_tc_ms"] / 1e9
os.environ["EMS_DIAG_SIMT"] = "1"
res["redundancy_simt_ms"] = timed(lambda: ems.redundancy_rate(k, v, 0.6), reps=1)
print(json.dumps(res))
