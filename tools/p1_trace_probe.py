"""Per-pair phase times of P1 from an instrumented variant (tools/make_trace_variants.py):
start -> first S ready -> last PV done -> epilogue done -> exit, and the idle gap between
consecutive pairs on one SM.  EMS_LIB_PATH=_variants/p1trace.so python tools/p1_trace_probe.py"""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2412_08521_b200 import ems  # noqa: E402

dev = torch.device("cuda")
for (B, L) in [(1, 32768), (64, 4096), ("cfg3", 32768)]:
    Hq, Hkv, d = 32, 8, 128
    if B == "cfg3":  # the bench workload's inputs (RoPE, planted span)
        from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch
        q, k, _, v = make_batch_torch(CONFIGS["cfg3"], seed=1, device=dev)
        B = 1
    else:
        g = torch.Generator(device=dev).manual_seed(1)
        q = torch.randn(B, Hq, L, d, device=dev, generator=g).bfloat16()
        k = torch.randn(B, Hkv, L, d, device=dev, generator=g).bfloat16()
        v = torch.randn(B, Hkv, L, d, device=dev, generator=g).bfloat16()
    plan = ems.Plan(B, Hq, Hkv, L, d, q.dtype, ems.EmsConfig(256, 32, 0.6, 4.0), dev, "tcgen05", want_out=True)
    for _ in range(3):
        plan.score(q, k, v)
    torch.cuda.synchronize()
    pairs = B * Hkv * (4 * (L // 128) // 2)
    buf = np.zeros((pairs, 6), dtype=np.uint64)
    rc = ems.lib().ems_debug_fwd2_trace(C.c_void_p(buf.ctypes.data), C.c_size_t(buf.nbytes))
    assert rc == 0, rc
    t = buf[:, :5].astype(np.int64)
    t -= t[:, 0].min()
    jmax = (buf[:, 5] & 0xFFFFFFFF).astype(np.int64)
    sm = (buf[:, 5] >> 32).astype(np.int64)
    startup, loop, epi, ex = t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 3] - t[:, 2], t[:, 4] - t[:, 3]
    steps = jmax + 1
    gaps = []
    for s in np.unique(sm):
        idx = np.where(sm == s)[0]
        o = idx[np.argsort(t[idx, 0])]
        gaps += list(t[o[1:], 0] - t[o[:-1], 4])
    gaps = np.array(gaps)
    span = t[:, 4].max()
    busy = (t[:, 4] - t[:, 0]).sum() / (len(np.unique(sm)))
    print(json.dumps({"B": B, "L": L, "pairs": pairs, "span_us": span / 1e3, "sms": int(len(np.unique(sm))),
                      "mean_busy_per_sm_us": busy / 1e3,
                      "startup_us": float(np.median(startup) / 1e3), "loop_us_per_step": float(np.median(loop / steps) / 1e3),
                      "epilogue_us": float(np.median(epi) / 1e3), "exit_us": float(np.median(ex) / 1e3),
                      "gap_us_median": float(np.median(gaps) / 1e3), "gap_us_mean": float(gaps.mean() / 1e3),
                      "overhead_share": float((startup + epi + ex).sum() / (t[:, 4] - t[:, 0]).sum()),
                      "tail_us": float((span - np.sort(t[:, 4])[int(0.5 * len(t))]) / 1e3)}), flush=True)
    del q, k, v, plan
    torch.cuda.empty_cache()
