"""Per-CTA phase times of P2 from an instrumented variant (tools/make_trace_variants.py):
start -> first S -> loop end -> combine done -> exit, and the gap between CTAs on one SM.
EMS_LIB_PATH=_variants/p2trace.so python tools/p2_trace_probe.py"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_batch_torch  # noqa: E402

dev = torch.device("cuda")
for cfg in ["cfg3", "cfg2"]:
    w = CONFIGS[cfg]
    q, k, _, v = make_batch_torch(w, seed=1, device=dev)
    B, Hq, L, d = q.shape
    plan = ems.Plan(B, Hq, w.heads_kv, L, d, q.dtype, ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma), dev,
                    "tcgen05", want_out=True)
    for _ in range(3):
        plan.score(q, k, v)
    torch.cuda.synchronize()
    N = 1 << 16
    buf = np.zeros((N, 5), dtype=np.uint64)
    assert ems.lib().ems_debug_colsum_trace(C.c_void_p(buf.ctypes.data), C.c_size_t(buf.nbytes)) == 0
    units = B * w.heads_kv
    G = Hq // w.heads_kv
    nT = (L + 127) // 128
    hs = 1
    while hs < G and G % (2 * hs) == 0 and ((nT + 1) // 2) * units * hs < 4 * 148:
        hs *= 2
    n = ((nT + 1) // 2) * units * hs
    t = buf[:n, :4].astype(np.int64)
    sm = (buf[:n, 4] >> 40).astype(np.int64)
    tend = (buf[:n, 4] & 0xFFFFFFFFFF).astype(np.int64)
    base = t[:, 0].min()
    t0, t1, t2, t3 = (t[:, i] - base for i in range(4))
    te = tend - (base & 0xFFFFFFFFFF)
    gaps = []
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        o = idx[np.argsort(t0[idx])]
        gaps += list(t0[o[1:]] - te[o[:-1]])
    gaps = np.array(gaps)
    busy = (te - t0).sum()
    print(json.dumps({"cfg": cfg, "ctas": n, "span_us": float(te.max() / 1e3),
                      "startup_us": float(np.median(t1 - t0) / 1e3), "loop_us_median": float(np.median(t2 - t1) / 1e3),
                      "combine_us": float(np.median(t3 - t2) / 1e3), "exit_us": float(np.median(te - t3) / 1e3),
                      "gap_us": float(np.median(gaps) / 1e3),
                      "overhead_share": float(((t1 - t0) + (t3 - t2) + (te - t3)).sum() / busy + np.clip(gaps, 0, None).sum() / busy)}),
          flush=True)
