"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of libems_b200.so once, on shapes that keep the tools' slowdown in seconds.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py

Covered: RoPE, the tcgen05 score pass (P1 CTA pairs + P2, a partial last tile, odd G), the SIMT
score pass (fp32), select (both variants), the tensor-core and SIMT merge assignment, the
weighted-merge bucket + accumulate kernels (config M merges), compact + LUT + check_integrity,
keep-all, the decode step (one CTA and cluster variants) and the diagnostics."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_unit_np  # noqa: E402


def run():
    dev = torch.device("cuda")
    w = CONFIGS["cfgM"]
    units = [make_unit_np(w, seed=3, seq_len=700, unit=u) for u in range(3)]
    t = lambda a, dt: torch.tensor(np.stack(a), dtype=torch.float64).to(dt).to(dev)  # noqa: E731
    for dt, impl in ((torch.bfloat16, "auto"), (torch.float32, "simt")):
        q = t([u.q_rot for u in units], dt).reshape(1, 3, 700, 128).contiguous()
        kr = t([u.k_rot for u in units], dt).reshape(1, 3, 700, 128).contiguous()
        kw = t([u.k_raw for u in units], dt).reshape(1, 3, 700, 128).contiguous()
        v = t([u.v for u in units], dt).reshape(1, 3, 700, 128).contiguous()
        cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
        plan = ems.prefill_compress(q, kr, kw, v, cfg, score_impl=impl)
        plan.sync_status()
    # odd G, raw inputs with RoPE, keep-all
    g = torch.Generator(device=dev).manual_seed(1)
    q = torch.randn((1, 3, 333, 128), generator=g, device=dev).to(torch.bfloat16)
    k = torch.randn((1, 1, 333, 128), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((1, 1, 333, 128), generator=g, device=dev).to(torch.bfloat16)
    ems.prefill(q, k, v, ems.EmsConfig(64, 16, 0.6, 4.0, 7), 1e4).sync_status()
    ems.prefill(q, k, v, ems.EmsConfig(512, 16, 0.6, 4.0, 7), 1e4).sync_status()
    # decode steps on the compressed cache (EMS and SnapKV)
    for pol in ("ems", "snapkv"):
        cfg = ems.EmsConfig(64, 16, 0.6, 4.0, 7, policy=pol)
        plan = ems.prefill(q, k, v, cfg, 1e4)
        ds = ems.DecodeState(1, 3, 1, 333, 128, torch.bfloat16, cfg, 1e4, 333 + 8)
        ds.init_from_plan(plan)
        for _ in range(6):
            ds.step(torch.randn((1, 3, 128), generator=g, device=dev).to(torch.bfloat16),
                    torch.randn((1, 1, 128), generator=g, device=dev).to(torch.bfloat16),
                    torch.randn((1, 1, 128), generator=g, device=dev).to(torch.bfloat16))
        ds.sync_status()
    # diagnostics
    glo = torch.rand((2, 500), device=dev)
    ems.sparsity_rate(glo, glo, 0.9)
    ems.redundancy_rate(torch.randn((2, 300, 128), device=dev).to(torch.bfloat16),
                        torch.randn((2, 300, 128), device=dev).to(torch.bfloat16), 0.5)
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    run()
