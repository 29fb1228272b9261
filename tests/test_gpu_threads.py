"""Reentrancy of the C ABI (SURVEY.md 8b "Threading"): the reference runs its per-head
functions from OpenMP threads (proj/src/engine.cpp:65-76); the boundary must be safe across
host threads on distinct streams and workspaces.  Four host threads each run prefill +
the decode loop on their own stream, plan and state; every result equals the same work run
alone, bit for bit (the kernels are deterministic)."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2412_08521_b200 import ems  # noqa: E402


def _inputs(seed, B=1, H=2, G=2, L=1024, d=128):
    g = torch.Generator(device="cuda").manual_seed(seed)
    mk = lambda *s: torch.randn(s, generator=g, device="cuda").to(torch.bfloat16)  # noqa: E731
    return mk(B, H * G, L, d), mk(B, H, L, d), mk(B, H, L, d), [(mk(B, H * G, d), mk(B, H, d), mk(B, H, d))
                                                                 for _ in range(6)]


def _work(seed, stream, out):
    cfg = ems.EmsConfig(n_budget=96, l_win=16, tau=0.5, gamma=3.0, kernel_size=5)
    with torch.cuda.stream(stream):
        q, k, v, steps = _inputs(seed)
        plan = ems.Plan(1, q.shape[1], k.shape[1], q.shape[2], q.shape[3], q.dtype, cfg, "cuda")
        plan.run_raw(q, k, v, 1e4)
        ds = ems.DecodeState(1, q.shape[1], k.shape[1], q.shape[2], q.shape[3], q.dtype, cfg, 1e4, q.shape[2] + 8)
        ds.init_from_plan(plan)
        outs = [ds.step(*x, stream=stream)[0].clone() for x in steps]
        plan.sync_status(stream)
    out[seed] = (plan.glo.clone(), {kk: t.clone() for kk, t in plan.cache.items()}, outs)


def test_concurrent_host_threads_match_sequential():
    seeds = [11, 12, 13, 14]
    seq = {}
    for s in seeds:
        _work(s, torch.cuda.Stream(), seq)
    par = {}
    threads = [threading.Thread(target=_work, args=(s, torch.cuda.Stream(), par)) for s in seeds]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert set(par) == set(seeds)
    for s in seeds:
        g0, c0, o0 = seq[s]
        g1, c1, o1 = par[s]
        assert torch.equal(g0, g1)
        for k in c0:
            assert torch.equal(c0[k], c1[k]), (s, k)
        for a, b in zip(o0, o1):
            assert torch.equal(a, b)
    # different inputs gave different caches (the threads did not share state)
    assert not np.array_equal(seq[11][1]["center_pos"].cpu().numpy(), seq[12][1]["center_pos"].cpu().numpy())
