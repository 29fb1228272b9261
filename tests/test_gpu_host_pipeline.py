"""ems_prefill_host: engine::prefill from pinned host tensors with the copy/compute pipeline.

* chunks == 1 must reproduce the device-resident path bit for bit (same kernels, same order);
* chunks > 1 runs contiguous unit groups as sub-problems (possibly with a different colsum
  head split, i.e. a different fp64 summation order), so it is checked against the oracle
  with the usual parity bars, and for determinism.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.oracle import Config  # noqa: E402
from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_unit_np  # noqa: E402
from tests.test_gpu_parity import check_unit  # noqa: E402


def _host(a, dtype):
    return torch.tensor(a).to(dtype).contiguous().pin_memory()


def _cfg(w):
    return Config(n_budget=w.n_budget, l_win=w.l_win, tau=w.tau, gamma=w.gamma, kernel_size=w.kernel_size)


def _ecfg(c: Config):
    return ems.EmsConfig(c.n_budget, c.l_win, c.tau, c.gamma, c.kernel_size, c.zero_class, c.key_only)


def _stack(units, attr):
    a = np.stack([getattr(u, attr) for u in units])
    n, d = a.shape[-2], a.shape[-1]
    return a.reshape(1, -1, n, d)


@pytest.mark.parametrize("chunks", [1, 2, 3])
def test_host_pipeline_prerotated_vs_oracle(chunks, oracle):
    w = CONFIGS["cfgM"]
    units = [make_unit_np(w, seed=13, seq_len=1024, unit=u) for u in range(3)]
    cfg = _cfg(w)
    dt = torch.bfloat16
    hq, hkr, hkw, hv = (_host(_stack(units, a), dt) for a in ("q_rot", "k_rot", "k_raw", "v"))
    G = units[0].q_rot.shape[0]
    plan = ems.Plan(1, 3 * G, 3, 1024, 128, dt, _ecfg(cfg), "cuda", want_out=True)
    hc = plan.run_host(hq, hkr, hv, 0.0, h_k_raw=hkw, chunks=chunks)
    plan.sync_status()
    for name in hc:  # the host copy is the device cache
        assert torch.equal(hc[name], plan.cache[name].cpu()), name
    for i, un in enumerate(units):
        ref = oracle.prefill_unit(un.q_rot, un.k_rot, un.k_raw, un.v, cfg)
        rep = check_unit(plan, i, un, ref, ref.extra["glo"], ref.extra["loc"], "bf16", cfg, oracle)
        assert rep["merged"] > 0
    if chunks == 1:  # identical to the device-resident path
        d = ems.prefill_compress(hq.cuda(), hkr.cuda(), hkw.cuda(), hv.cuda(), _ecfg(cfg))
        torch.cuda.synchronize()
        for name in d.cache:
            assert torch.equal(d.cache[name], plan.cache[name]), name
        assert torch.equal(d.out, plan.out)


@pytest.mark.parametrize("chunks", [1, 4])
def test_host_pipeline_raw_rope(chunks):
    """Raw inputs: RoPE on the device per chunk; equals ems_prefill (device-resident, raw)."""
    w = CONFIGS["cfg3"]
    rng = np.random.default_rng(3)
    H, G, L = 4, 4, 2048
    dt = torch.bfloat16
    q = torch.tensor(rng.standard_normal((1, H * G, L, 128))).to(dt)
    k = torch.tensor(rng.standard_normal((1, H, L, 128))).to(dt)
    v = torch.tensor(rng.standard_normal((1, H, L, 128))).to(dt)
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    plan = ems.prefill_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), cfg, w.rope_base, chunks=chunks)
    ref = ems.prefill(q.cuda(), k.cuda(), v.cuda(), cfg, w.rope_base)
    torch.cuda.synchronize()
    assert torch.equal(plan.q_rot, ref.q_rot) and torch.equal(plan.k_rot, ref.k_rot)
    hc = plan.host_cache()
    if chunks == 1:
        for name in ref.cache:
            assert torch.equal(hc[name], ref.cache[name].cpu()), name
    else:  # same selection (scores agree to fp32 rounding), identical positions
        np.testing.assert_allclose(plan.glo.cpu().numpy(), ref.glo.cpu().numpy(), rtol=1e-6)
        for name in ("center_pos", "lut_pos", "lut_slot", "local_pos", "counts"):
            assert torch.equal(hc[name], ref.cache[name].cpu()), name
    # PrefillResult.per_head outputs come back to the host with the caches; every (head, query
    # tile) item is computed the same way whatever the grouping (chunks = 4 also runs the first
    # group's forward pass in two halves of the heads), so O is bit-identical
    assert torch.equal(plan.host_out, plan.out.cpu())
    assert torch.equal(plan.out, ref.out)
    # determinism of the chunked pipeline
    again = ems.prefill_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), cfg, w.rope_base, chunks=chunks)
    for name, t in again.host_cache().items():
        assert torch.equal(t, hc[name]), name


def test_host_pipeline_rejects_pageable_and_missing_kraw():
    cfg = ems.EmsConfig(64, 8, 0.6, 4.0, 7)
    plan = ems.Plan(1, 2, 1, 256, 128, torch.bfloat16, cfg, "cuda")
    x = torch.zeros((1, 2, 256, 128), dtype=torch.bfloat16)
    kk = torch.zeros((1, 1, 256, 128), dtype=torch.bfloat16)
    with pytest.raises(ems.InvalidArgument):
        plan.run_host(x, kk.pin_memory(), kk.pin_memory(), 1e4)  # pageable q
    with pytest.raises(ems.InvalidArgument):
        plan.run_host(x.pin_memory(), kk.pin_memory(), kk.pin_memory(), 0.0)  # no k_raw


def test_host_pipeline_concurrent_groups_equal_sequential():
    """Two unit groups in flight (second stream + workspace) give the same bits as one at a time."""
    w = CONFIGS["cfg3"]
    rng = np.random.default_rng(4)
    H, G, L = 6, 4, 1024
    dt = torch.bfloat16
    q, k, v = (torch.tensor(rng.standard_normal(s)).to(dt).pin_memory()
               for s in ((1, H * G, L, 128), (1, H, L, 128), (1, H, L, 128)))
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    plan = ems.Plan(1, H * G, H, L, 128, dt, cfg, "cuda")
    res = []
    for concurrent in (False, True):
        hc = plan.run_host(q, k, v, w.rope_base, chunks=6, concurrent=concurrent)
        plan.sync_status()
        res.append(({n: t.clone() for n, t in hc.items()}, plan.glo.clone(), plan.out.clone()))
    for n in res[0][0]:
        assert torch.equal(res[0][0][n], res[1][0][n]), n
    assert torch.equal(res[0][1], res[1][1]) and torch.equal(res[0][2], res[1][2])


def test_host_pipeline_split_first_group_odd_part():
    """G = 6: the first group's forward pass runs in two parts of 3 heads (pairs straddle query
    tiles, an odd item count gets a dummy partner); O, LSE-derived scores and caches equal the
    device-resident path."""
    w = CONFIGS["cfg3"]
    rng = np.random.default_rng(6)
    H, G, L = 3, 6, 1100
    dt = torch.bfloat16
    q = torch.tensor(rng.standard_normal((1, H * G, L, 128))).to(dt)
    k = torch.tensor(rng.standard_normal((1, H, L, 128))).to(dt)
    v = torch.tensor(rng.standard_normal((1, H, L, 128))).to(dt)
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    plan = ems.prefill_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), cfg, w.rope_base, chunks=3)
    ref = ems.prefill(q.cuda(), k.cuda(), v.cuda(), cfg, w.rope_base)
    torch.cuda.synchronize()
    assert torch.equal(plan.q_rot, ref.q_rot) and torch.equal(plan.k_rot, ref.k_rot)
    assert torch.equal(plan.out, ref.out)
    np.testing.assert_allclose(plan.glo.cpu().numpy(), ref.glo.cpu().numpy(), rtol=1e-6)
    hc = plan.host_cache()
    for name in ("center_pos", "lut_pos", "lut_slot", "local_pos", "counts"):
        assert torch.equal(hc[name], ref.cache[name].cpu()), name


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_host_pipeline_rope_table_first_position(dtype):
    """The host pipeline's once-per-call RoPE table (positions first_position + l) rotates exactly
    like the device-resident path's per-launch sines, for bf16 and fp32."""
    w = CONFIGS["cfg3"]
    rng = np.random.default_rng(8)
    H, G, L, first = 2, 2, 700, 1234
    q = torch.tensor(rng.standard_normal((1, H * G, L, 128))).to(dtype)
    k = torch.tensor(rng.standard_normal((1, H, L, 128))).to(dtype)
    v = torch.tensor(rng.standard_normal((1, H, L, 128))).to(dtype)
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    plan = ems.prefill_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), cfg, w.rope_base, chunks=2,
                            first_position=first)
    ref = ems.prefill(q.cuda(), k.cuda(), v.cuda(), cfg, w.rope_base, first_position=first)
    torch.cuda.synchronize()
    assert torch.equal(plan.q_rot, ref.q_rot) and torch.equal(plan.k_rot, ref.k_rot)
    assert torch.equal(plan.out, ref.out)
