"""Diagnostics on the GPU (csrc/diag.cu) against the oracle
(ems_oracle_sparsity_rate / ems_oracle_redundancy_rate_direct, pinned to the reference in
tests/test_oracle_diagnostics.py):

* sparsity_rate(combine_glo_loc(glo, loc), zeta): identical rates on the same fp32 glo/loc
  (the oracle widens them to fp64), over zeta in (0, 1], ties, zeros, L up to 32768, and the
  criterion-11 brute force with glo = loc = score (align = 1, combined = score);
* redundancy_rate_direct(k, v, tau): the tensor-core path (bf16, d = 128) and the SIMT path
  (fp32 / other d) against the oracle on the same values (fp32 accumulation against fp64:
  tokens whose best similarity sits within 1e-5 of tau are excluded from the comparison);
* analyze() (analyze_trace) through device RoPE + prefill_scores;
* DegenerateInputError when a unit has no score mass.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2412_08521_b200 import ems  # noqa: E402
from tests.test_oracle_diagnostics import brute_sparsity  # noqa: E402


def _best_r(k, v):
    """Per-token best R over earlier tokens (fp64), for the near-tau exclusion."""
    def unit(a):
        n = np.linalg.norm(a, axis=1, keepdims=True)
        return np.where(n > 0, a / np.where(n > 0, n, 1), 0)
    ck = np.clip(unit(k) @ unit(k).T, -1, 1)
    cv = np.clip(unit(v) @ unit(v).T, -1, 1)
    r = ck * cv
    r[np.triu_indices(len(k))] = -np.inf
    return r.max(axis=1)


def _check_redundancy(oracle, k, v, tau, got):
    """got = the GPU rate; exact unless tokens lie within 1e-5 of tau (counted as either)."""
    want = oracle.redundancy_rate_direct(k, v, tau)
    best = _best_r(k, v)[1:]
    near = int(np.sum(np.abs(best - tau) < 1e-5))
    assert abs(got - want) * len(k) <= near + 1e-9, (got, want, near)


@pytest.mark.parametrize("L", [1, 5, 1000, 4096, 32768])
def test_sparsity_matches_oracle(oracle, L):
    rng = np.random.default_rng(L)
    U = 3
    glo = (rng.exponential(1.0, (U, L)) ** 2).astype(np.float32)
    loc = np.where(rng.random((U, L)) < 0.1, rng.exponential(0.5, (U, L)), 0).astype(np.float32)
    glo[1, rng.integers(0, L, L // 4)] = 0
    loc[:, -1] = 0.25  # some local mass in every unit (align > 0)
    glo[2] = np.round(glo[2] * 2) / 2 + 0.5  # many exact ties
    g, lo = torch.tensor(glo, device="cuda"), torch.tensor(loc, device="cuda")
    for zeta in (0.01, 0.5, 0.9, 0.95, 1.0):
        got = ems.sparsity_rate(g, lo, zeta).cpu().numpy()
        for u in range(U):
            comb = oracle.combine(glo[u], loc[u])
            want = oracle.sparsity_rate(comb, zeta)
            if zeta == 1.0:  # whether the running sum reaches exactly 1 is rounding (either answer)
                assert got[u] in (want, 1.0 - np.count_nonzero(comb) / L), (u, got[u], want)
            else:
                assert got[u] == want, (u, zeta, got[u], want)


def test_sparsity_criterion_11_brute_force():
    rng = np.random.default_rng(23000)
    scores = (rng.uniform(0, 1, (10, 32)) + 1e-6).astype(np.float32)
    s = torch.tensor(scores, device="cuda")
    prev = np.ones(10)
    for zi in range(1, 11):
        got = ems.sparsity_rate(s, s, 0.1 * zi).cpu().numpy()  # glo = loc: align 1, combined = score
        for r in range(10):
            assert got[r] == brute_sparsity(scores[r].astype(np.float64), 0.1 * zi)
        assert (got <= prev + 1e-15).all()
        prev = got


def test_sparsity_degenerate_and_arguments():
    g = torch.zeros((2, 64), device="cuda")
    with pytest.raises(ems.DegenerateInputError):
        ems.sparsity_rate(g, torch.ones_like(g), 0.5)
    with pytest.raises(ems.InvalidArgument):
        ems.sparsity_rate(torch.ones_like(g), g, 0.0)
    with pytest.raises(ems.InvalidArgument):
        ems.sparsity_rate(torch.ones_like(g), g, 1.5)


@pytest.mark.parametrize("dtype,d,L", [(torch.float32, 16, 300), (torch.float32, 64, 1000),
                                       (torch.bfloat16, 32, 700), (torch.bfloat16, 128, 100),
                                       (torch.bfloat16, 128, 1000), (torch.bfloat16, 128, 4096)])
def test_redundancy_matches_oracle(oracle, reflib, dtype, d, L):
    U = 2
    q, k, v = reflib.gen_trace(1, 900 + L + d, L, U, d, 1, level=0.8)  # redundant: merges and misses
    kt = torch.tensor(k[:, :L], dtype=torch.float32).to(dtype).cuda()
    vt = torch.tensor(v[:, :L], dtype=torch.float32).to(dtype).cuda()
    kt[0, 7] = 0  # a zero-norm token
    kk, vv = kt.double().cpu().numpy(), vt.double().cpu().numpy()
    for tau in (0.3, 0.6, 0.9):
        got = ems.redundancy_rate(kt, vt, tau).cpu().numpy()
        for u in range(U):
            _check_redundancy(oracle, kk[u], vv[u], tau, got[u])


def test_redundancy_random_tensor_cores_vs_simt(oracle):
    rng = np.random.default_rng(5)
    U, L, d = 2, 2000, 128
    k = torch.tensor(rng.standard_normal((U, L, d)), dtype=torch.float32).to(torch.bfloat16).cuda()
    v = torch.tensor(rng.standard_normal((U, L, d)), dtype=torch.float32).to(torch.bfloat16).cuda()
    k[:, 1000:1100] = k[:, 10:110]  # exact duplicates: R = 1
    v[:, 1000:1100] = v[:, 10:110]
    for tau in (0.05, 0.1, 0.999):
        tc = ems.redundancy_rate(k, v, tau).cpu().numpy()
        os.environ["EMS_DIAG_SIMT"] = "1"
        try:
            simt = ems.redundancy_rate(k, v, tau).cpu().numpy()
        finally:
            del os.environ["EMS_DIAG_SIMT"]
        kk, vv = k.double().cpu().numpy(), v.double().cpu().numpy()
        for u in range(U):
            _check_redundancy(oracle, kk[u], vv[u], tau, tc[u])
            _check_redundancy(oracle, kk[u], vv[u], tau, simt[u])
    assert (ems.redundancy_rate(k, v, 0.999).cpu().numpy() >= 100 / L).all()


def test_analyze_matches_reference_pipeline(oracle, reflib):
    """analyze_trace: RoPE + prefill_scores(min(l_win, n)) + combine + sparsity, redundancy of raw K/V."""
    from paper_2412_08521_b200.inputs import rope_np
    H, n, d = 2, 257, 32
    q, k, v = reflib.gen_trace(0, 77, n, H, d, 1)
    q, k, v = (np.asarray(a[:, :n], dtype=np.float32).astype(np.float64) for a in (q, k, v))
    cfg = ems.EmsConfig(n_budget=64, l_win=16, tau=0.5)
    t = lambda a: torch.tensor(a[None], dtype=torch.float32, device="cuda")  # noqa: E731
    sp, rd = ems.analyze(t(q), t(k), t(v), cfg, 1e4)
    glo, loc = ems.prefill_scores(ems.rope(t(q), 1e4), ems.rope(t(k), 1e4), 16)
    for h in range(H):
        g, lo = glo[0, h].double().cpu().numpy(), loc[0, h].double().cpu().numpy()
        assert sp[0, h].item() == oracle.sparsity_rate(oracle.combine(g, lo), cfg.zeta)
        _check_redundancy(oracle, k[h], v[h], cfg.tau, rd[0, h].item())
        # against the reference's fp64 scores: the same rate up to score rounding
        _, gr, lr = reflib.prefill_attention(rope_np(q[h], 1e4), rope_np(k[h], 1e4), None, 16)
        assert abs(sp[0, h].item() - oracle.sparsity_rate(oracle.combine(gr, lr), cfg.zeta)) <= 2.0 / n
