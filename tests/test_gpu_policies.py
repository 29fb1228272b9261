"""Baseline prefill policies on the device select/compact kernels:
policy_prefill_compress (proj/src/policies.cpp:131-180) for full, streaming_llm, h2o and
snapkv, against the oracle restatement (pinned to the reference in test_oracle_policies.py).

Kept sets must be identical except tokens whose oracle ranking score lies within 1e-5
relative of the k-th (cut) value, the same exclusion band as the EMS partition (D10).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.oracle import POLICY, Config  # noqa: E402
from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_unit_np  # noqa: E402

CUT_RTOL = 1e-5


def _ecfg(c: Config, policy: str, sink: int = 4):
    return ems.EmsConfig(c.n_budget, c.l_win, c.tau, c.gamma, c.kernel_size, policy=policy, sink_count=sink)


def _cut_band(score, n_cand, k):
    order = sorted(range(n_cand), key=lambda i: (-score[i], i))
    if k >= n_cand:
        return set()
    cut = score[order[k - 1]]
    return {i for i in range(n_cand) if abs(score[i] - cut) <= CUT_RTOL * max(abs(cut), 1e-30)}


@pytest.mark.parametrize("policy", ["streaming", "h2o", "snapkv", "full"])
@pytest.mark.parametrize("wname,L", [("cfg3", 2048), ("cfgM", 1024), ("cfg1", 1024)])
def test_policy_vs_oracle(policy, wname, L, oracle):
    w = CONFIGS[wname]
    units = [make_unit_np(w, seed=17, seq_len=L, unit=u) for u in range(2)]
    c = Config(n_budget=w.n_budget, l_win=w.l_win, tau=w.tau, gamma=w.gamma, kernel_size=w.kernel_size)
    dt = torch.float32 if w.dtype == "f32" else torch.bfloat16
    dev = torch.device("cuda")
    T = lambda a: torch.tensor(np.stack(a), dtype=torch.float64).to(dt).to(dev)  # noqa: E731
    G, n, d = units[0].q_rot.shape
    q = T([u.q_rot for u in units]).reshape(1, 2 * G, n, d).contiguous()
    kr = T([u.k_rot for u in units]).reshape(1, 2, n, d).contiguous()
    kw = T([u.k_raw for u in units]).reshape(1, 2, n, d).contiguous()
    v = T([u.v for u in units]).reshape(1, 2, n, d).contiguous()
    plan = ems.prefill_compress(q, kr, kw, v, _ecfg(c, policy))
    torch.cuda.synchronize()
    for i, un in enumerate(units):
        ref = oracle.prefill_unit(un.q_rot, un.k_rot, un.k_raw, un.v, c)
        glo, loc = ref.extra["glo"], ref.extra["loc"]
        want = oracle.policy_prefill(POLICY[policy], 4, un.k_raw, un.v, glo, loc, c)
        got = plan.unit_cache(i)
        assert got["compressed"] == want.compressed
        np.testing.assert_array_equal(got["local_position"], want.local_position)
        if policy == "full":
            assert len(got["local_position"]) == n and len(got["position"]) == 0
            continue
        n_cand = n - c.l_win
        k = c.n_budget - c.l_win
        if policy == "h2o":
            band = _cut_band(glo, n_cand, k)
        elif policy == "snapkv":
            band = _cut_band(oracle.mean_pool(loc, min(c.kernel_size, n)), n_cand, k)
        else:
            band = set()
        gp, wp = set(got["position"].tolist()), set(want.position.tolist())
        assert (gp ^ wp) <= band, f"kept sets differ outside the cut band: {sorted((gp ^ wp) - band)[:10]}"
        assert len(gp) == len(wp)
        # self-mapped LUT, no merge: slot s <-> s-th kept position
        np.testing.assert_array_equal(got["lut_slot"], np.arange(len(gp)))
        np.testing.assert_array_equal(got["lut_position"], got["position"])
        if not band & (gp ^ wp):
            tol = 1e-4 if w.dtype == "f32" else 2e-2
            err = np.linalg.norm(got["unit_key"] - want.unit_key, axis=1) / np.maximum(
                np.linalg.norm(want.unit_key, axis=1), 1e-30)
            assert err.max() <= tol
            np.testing.assert_allclose(got["score"], want.score, rtol=2e-5 * 10, atol=1e-7)


def test_streaming_known_answer():  # proj/tests/test_policies.cpp:59-72 through the staged ABI
    c = ems.EmsConfig(n_budget=10, l_win=4, gamma=4.0, kernel_size=7, policy="streaming", sink_count=4)
    plan = ems.Plan(1, 1, 1, 100, 8, torch.float32, c, "cuda", want_out=False)
    k = torch.randn((1, 1, 100, 8), device="cuda")
    v = torch.randn((1, 1, 100, 8), device="cuda")
    plan.glo.fill_(1.0)
    plan.loc.fill_(0.1)
    plan.select()
    plan.merge(k, v)
    plan.compact(k, v)
    plan.sync_status()
    got = plan.unit_cache(0)
    kept = set(got["position"].tolist()) | set(got["local_position"].tolist())
    assert kept == {0, 1, 2, 3, 94, 95, 96, 97, 98, 99}


def test_streaming_rejects_small_budget():
    c = ems.EmsConfig(n_budget=6, l_win=4, policy="streaming", sink_count=4)
    with pytest.raises(ems.InvalidArgument):
        ems.Plan(1, 1, 1, 64, 8, torch.float32, c, "cuda")
    with pytest.raises(ems.InvalidArgument):
        ems.make_desc(1, 1, 1, 64, 8, torch.float32, ems.EmsConfig(policy="pyramid"))
