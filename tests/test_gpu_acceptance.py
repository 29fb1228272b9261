"""The reference's acceptance battery (proj/tests/acceptance.cpp) restated against the GPU path
(SURVEY.md 8f, f3): the device prefill (scores, select, merge, compact, RoPE) and the device
EMS decode loop, on the reference's own synthetic traces (gen_synthetic through oracle/_ref,
test infrastructure only) and a numpy fp64 dense reference (run_reference,
proj/src/experiment.cpp:42-80).

Differences from the reference battery, each deliberate:
  * the GPU computes in fp32 (keys/values/logits) with fp64 score accumulators, so the fp64
    reference's 1e-9 / 1e-12 thresholds become fp32-level ones (stated per criterion);
  * head_dim is restricted to the sizes the kernels support (8..128);
  * criterion 4 (identity policy, "errors exactly 0") becomes "errors at fp32 rounding level";
  * criterion 11 runs the GPU diagnostics (csrc/diag.cu) against the brute-force oracles.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import rope_np  # noqa: E402

BASE = 1e4  # run_experiment's RoPE base (proj/src/experiment.cpp:167)


def _t(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def dense_reference(q, k, v, n):
    """Dense full-cache run: causal prefill outputs [H][n][d], decode outputs [S][H][d], argmax [S][H]."""
    H, T, d = q.shape
    qr, kr = rope_np(q, BASE), rope_np(k, BASE)
    scale = 1.0 / np.sqrt(d)
    pre = np.zeros((H, n, d))
    outs = np.zeros((T - n, H, d))
    am = np.zeros((T - n, H), dtype=np.int64)
    for h in range(H):
        s = qr[h, :n] @ kr[h, :n].T * scale
        s[np.triu_indices(n, 1)] = -np.inf
        p = np.exp(s - s.max(axis=1, keepdims=True))
        pre[h] = (p / p.sum(axis=1, keepdims=True)) @ v[h, :n]
        for st in range(T - n):
            row = n + st
            lg = kr[h, :row + 1] @ qr[h, row] * scale
            pr = np.exp(lg - lg.max())
            pr /= pr.sum()
            outs[st, h] = pr @ v[h, :row + 1]
            am[st, h] = int(np.argmax(pr))
    return pre, outs, am


def gpu_run(q, k, v, n, cfg: ems.EmsConfig):
    """ems.prefill on the prompt (raw, device RoPE) then the device decode loop."""
    H, T, d = q.shape
    plan = ems.prefill(_t(q[None, :, :n]), _t(k[None, :, :n]), _t(v[None, :, :n]), cfg, BASE)
    ds = ems.DecodeState(1, H, H, n, d, torch.float32, cfg, BASE, T + 1)
    ds.init_from_plan(plan)
    outs, ams, entries = [], [], []
    for s in range(T - n):
        o, a = ds.step(_t(q[None, :, n + s]), _t(k[None, :, n + s]), _t(v[None, :, n + s]))
        outs.append(o[0].double().cpu().numpy())
        ams.append(a[0].long().cpu().numpy())
        meta = ds.state["meta"].cpu().numpy()
        entries.append(meta[:, 1] + meta[:, 5])  # locals + live centers per head
    return plan, ds, plan.out[0].double().cpu().numpy(), np.array(outs), np.array(ams), np.array(entries)


def l2(a, b):  # concat_l2, proj/src/experiment.cpp:86-95
    return float(np.sqrt(((a - b) ** 2).sum()))


# -- 1. streaming scores vs the dense three-step oracle ---------------------------------
def test_c1_scores_vs_three_step(oracle):
    worst = 0.0
    for heads in (1, 4):
        for n in (1, 2, 31, 32, 33, 128, 1024):
            rng = np.random.default_rng(100 * n + heads)
            q, k = _f32(rng.standard_normal((heads, n, 16))), _f32(rng.standard_normal((heads, n, 16)))
            lw = min(32, n)
            glo, loc = ems.prefill_scores(_t(q[None]), _t(k[None]), lw)
            for h in range(heads):
                g3, l3 = oracle.three_step_scores(q[h], k[h], lw)
                g, lo = glo[0, h].double().cpu().numpy(), loc[0, h].double().cpu().numpy()
                worst = max(worst, float(np.max(np.abs(g - g3) / np.maximum(np.abs(g3), 1e-300))))
                worst = max(worst, float(np.max(np.abs(lo - l3) / np.maximum(np.abs(l3), 1e-12))))
    assert worst <= 2e-5, worst  # fp32 (reference fp64: 1e-9)


# -- 2. mass conservation after prefill -----------------------------------------------
def test_c2_mass_conservation():
    worst_g = worst_l = 0.0
    for seed in range(50):
        rng = np.random.default_rng(7000 + seed)
        q, k = rng.standard_normal((1, 1, 96, 8)), rng.standard_normal((1, 1, 96, 8))
        glo, loc = ems.prefill_scores(_t(q), _t(k), 24)
        worst_g = max(worst_g, abs(glo.double().sum().item() - 96))
        worst_l = max(worst_l, abs(loc.double().sum().item() - 24))
    assert worst_g <= 1e-4 and worst_l <= 1e-4, (worst_g, worst_l)  # fp32 (reference: 1e-6)


# -- 3. Glo-Loc combination properties (select kernel, pooling window 1) ---------------
def test_c3_combine_properties():
    rng = np.random.default_rng(42)
    dom, worst_mean, stable = True, 0.0, True
    cfg = ems.EmsConfig(n_budget=8, l_win=2, gamma=1.0, kernel_size=1)
    for rep in range(100):
        n = 32
        glo, loc = rng.uniform(0, 4, n), rng.uniform(0, 4, n)
        glo[rep % n] += 0.5
        alpha = rng.uniform(1e-3, 1e3)
        outs = []
        for g in (glo, glo * alpha):
            plan = ems.Plan(1, 1, 1, n, 8, torch.float32, cfg, "cuda", want_out=False)
            plan.glo.copy_(torch.tensor(g, dtype=torch.float32).reshape(1, 1, n))
            plan.loc.copy_(torch.tensor(loc, dtype=torch.float32).reshape(1, 1, n))
            plan.select()
            plan.sync_status()
            outs.append(plan.stage["pooled"][0].double().cpu().numpy())
        g32, l32 = _f32(glo), _f32(loc)
        dom = dom and bool(np.all(outs[0] >= l32 * (1 - 1e-7)))
        worst_mean = max(worst_mean, abs((g32 * (l32.sum() / g32.sum())).sum() - l32.sum()) / n)
        o1 = sorted(range(n), key=lambda i: (-outs[0][i], i))
        o2 = sorted(range(n), key=lambda i: (-outs[1][i], i))
        stable = stable and (o1 == o2 or np.allclose(outs[0][o1], outs[0][o2], rtol=1e-6))
    assert dom and worst_mean <= 1e-9 and stable


# -- 4. identity policy: the full cache reproduces dense attention ---------------------------
def test_c4_full_policy_is_dense_attention(reflib):
    from paper_2412_08521_b200.trace import Trace, TraceStep, run_experiment
    cfg = ems.EmsConfig(n_budget=32, l_win=8, policy="full")
    worst = 0.0
    for seed in range(10):
        q, k, v = reflib.gen_trace(0, 9000 + seed, 48, 2, 16, 256)
        tr = Trace(2, 16, [TraceStep(0, _f32(q[:, :48]), _f32(k[:, :48]), _f32(v[:, :48]))] +
                   [TraceStep(1, _f32(q[:, i:i + 1]), _f32(k[:, i:i + 1]), _f32(v[:, i:i + 1]))
                    for i in range(48, 48 + 256)])
        r = run_experiment(tr, cfg, label=f"identity-{seed}")["policies"][0]
        assert r["policy"] == "full" and not r["compression_applied"]
        assert all(m["argmax_match"] for m in r["steps"])
        assert [m["entries"] for m in r["steps"]] == [2 * (48 + s) for s in range(257)]
        worst = max(worst, max(m["l2_error"] for m in r["steps"]), max(m["cos_error"] for m in r["steps"]))
    assert worst <= 1e-5, worst  # fp32 keys/values/logits (reference fp64: exactly 0)


# -- 5. zero-class merge path vs explicit eviction path --------------------------------
def test_c5_zero_class_equals_explicit_removal(reflib):
    rng = np.random.default_rng(77)
    worst = 0.0
    for rep in range(20):
        n = int(rng.integers(40, 161))
        d = 8 if rep % 2 else 16
        steps = int(rng.integers(8, 41))
        l_win = 4 + n % 5
        cfg = dict(n_budget=max(l_win + 4, n // 4), l_win=l_win, tau=float(rng.uniform(0, 1)),
                   gamma=float(rng.uniform(1, 5)), kernel_size=1 + 2 * (rep % 4))
        q, k, v = reflib.gen_trace(0 if rep % 2 == 0 else 1, 11000 + rep, n, 1, d, steps, level=0.5)
        q, k, v = _f32(q), _f32(k), _f32(v)
        _, _, pa, oa, _, _ = gpu_run(q, k, v, n, ems.EmsConfig(**cfg, zero_class=True))
        _, _, pb, ob, _, _ = gpu_run(q, k, v, n, ems.EmsConfig(**cfg, zero_class=False))
        worst = max(worst, float(np.abs(pa - pb).max()), float(np.abs(oa - ob).max()))
    assert worst == 0.0, worst  # the two realisations expand the same rows: bit-identical


# -- 6. tau = 1 and gamma = 1 reductions -------------------------------------------------
def test_c6_tau_one_and_gamma_one(oracle):
    for seed in range(20):
        rng = np.random.default_rng(13000 + seed)
        q, k, v = (_f32(rng.standard_normal((1, 96, 8))) for _ in range(3))
        base = dict(n_budget=24, l_win=8, kernel_size=5)
        a = ems.prefill(_t(q[None]), _t(k[None]), _t(v[None]), ems.EmsConfig(**base, tau=1.0, gamma=4.0), BASE)
        b = ems.prefill(_t(q[None]), _t(k[None]), _t(v[None]), ems.EmsConfig(**base, gamma=1.0), BASE)
        ca, cb = a.unit_cache(0), b.unit_cache(0)
        for name in ("position", "unit_key", "key_norm", "value", "local_position", "local_key", "local_value"):
            np.testing.assert_array_equal(ca[name], cb[name], err_msg=name)
        # gamma = 1 is pure pooled-score top-k eviction
        qr, kr = rope_np(q[0], BASE), rope_np(k[0], BASE)
        _, glo, loc, _ = oracle.prefill_attention(_f32(qr), _f32(kr), None, l_win=8)
        pooled = oracle.effective_score(glo, loc, np.zeros(96), 5)
        order = sorted(range(88), key=lambda i: (-pooled[i], i))
        cut = pooled[order[15]]
        band = {i for i in range(88) if abs(pooled[i] - cut) <= 1e-5 * cut}
        assert (set(cb["position"].tolist()) ^ set(order[:16])) <= band


# -- 7. duplicate losslessness at a 25% budget --------------------------------------------
def test_c7_duplicates_are_lossless():
    worst, constructed = 0.0, True
    for seed in range(5):
        rng = np.random.default_rng(15000 + seed)
        n, d, n_base = 256, 16, 48
        k = np.zeros((n + 4, d))
        v = np.zeros((n + 4, d))
        k[:n_base], v[:n_base] = _f32(rng.standard_normal((n_base, d))), _f32(rng.standard_normal((n_base, d)))
        for i in range(n_base, n + 4):
            src = rng.integers(0, n_base)
            k[i], v[i] = k[src], v[src]
        q = _f32(0.02 * rng.standard_normal((n + 4, d)))
        cfg = ems.EmsConfig(n_budget=64, l_win=16, tau=0.6, gamma=4.0, kernel_size=7)
        plan, ds, pre, outs, _, _ = gpu_run(q[None], k[None], v[None], n, cfg)
        ref_pre, ref_outs, _ = dense_reference(q[None], k[None], v[None], n)
        worst = max(worst, l2(pre, ref_pre[0]) / max(l2(ref_pre[0], 0 * ref_pre[0]), 1e-30))
        for s in range(4):
            worst = max(worst, l2(outs[s], ref_outs[s]) / max(l2(ref_outs[s], 0 * ref_outs[s]), 1e-30))
        constructed = constructed and bool((plan.unit_cache(0)["lut_slot"] >= 0).all())
    assert constructed, "a duplicate token went to the zero class"
    assert worst <= 1e-5, worst  # fp32 (reference fp64: 1e-9)


# -- 8. budget and byte-accounting invariants over a long decode ---------------------------
def test_c8_budget_over_1000_decodes():
    rng = np.random.default_rng(16000)
    n, d, steps = 256, 8, 1000
    q, k, v = (_f32(rng.standard_normal((2, n + steps, d))) for _ in range(3))
    cfg = ems.EmsConfig(n_budget=64, l_win=16, tau=0.6, gamma=3.0, kernel_size=7)
    _, ds, _, _, _, entries = gpu_run(q, k, v, n, cfg)
    assert (entries == cfg.n_budget).all(), "stored entries != budget"
    meta = ds.state["meta"].cpu().numpy()
    lut_cap = int(cfg.gamma * cfg.n_budget)
    assert (meta[:, 2] <= lut_cap).all()
    for h in range(2):  # bytes_stored identity (cache.cpp:40-46): 8 (2 E d + 4 E + lut)
        c = ds.unit_cache(h)
        e = len(c["position"]) + len(c["local_position"])
        assert e == cfg.n_budget and 8 * (2 * e * d + 4 * e + len(c["lut_position"])) > 0


# -- 9. needle retrieval analog at a 2% budget (EMS arm vs the H2O arm) ------------------
def test_c9_needle_retained_at_two_percent(reflib):
    n, retained, h2o = 4096, 0, 0
    cfg = ems.EmsConfig(n_budget=81, l_win=16, tau=0.55, gamma=4.0, kernel_size=7)
    cfg_h2o = ems.EmsConfig(n_budget=81, l_win=16, tau=0.55, gamma=4.0, kernel_size=7, policy="h2o")
    depths = (0.1, 0.3, 0.5, 0.7, 0.9)
    runs = 0
    for seed in range(8):
        for depth in depths:
            q, k, v = reflib.gen_trace(2, 20000 + seed, n, 1, 32, 8, depth=depth)
            q, k, v = _f32(q), _f32(k), _f32(v)
            _, _, ref_am = dense_reference(q, k, v, n)
            _, _, _, _, ams, _ = gpu_run(q, k, v, n, cfg)
            retained += int((ams == ref_am).all())
            _, _, _, _, ams, _ = gpu_run(q, k, v, n, cfg_h2o)
            h2o += int((ams == ref_am).all())
            runs += 1
    assert retained >= 0.95 * runs and h2o < retained, f"ems retained {retained}/{runs}, h2o {h2o}/{runs}"


# -- 10. merging beats evict-only on redundant traces ---------------------------------------
def test_c10_merge_beats_evict_only(reflib):
    wins = 0
    base = dict(n_budget=96, l_win=16, tau=0.6, kernel_size=7)
    for seed in range(10):
        q, k, v = reflib.gen_trace(1, 21000 + seed, 512, 2, 16, 32, level=0.8)
        q, k, v = _f32(q), _f32(k), _f32(v)
        _, ref_outs, _ = dense_reference(q, k, v, 512)
        _, _, _, oa, _, _ = gpu_run(q, k, v, 512, ems.EmsConfig(**base, gamma=4.0))
        _, _, _, ob, _, _ = gpu_run(q, k, v, 512, ems.EmsConfig(**base, gamma=1.0))
        la = np.mean([l2(oa[s], ref_outs[s]) for s in range(32)])
        lb = np.mean([l2(ob[s], ref_outs[s]) for s in range(32)])
        wins += int(la < lb)
    assert wins >= 8, f"merge beats evict-only in {wins}/10"


# -- 11. sparsity / redundancy rates against brute force, monotone in zeta and tau -------------
def test_c11_diagnostics_vs_brute_force():
    from tests.test_oracle_diagnostics import brute_redundancy, brute_sparsity
    rng = np.random.default_rng(23000)
    worst = 0.0
    for _ in range(10):
        n = 32
        k, v = _f32(rng.standard_normal((n, 8))), _f32(rng.standard_normal((n, 8)))
        score = _f32(rng.uniform(0.0, 1.0, n) + 1e-6)
        s = _t(score)[None]
        prev = 1.0
        for zi in range(1, 11):  # glo = loc = score: align 1, combined = score
            p = ems.sparsity_rate(s, s, 0.1 * zi).item()
            worst = max(worst, abs(p - brute_sparsity(score, 0.1 * zi)))
            assert p <= prev + 1e-15
            prev = p
        prev = 1.0
        for ti in range(10):
            r = ems.redundancy_rate(_t(k)[None], _t(v)[None], 0.1 * ti).item()
            want = brute_redundancy(k, v, 0.1 * ti)
            # fp32 similarities: a token within 1e-5 of tau may land on either side
            best = np.array([max(float(np.dot(k[t], k[j]) / np.linalg.norm(k[t]) / np.linalg.norm(k[j])) *
                                 float(np.dot(v[t], v[j]) / np.linalg.norm(v[t]) / np.linalg.norm(v[j]))
                                 for j in range(t)) for t in range(1, n)])
            near = int(np.sum(np.abs(best - 0.1 * ti) < 1e-5))
            assert abs(r - want) * n <= near + 1e-9, (ti, r, want)
            assert r <= prev + 1e-15
            prev = r
    assert worst <= 1e-12, worst


# -- 12. determinism: the whole run twice, byte-identical ----------------------------------
def test_c12_two_runs_identical(reflib):
    q, k, v = reflib.gen_trace(1, 31000, 300, 2, 16, 20, level=0.8)
    q, k, v = _f32(q), _f32(k), _f32(v)
    cfg = ems.EmsConfig(n_budget=48, l_win=8, tau=0.5, gamma=3.0, kernel_size=5)
    r1 = gpu_run(q, k, v, 300, cfg)
    r2 = gpu_run(q, k, v, 300, cfg)
    assert np.array_equal(r1[2], r2[2]) and np.array_equal(r1[3], r2[3]) and np.array_equal(r1[4], r2[4])
    for key in r1[1].state:
        assert torch.equal(r1[1].state[key], r2[1].state[key]), key
