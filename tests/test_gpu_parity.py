"""GPU parity: the CUDA path (through the C ABI) against the oracle on identical inputs.

Bars (BASELINE.json north_star; see tests/parity.py):
  * important / TBM sets bit-exact outside the 1e-5 cut band,
  * merge destinations identical outside the 1e-5 R band,
  * merged K/V and scores within 2e-2 (bf16) / 1e-4 (fp32) per-row relative error,
  * glo/loc within SCORE_RTOL of the fp64 oracle (the scores feed the cut).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.oracle import Cache, Config  # noqa: E402
from paper_2412_08521_b200 import ems  # noqa: E402
from paper_2412_08521_b200.inputs import CONFIGS, make_unit_np, rope_np, round_to  # noqa: E402
from tests.parity import compare_unit  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCORE_RTOL = {"f32": 2e-5, "bf16": 2e-5}


def _tdt(dtype):
    return torch.float32 if dtype == "f32" else torch.bfloat16


def run_gpu(units, dtype, cfg: Config, score_impl="auto"):
    """units: list of UnitInputs-like (q_rot [G,n,d], k_rot, k_raw, v [n,d]) -> Plan (B=1, H_kv=U)."""
    dev = torch.device("cuda")
    t = lambda a: torch.tensor(np.stack(a), dtype=torch.float64).to(_tdt(dtype)).to(dev)  # noqa: E731
    G, n, d = units[0].q_rot.shape
    q = t([u.q_rot for u in units]).reshape(1, len(units) * G, n, d).contiguous()
    kr = t([u.k_rot for u in units]).reshape(1, len(units), n, d).contiguous()
    kw = t([u.k_raw for u in units]).reshape(1, len(units), n, d).contiguous()
    v = t([u.v for u in units]).reshape(1, len(units), n, d).contiguous()
    ecfg = ems.EmsConfig(cfg.n_budget, cfg.l_win, cfg.tau, cfg.gamma, cfg.kernel_size,
                         cfg.zero_class, cfg.key_only)
    plan = ems.prefill_compress(q, kr, kw, v, ecfg, want_out=True, score_impl=score_impl)
    torch.cuda.synchronize()
    return plan


class U:  # minimal UnitInputs
    def __init__(self, q_rot, k_rot, k_raw, v):
        self.q_rot, self.k_rot, self.k_raw, self.v = q_rot, k_rot, k_raw, v


def check_unit(plan, u, unit_in, ref_cache: Cache, glo_ref, loc_ref, dtype, cfg: Config, oracle,
               out_ref=None):
    n = unit_in.k_raw.shape[0]
    glo = plan.glo[0, u].double().cpu().numpy()
    loc = plan.loc[0, u].double().cpu().numpy()
    g_err = np.max(np.abs(glo - glo_ref) / np.maximum(glo_ref, 1e-30))
    l_mask = loc_ref > 1e-6
    l_err = np.max(np.abs(loc - loc_ref)[l_mask] / loc_ref[l_mask]) if l_mask.any() else 0.0
    assert g_err <= SCORE_RTOL[dtype], f"glo rel err {g_err}"
    assert l_err <= SCORE_RTOL[dtype] * 10, f"loc rel err {l_err}"
    if out_ref is not None:
        G = unit_in.q_rot.shape[0]
        o = plan.out[0, u * G:(u + 1) * G].double().cpu().numpy()
        tol = 1e-4 if dtype == "f32" else 2e-2
        err = np.max(np.linalg.norm(o - out_ref, axis=-1) / np.maximum(np.linalg.norm(out_ref, axis=-1), 1e-30))
        assert err <= tol, f"attention output rel err {err}"
    # reference R on the reference's own TBM set, for the destination exclusion band
    r_ref, tbm_ref = None, None
    if ref_cache.compressed and "cls" in ref_cache.extra:
        cls = ref_cache.extra["cls"]
        tbm_ref = np.nonzero(cls == 1)[0]
        imp_ref = np.nonzero(cls == 2)[0]
        if len(tbm_ref):
            r_ref = oracle.redundancy_cross(unit_in.k_raw[tbm_ref], unit_in.v[tbm_ref],
                                            unit_in.k_raw[imp_ref], unit_in.v[imp_ref], cfg.key_only)
    pooled_ref = ref_cache.extra.get("pooled")
    if pooled_ref is None:
        pooled_ref = oracle.effective_score(glo_ref, loc_ref, np.zeros(n), min(cfg.kernel_size, n))
    return compare_unit(plan.unit_cache(u), ref_cache, dtype, pooled_ref, cfg, n, r_ref, tbm_ref)


# ---------------------------------------------------------------------------------------
def test_gpu_golden_cache(oracle):
    """The reference's golden fixture, through the GPU path (fp32 inputs, d = 8)."""
    tr = np.load(os.path.join(GOLDEN, "golden_trace.npz"))
    with open(os.path.join(GOLDEN, "golden_cache.json")) as f:
        want = Cache.from_dump_json(f.read())
    cfg = Config(n_budget=12, l_win=4, tau=0.6, gamma=2.0, kernel_size=3)
    units = []
    for h in range(2):
        q_rot = round_to(rope_np(tr["q"][h], 10000.0), "f32")
        k_rot = round_to(rope_np(tr["k"][h], 10000.0), "f32")
        units.append(U(q_rot[None], k_rot, tr["k"][h], tr["v"][h]))
    plan = run_gpu(units, "f32", cfg)
    ref0 = oracle.prefill_unit(units[0].q_rot, units[0].k_rot, units[0].k_raw, units[0].v, cfg)
    rep = check_unit(plan, 0, units[0], ref0, ref0.extra["glo"], ref0.extra["loc"], "f32", cfg, oracle)
    # and directly against the fixture
    got = plan.unit_cache(0)
    np.testing.assert_array_equal(got["position"], want.position)
    np.testing.assert_array_equal(got["lut_position"], want.lut_position)
    np.testing.assert_array_equal(got["lut_slot"], want.lut_slot)
    np.testing.assert_allclose(got["unit_key"], want.unit_key, rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(got["score"], want.score, rtol=1e-4, atol=1e-7)
    assert rep["excluded_tokens"] <= 2  # pooled ties at the cut (golden has two)


with open(os.path.join(GOLDEN, "ref_cases.json")) as _f:
    REF_META = json.load(_f)


@pytest.mark.parametrize("name", sorted(REF_META))
def test_gpu_reference_cases(name, oracle):
    """Reference-generated fixtures (tests/golden/make_golden.py): merges, zero class,
    explicit removal, keep-all, gamma = 1, tau = 0, GQA, bf16."""
    meta = REF_META[name]
    arr = np.load(os.path.join(GOLDEN, "ref_cases.npz"))
    cfg = Config(**meta["config"])
    u = U(arr[f"{name}/q_rot"], arr[f"{name}/k_rot"], arr[f"{name}/k_raw"], arr[f"{name}/v"])
    plan = run_gpu([u], meta["dtype"], cfg)
    ref = oracle.prefill_unit(u.q_rot, u.k_rot, u.k_raw, u.v, cfg)  # pinned == reference
    ref_json = Cache.from_dump_json(meta["cache_json"])
    np.testing.assert_array_equal(ref.lut_position, ref_json.lut_position)
    check_unit(plan, 0, u, ref, arr[f"{name}/glo"], arr[f"{name}/loc"], meta["dtype"], cfg, oracle,
               out_ref=arr[f"{name}/out"])


def _cfg_of(w):
    return Config(n_budget=w.n_budget, l_win=w.l_win, tau=w.tau, gamma=w.gamma,
                  kernel_size=w.kernel_size)


@pytest.mark.parametrize("wname,L,n_units", [("cfg1", None, 8), ("cfgM", 2048, 2), ("cfg3", 4096, 1),
                                             ("cfg4", 2048, 4), ("cfg2", 2048, 2)])
def test_gpu_configs_vs_oracle(wname, L, n_units, oracle):
    """BASELINE configs (config 1 in full; the others at oracle-tractable L)."""
    w = CONFIGS[wname]
    units = [make_unit_np(w, seed=7, seq_len=L, unit=u) for u in range(n_units)]
    cfg = _cfg_of(w)
    plan = run_gpu(units, w.dtype, cfg)
    reps = []
    for i, un in enumerate(units):
        ref = oracle.prefill_unit(un.q_rot, un.k_rot, un.k_raw, un.v, cfg)
        reps.append(check_unit(plan, i, un, ref, ref.extra["glo"], ref.extra["loc"], w.dtype, cfg,
                               oracle))
    if wname == "cfgM":
        assert all(r["merged"] > 0 and r["zero_class"] > 0 for r in reps), reps


def test_gpu_determinism():
    w = CONFIGS["cfgM"]
    units = [make_unit_np(w, seed=3, seq_len=1024, unit=u) for u in range(2)]
    a = run_gpu(units, w.dtype, _cfg_of(w))
    b = run_gpu(units, w.dtype, _cfg_of(w))
    for k in a.cache:
        assert torch.equal(a.cache[k], b.cache[k]), k
    assert torch.equal(a.glo, b.glo) and torch.equal(a.loc, b.loc)
    assert torch.equal(a.out, b.out)


def test_gpu_degenerate_input_raises():
    """combine_glo_loc: zero global mass -> DegenerateInputError (scoring.cpp:115-117)."""
    cfg = ems.EmsConfig(n_budget=8, l_win=2, gamma=2.0, kernel_size=3)
    plan = ems.Plan(1, 1, 1, 64, 16, torch.float32, cfg, "cuda", want_out=False)
    plan.glo.zero_()
    plan.loc.fill_(1.0)
    plan.select()
    with pytest.raises(ems.DegenerateInputError):
        plan.sync_status()


def test_gpu_redundancy_cross_matches_oracle(oracle):
    rng = np.random.default_rng(5)
    kr, vr = rng.standard_normal((37, 64)), rng.standard_normal((37, 64))
    kc, vc = rng.standard_normal((21, 64)), rng.standard_normal((21, 64))
    kc[3] = 0.0  # zero-norm token -> similarity 0
    kr[5], vr[5] = kc[7] * 2.0, vc[7] * 0.5  # duplicate direction -> R = 1
    dev = torch.device("cuda")
    T = lambda a: torch.tensor(a, dtype=torch.float32, device=dev)  # noqa: E731
    r = ems.redundancy_cross(T(kr), T(vr), T(kc), T(vc)).cpu().numpy()
    want = oracle.redundancy_cross(kr, vr, kc, vc)
    np.testing.assert_allclose(r, want, atol=2e-6)
    assert abs(r[5, 7] - 1.0) < 1e-5 and np.all(r[:, 3] == 0.0)


@pytest.mark.parametrize("wname,L,key_only,budget", [("cfgM", 2048, False, None), ("cfgM", 2048, True, None),
                                                    ("cfg3b", 4096, False, None), ("cfgM", 4096, False, 1024)])
def test_gpu_tc_merge_matches_simt_and_oracle(wname, L, key_only, budget, oracle):
    """Tensor-core similarity/argmax (merge_tc.cu) vs the SIMT kernels and the oracle; the
    budget-1024 merge case streams 8 center tiles through the 2-stage ring (stage reuse)."""
    w = CONFIGS[wname]
    units = [make_unit_np(w, seed=5, seq_len=L, unit=u) for u in range(2)]
    cfg = _cfg_of(w)
    cfg.key_only = key_only
    if budget:
        cfg.n_budget = budget
    a = run_gpu(units, w.dtype, cfg, score_impl="auto")
    b = run_gpu(units, w.dtype, cfg, score_impl="simt")
    for i, un in enumerate(units):
        ref = oracle.prefill_unit(un.q_rot, un.k_rot, un.k_raw, un.v, cfg)
        rep = check_unit(a, i, un, ref, ref.extra["glo"], ref.extra["loc"], w.dtype, cfg, oracle)
        check_unit(b, i, un, ref, ref.extra["glo"], ref.extra["loc"], w.dtype, cfg, oracle)
        if wname == "cfgM":
            assert rep["merged"] > 0


@pytest.mark.parametrize("forced", ["0", "1"])
def test_gpu_select_variants_forced(forced):
    """Both select kernels (one CTA per unit / the 8-CTA cluster) against the oracle on every
    config case; the launch picks one by shape, so each is forced once in a fresh process."""
    import subprocess
    import sys
    env = dict(os.environ, EMS_SELECT_CLUSTER=forced)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__,
                        "-k", "configs_vs_oracle or golden_cache or reference_cases"],
                       env=env, capture_output=True, text=True, cwd=os.path.dirname(os.path.dirname(__file__)))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_gpu_cache_dump_json_round_trips_through_reference_schema():
    """ems.cache_dump_json writes the reference's cache_dump_json schema (cache.cpp:114-150):
    read back with the parser of that schema, every field of the GPU cache is unchanged."""
    w = CONFIGS["cfgM"]
    un = make_unit_np(w, seed=21, seq_len=1024, unit=0)
    cfg = _cfg_of(w)
    plan = run_gpu([un], w.dtype, cfg)
    c = plan.unit_cache(0)
    back = Cache.from_dump_json(ems.cache_dump_json(c, un.q_rot.shape[2]))
    np.testing.assert_array_equal(back.position, c["position"])
    np.testing.assert_array_equal(back.lut_position, c["lut_position"])
    np.testing.assert_array_equal(back.lut_slot, c["lut_slot"])
    np.testing.assert_array_equal(back.local_position, c["local_position"])
    np.testing.assert_array_equal(back.unit_key, c["unit_key"])
    np.testing.assert_array_equal(back.score, c["score"])
    np.testing.assert_array_equal(back.value, c["value"])
    np.testing.assert_array_equal(back.local_key, c["local_key"])
    assert back.compressed == c["compressed"] and back.extra["slots"] == list(range(len(c["position"])))


def test_gpu_degenerate_full_path_leaves_valid_stage():
    """NaN inputs reach the select kernel as zero / NaN global mass: the whole prefill (score ->
    select -> merge -> compact) over a workspace of garbage (0xFF) raises DegenerateInputError
    (scoring.cpp:115-117) without touching memory outside its buffers, and the next call on the
    same plan is clean."""
    w = CONFIGS["cfgM"]
    un = make_unit_np(w, seed=4, seq_len=1024, unit=0)
    dev = torch.device("cuda")
    t = lambda a, s: torch.tensor(a, dtype=torch.float64).to(torch.bfloat16).to(dev).reshape(s).contiguous()  # noqa: E731
    q, kr, kw, v = t(un.q_rot, (1, 1, 1024, 128)), t(un.k_rot, (1, 1, 1024, 128)), \
        t(un.k_raw, (1, 1, 1024, 128)), t(un.v, (1, 1, 1024, 128))
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    plan = ems.Plan(1, 1, 1, 1024, 128, torch.bfloat16, cfg, dev)
    plan.workspace.fill_(0xFF)
    for name in plan.stage:
        plan.stage[name].view(torch.uint8).fill_(0xFF)
    qn = q.clone()
    qn[0, 0, 5] = float("nan")
    plan.run(qn, kr, kw, v)
    with pytest.raises(ems.DegenerateInputError):
        plan.sync_status()
    cnt = plan.cache["counts"][0].tolist()
    assert cnt[0] == 0 and cnt[2] == 0 and cnt[1] == w.l_win  # no centers, no LUT, exact locals
    plan.run(q, kr, kw, v)
    plan.sync_status()  # clean again
    assert plan.cache["counts"][0, 0].item() == w.n_budget - w.l_win


def test_gpu_corrupt_stage_raises_corruption_error():
    """HeadCacheState::check_integrity (cache.cpp:66-80) on the device: a caller-supplied stage
    whose merge destination names a nonexistent center slot gives CorruptionError from the
    compact step (and the merge kernels skip the bad entry instead of writing out of bounds)."""
    w = CONFIGS["cfgM"]
    un = make_unit_np(w, seed=6, seq_len=1024, unit=0)
    dev = torch.device("cuda")
    t = lambda a: torch.tensor(a, dtype=torch.float64).to(torch.bfloat16).to(dev).reshape(1, 1, 1024, 128).contiguous()  # noqa: E731
    q, kr, kw, v = t(un.q_rot), t(un.k_rot), t(un.k_raw), t(un.v)
    cfg = ems.EmsConfig(w.n_budget, w.l_win, w.tau, w.gamma, w.kernel_size)
    plan = ems.Plan(1, 1, 1, 1024, 128, torch.bfloat16, cfg, dev)
    plan.score(q, kr, v)
    plan.select()
    plan.merge(kw, v)
    plan.sync_status()
    plan.stage["dest"][0, 3] = 10 ** 6  # no such slot
    plan.compact(kw, v)
    with pytest.raises(ems.CorruptionError):
        plan.sync_status()


def _path_fuzz_cases(n=8, seed=77):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        L = int(rng.integers(200, 1400))
        l_win = int(rng.integers(4, 48))
        budget = int(rng.integers(l_win + 8, max(l_win + 9, L // 3)))
        gamma = float(rng.choice([1.0, 1.5, 2.0, 4.0]))
        tau = float(rng.choice([0.0, 0.3, 0.6, 0.9]))
        k = int(rng.choice([1, 3, 7]))
        G = int(rng.choice([1, 2, 4]))
        out.append((i, L, l_win, budget, gamma, tau, k, G))
    return out


@pytest.mark.parametrize("case", _path_fuzz_cases())
def test_gpu_path_fuzz_vs_oracle(case, oracle):
    """Seeded random (L, l_win, budget, gamma, tau, pooling kernel, G) on redundant K/V (merges
    and zero-class tokens both occur): the whole bf16 prefill-compress path against the C
    restatement of the reference, with the D10 bands."""
    i, L, l_win, budget, gamma, tau, k, G = case
    w = CONFIGS["cfgM"]
    rng = np.random.default_rng([i, L])
    units = []
    for u in range(2):
        base = make_unit_np(w, seed=100 + i, seq_len=L, unit=u)
        q = round_to(rng.standard_normal((G, L, base.q_rot.shape[-1])), "bf16")
        units.append(U(q, base.k_rot, base.k_raw, base.v))
    cfg = Config(n_budget=budget, l_win=l_win, tau=tau, gamma=gamma, kernel_size=k)
    plan = run_gpu(units, "bf16", cfg)
    for u, un in enumerate(units):
        ref = oracle.prefill_unit(un.q_rot, un.k_rot, un.k_raw, un.v, cfg)
        check_unit(plan, u, un, ref, ref.extra["glo"], ref.extra["loc"], "bf16", cfg, oracle)
