"""Pins the C restatement (oracle/ems_oracle.c) before anything is compared to it.

1. the reference's own golden fixture (golden_cache.json) from the golden trace;
2. reference outputs committed in tests/golden/ref_cases.* (made by the reference
   itself, tests/golden/make_golden.py);
3. the known-answer cases of proj/tests/test_{scoring,numerics,compressor,analysis}.cpp.
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import Cache, Config, DegenerateInput, InvalidArgument

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def assert_cache_equal(got: Cache, want: Cache, rtol=1e-12, atol=1e-12):
    assert got.compressed == want.compressed
    np.testing.assert_array_equal(got.position, want.position)
    np.testing.assert_array_equal(got.local_position, want.local_position)
    np.testing.assert_array_equal(got.lut_position, want.lut_position)
    np.testing.assert_array_equal(got.lut_slot, want.lut_slot)
    for name in ("unit_key", "key_norm", "value", "score", "local_key", "local_value",
                 "local_score"):
        np.testing.assert_allclose(getattr(got, name), getattr(want, name), rtol=rtol, atol=atol,
                                   err_msg=name)


# -- 1. golden fixture -------------------------------------------------------------
def test_golden_cache_from_golden_trace(oracle):
    """test_experiment.cpp:163-170: head-0 cache after EMS prefill of the golden trace,
    config {budget 12, w 4, tau 0.6, gamma 2, kernel 3} (test_experiment.cpp:22-31)."""
    tr = np.load(os.path.join(GOLDEN, "golden_trace.npz"))
    with open(os.path.join(GOLDEN, "golden_cache.json")) as f:
        want = Cache.from_dump_json(f.read())
    cfg = Config(n_budget=12, l_win=4, tau=0.6, gamma=2.0, kernel_size=3)
    q_rot = oracle.rope(tr["q"][0], 10000.0)
    k_rot = oracle.rope(tr["k"][0], 10000.0)
    got = oracle.prefill_unit(q_rot[None], k_rot, tr["k"][0], tr["v"][0], cfg)
    assert_cache_equal(got, want)
    # fixture facts quoted in SURVEY.md section 4
    assert list(want.position) == [0, 1, 2, 3, 5, 6, 7, 11]
    assert list(want.local_position) == [12, 13, 14, 15]
    assert [int(p) for p, s in zip(want.lut_position, want.lut_slot) if s < 0] == [4, 8, 9, 10]


# -- 2. reference-generated cases ----------------------------------------------------
with open(os.path.join(GOLDEN, "ref_cases.json")) as _f:
    REF_META = json.load(_f)


@pytest.mark.parametrize("name", sorted(REF_META))
def test_ref_case(oracle, name):
    meta = REF_META[name]
    arr = np.load(os.path.join(GOLDEN, "ref_cases.npz"))
    cfg = Config(**meta["config"])
    got = oracle.prefill_unit(arr[f"{name}/q_rot"], arr[f"{name}/k_rot"], arr[f"{name}/k_raw"],
                              arr[f"{name}/v"], cfg, want_out=True)
    np.testing.assert_allclose(got.extra["glo"], arr[f"{name}/glo"], rtol=1e-12)
    np.testing.assert_allclose(got.extra["loc"], arr[f"{name}/loc"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(got.extra["out"], arr[f"{name}/out"], rtol=1e-11, atol=1e-13)
    assert_cache_equal(got, Cache.from_dump_json(meta["cache_json"]))


# -- 3. known answers ------------------------------------------------------------------
def test_single_token_unit_glo(oracle):  # test_scoring.cpp:37-44
    rng = np.random.default_rng(1)
    _, glo, loc, _ = oracle.prefill_attention(rng.standard_normal((1, 8)), rng.standard_normal((1, 8)))
    assert glo.tolist() == [1.0]


def test_harmonic_closed_form(oracle):  # test_scoring.cpp:46-63
    n = 40
    q = np.zeros((n, 4))
    _, glo, _, _ = oracle.prefill_attention(q, q.copy(), l_win=8)
    want = np.array([sum(1.0 / (i + 1) for i in range(j, n)) for j in range(n)])
    np.testing.assert_allclose(glo, want, rtol=1e-12)
    g3, _ = oracle.three_step_scores(q, q, 8)
    np.testing.assert_allclose(glo, g3, rtol=1e-12)


def test_streaming_matches_three_step(oracle):  # test_scoring.cpp:65-77, acceptance criterion 1
    for n in (1, 2, 31, 32, 33, 128, 300):
        rng = np.random.default_rng(100 * n)
        q, k = rng.standard_normal((n, 16)), rng.standard_normal((n, 16))
        lw = min(32, n)
        _, glo, loc, _ = oracle.prefill_attention(q, k, l_win=lw)
        g3, l3 = oracle.three_step_scores(q, k, lw)
        np.testing.assert_allclose(glo, g3, rtol=1e-9)
        np.testing.assert_allclose(loc, l3, rtol=1e-9, atol=1e-300)


def test_window_edges(oracle):  # test_scoring.cpp:79-101
    rng = np.random.default_rng(7)
    q, k = rng.standard_normal((24, 8)), rng.standard_normal((24, 8))
    _, glo, loc, _ = oracle.prefill_attention(q, k, l_win=24)
    np.testing.assert_allclose(loc, glo, rtol=1e-15)
    q, k = rng.standard_normal((17, 8)), rng.standard_normal((17, 8))
    _, glo, loc, _ = oracle.prefill_attention(q, k, l_win=1)
    _, l3 = oracle.three_step_scores(q, k, 1)
    np.testing.assert_allclose(loc, l3, atol=1e-12)


def test_mass_conservation(oracle):  # test_scoring.cpp:110-123, acceptance criterion 2
    for seed in range(10):
        rng = np.random.default_rng(7000 + seed)
        q, k = 2 * rng.standard_normal((96, 8)), 2 * rng.standard_normal((96, 8))
        _, glo, loc, _ = oracle.prefill_attention(q, k, l_win=24)
        assert abs(glo.sum() - 96) < 1e-6 and abs(loc.sum() - 24) < 1e-6


def test_combine_known_answers(oracle):  # test_scoring.cpp:138-184
    s = np.array([0.5, 1.5, 2.0])
    assert oracle.combine(s, s).tolist() == s.tolist()
    np.testing.assert_allclose(oracle.combine([4.0, 0.0], [0.0, 2.0]), [2.0, 2.0], rtol=1e-15)
    with pytest.raises(DegenerateInput):
        oracle.combine([0.0, 0.0], [1.0, 1.0])


def test_mean_pool_known_answers(oracle):  # test_numerics.cpp:133-156
    s = np.array([3.0, 1.0, 4.0, 1.0, 5.0])
    assert oracle.mean_pool(s, 1).tolist() == s.tolist()
    assert oracle.mean_pool(np.full(9, 2.5), 5).tolist() == [2.5] * 9
    np.testing.assert_allclose(oracle.mean_pool([0, 0, 9.0, 0, 0], 3), [0, 3, 3, 3, 0], rtol=1e-15)
    with pytest.raises(InvalidArgument):
        oracle.mean_pool([1.0, 2.0, 3.0], 2)
    with pytest.raises(InvalidArgument):
        oracle.mean_pool([1.0, 2.0], 3)


def test_partition_known_answers(oracle):  # test_compressor.cpp:63-114
    c = Config(n_budget=8, l_win=4, tau=0.6, gamma=1.5, kernel_size=1)
    p = oracle.partition(20.0 - np.arange(20.0), c)
    assert p["important"].tolist() == [0, 1, 2, 3]
    assert p["tbm"].tolist() == [4, 5, 6, 7]
    assert p["irrelevant"].tolist() == list(range(8, 16))
    assert p["local"].tolist() == [16, 17, 18, 19]
    p = oracle.partition(np.ones(8), c)
    assert p["important"].tolist() == [0, 1, 2, 3] and p["tbm"].size == 0
    with pytest.raises(InvalidArgument):
        oracle.partition(np.ones(3), c)
    tiny = Config(n_budget=6, l_win=2, gamma=1.0, kernel_size=1)
    p = oracle.partition(np.full(9, 5.0), tiny)
    assert p["important"].tolist() == [0, 1, 2, 3] and p["irrelevant"].tolist() == [4, 5, 6]


def test_assign_known_answers(oracle):  # test_compressor.cpp:116-148
    r = np.array([[0.3, 0.7, 0.5]])
    assert oracle.assign(r, 0.6).tolist() == [1]
    assert oracle.assign(r, 0.71).tolist() == [-1]
    r = np.array([[0.0, -0.5], [0.2, 0.9], [0.1, 0.1]])
    assert oracle.assign(r, 0.0).tolist() == [0, 1, 0]


def test_redundancy_known_answers(oracle):  # test_analysis.cpp:39-111
    rng = np.random.default_rng(2)
    k, v = rng.standard_normal((4, 6)), rng.standard_normal((4, 6))
    k[3], v[3] = k[1], v[1]
    r = oracle.redundancy_cross(k, v, k, v)
    assert abs(r[3, 1] - 1) < 1e-12 and abs(r[1, 1] - 1) < 1e-12
    k2 = np.array([[1.0, 0.0], [1.0, 0.0]])
    v2 = np.array([[1.0, 0.0], [0.0, 1.0]])
    assert oracle.redundancy_cross(k2, v2, k2, v2)[1, 0] == 0.0
    kz = np.array([[0.0, 0.0], [1.0, 0.0]])
    vz = np.array([[0.0, 1.0], [0.0, 1.0]])
    rz = oracle.redundancy_cross(kz, vz, kz, vz)
    assert rz[1, 0] == 0.0 and rz[0, 0] == 0.0


def test_budget_exact_and_unit_norms(oracle):  # test_compressor.cpp:261-287
    rng = np.random.default_rng(40)
    n, c = 64, Config(n_budget=16, l_win=4, gamma=2.0, tau=0.6, kernel_size=7)
    k, v = rng.standard_normal((n, 8)), rng.standard_normal((n, 8))
    glo, lp = rng.uniform(0.05, 1, n), rng.uniform(0.05, 1, n)
    cache = oracle.compress_prefill(k, v, glo, lp, c=c)
    assert cache.compressed and len(cache.position) == c.center_capacity()
    assert len(cache.local_position) == c.l_win
    assert len(cache.lut_position) == c.center_capacity() + c.tbm_target()
    np.testing.assert_allclose(np.linalg.norm(cache.unit_key, axis=1), 1.0, atol=1e-9)


def test_tau_one_equals_evict_only(oracle):  # test_compressor.cpp:225-259, criterion 6a
    rng = np.random.default_rng(12)
    n = 32
    k, v = rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
    glo, lp = rng.uniform(0.05, 1, n), rng.uniform(0.05, 1, n)
    base = Config(n_budget=8, l_win=4, tau=0.6, gamma=1.5, kernel_size=1)
    a = oracle.compress_prefill(k, v, glo, lp, c=Config(**{**base.__dict__, "gamma": 1.0}))
    b = oracle.compress_prefill(k, v, glo, lp, c=Config(**{**base.__dict__, "tau": 1.0}))
    np.testing.assert_array_equal(a.position, b.position)
    np.testing.assert_array_equal(a.unit_key, b.unit_key)
    np.testing.assert_array_equal(a.value, b.value)
    assert set(zip(b.lut_position[b.lut_slot >= 0], b.lut_slot[b.lut_slot >= 0])) <= \
        set(zip(a.lut_position, a.lut_slot))


def test_keep_all_path(oracle):  # test_compressor.cpp:289-300
    rng = np.random.default_rng(41)
    c = Config(n_budget=8, l_win=4, gamma=1.5, kernel_size=1)
    k, v = rng.standard_normal((6, 4)), rng.standard_normal((6, 4))
    cache = oracle.compress_prefill(k, v, rng.uniform(size=6), rng.uniform(size=6), c=c)
    assert not cache.compressed and len(cache.position) == 0
    np.testing.assert_array_equal(cache.local_key, k)
    np.testing.assert_array_equal(cache.local_position, np.arange(6))
