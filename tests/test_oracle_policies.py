"""Pins the oracle's baseline policies (ems_oracle_policy_prefill, restating
proj/src/policies.cpp:131-180) before the GPU select/compact kernels are compared to them:

1. the prefill known answers of proj/tests/test_policies.cpp (streaming sinks + recent,
   short prompts unchanged, H2O under a uniform history, SnapKV = brute-force top-k of the
   pooled local score, H2O == evict-only EMS with a silenced local score, purity,
   PolicyHandle::validate);
2. the reference itself (oracle/_ref, policy_prefill_compress) on seeded inputs, including
   quantised scores with many exact ties.
"""
import numpy as np
import pytest

from oracle.oracle import POLICY, Config, InvalidArgument
from tests.test_oracle import assert_cache_equal


def kept_positions(cache):  # test_policies.cpp:33-45
    return set(cache.position.tolist()) | set(cache.local_position.tolist())


def flat(n):  # test_policies.cpp:47-54
    return np.ones(n), np.full(n, 0.1)


def test_streaming_keeps_sinks_plus_recent(oracle):  # test_policies.cpp:59-72
    rng = np.random.default_rng(1)
    n = 100
    k, v = rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
    c = Config(n_budget=10, l_win=4)
    cache = oracle.policy_prefill(POLICY["streaming"], 4, k, v, *flat(n), c)
    assert kept_positions(cache) == {0, 1, 2, 3, 94, 95, 96, 97, 98, 99}
    assert len(cache.position) + len(cache.local_position) == c.n_budget


@pytest.mark.parametrize("policy", ["streaming", "h2o", "snapkv", "full"])
def test_short_prompts_unchanged(oracle, policy):  # test_policies.cpp:74-85, 144-155
    rng = np.random.default_rng(2)
    k, v = rng.standard_normal((8, 4)), rng.standard_normal((8, 4))
    cache = oracle.policy_prefill(POLICY[policy], 4, k, v, *flat(8), Config(n_budget=10, l_win=4))
    assert not cache.compressed and len(cache.local_position) == 8 and len(cache.position) == 0


def test_h2o_uniform_history_keeps_earliest(oracle):  # test_policies.cpp:123-142
    n, d = 64, 4
    z = np.zeros((n, d))
    _, glo, loc, _ = oracle.prefill_attention(z, z, z, l_win=4)
    cache = oracle.policy_prefill(POLICY["h2o"], 4, z, z, glo, loc, Config(n_budget=12, l_win=4))
    assert kept_positions(cache) == set(range(8)) | set(range(60, 64))


def test_snapkv_is_topk_of_pooled_local(oracle):  # test_policies.cpp:193-231
    rng = np.random.default_rng(7)
    n, d = 80, 8
    q, k, v = (rng.standard_normal((n, d)) for _ in range(3))
    qr, kr = oracle.rope(q), oracle.rope(k)
    _, glo, loc, _ = oracle.prefill_attention(qr, kr, v, l_win=8)
    c = Config(n_budget=20, l_win=8, kernel_size=7)
    cache = oracle.policy_prefill(POLICY["snapkv"], 4, k, v, glo, loc, c)
    pooled = oracle.mean_pool(loc, 7)
    order = sorted(range(n - 8), key=lambda i: (-pooled[i], i))
    assert kept_positions(cache) == set(order[:12]) | set(range(n - 8, n))


def test_h2o_equals_evict_only_ems_with_silent_local(oracle):  # test_policies.cpp:233-260
    rng = np.random.default_rng(9)
    n = 64
    k, v = rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
    glo, loc = rng.uniform(0.1, 2.0, n), np.full(n, 1e-12)
    c = Config(n_budget=16, l_win=4, gamma=1.0, kernel_size=1)
    a = oracle.policy_prefill(POLICY["ems"], 4, k, v, glo, loc, c)
    b = oracle.policy_prefill(POLICY["h2o"], 4, k, v, glo, loc, c)
    assert kept_positions(a) == kept_positions(b)


def test_policies_are_pure(oracle):  # test_policies.cpp:262-277
    rng = np.random.default_rng(8)
    n = 48
    k, v = rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
    for p in POLICY.values():
        a = oracle.policy_prefill(p, 4, k, v, *flat(n), Config(n_budget=12, l_win=4))
        b = oracle.policy_prefill(p, 4, k, v, *flat(n), Config(n_budget=12, l_win=4))
        assert_cache_equal(a, b, rtol=0, atol=0)


def test_streaming_validate_rejects_small_budget(oracle):  # test_policies.cpp:279-289
    k = np.zeros((20, 4))
    with pytest.raises(InvalidArgument):
        oracle.policy_prefill(POLICY["streaming"], 4, k, k, *flat(20), Config(n_budget=6, l_win=4))


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("policy", sorted(POLICY))
def test_policies_match_reference(oracle, reflib, policy, seed):
    """The restatement against the reference's own policy_prefill_compress."""
    rng = np.random.default_rng(100 + seed)
    n, d = (300, 16) if seed < 2 else (97, 8)
    k, v = rng.standard_normal((n, d)), rng.standard_normal((n, d))
    glo = rng.random(n)
    loc = rng.random(n) * (np.arange(n) > n - 40)
    if seed == 1:  # quantised scores: many exact ties at the cut (ties -> lower index)
        glo, loc = np.round(glo * 8) / 8, np.round(loc * 4) / 4
    c = Config(n_budget=48, l_win=8, tau=0.6, gamma=2.5, kernel_size=5)
    got = oracle.policy_prefill(POLICY[policy], 5, k, v, glo, loc, c)
    want = reflib.policy_prefill(POLICY[policy], 5, k, v, glo, loc, c)
    assert_cache_equal(got, want, rtol=1e-12, atol=1e-12)
