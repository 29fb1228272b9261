"""Pins the oracle's diagnostics (ems_oracle_sparsity_rate / ems_oracle_redundancy_rate_direct,
restating proj/src/analysis.cpp:71-118) before the GPU kernels are compared to them:

1. acceptance criterion 11 (proj/tests/acceptance.cpp:574-650): a brute-force sparsity oracle
   over zeta = 0.1 .. 1.0, monotonicity in zeta, and the redundancy rate from the full matrix
   (redundancy_matrix + redundancy_rate, analysis.cpp:28-49, 120-136) equal to the direct form;
2. the reference itself (oracle/_ref) on seeded inputs, random and redundant;
3. the argument checks (zeta outside (0, 1], no mass).
"""
import numpy as np
import pytest

from oracle.oracle import DegenerateInput, InvalidArgument


def brute_sparsity(score, zeta):
    s = np.sort(score)[::-1]
    total = float(np.sum(score))
    cum = 0.0
    for i, x in enumerate(s):
        cum += x / total
        if cum >= zeta:
            return 1.0 - (i + 1) / len(s)
    return 0.0


def brute_redundancy(k, v, tau):
    def cz(a, b):
        na, nb = np.linalg.norm(a), np.linalg.norm(b)
        return 0.0 if na == 0 or nb == 0 else float(np.clip(a @ b / (na * nb), -1, 1))
    n = len(k)
    red = 0
    for t in range(1, n):
        best = max(cz(k[t], k[j]) * cz(v[t], v[j]) for j in range(t))
        red += best >= tau
    return red / n


def test_c11_sparsity_brute_force_and_monotone(oracle):
    rng = np.random.default_rng(23000)
    for _ in range(10):
        score = rng.uniform(0, 1, 32) + 1e-6
        prev = 1.0
        for zi in range(1, 11):
            p = oracle.sparsity_rate(score, 0.1 * zi)
            assert abs(p - brute_sparsity(score, 0.1 * zi)) == 0.0
            assert p <= prev + 1e-15
            prev = p


def test_c11_redundancy_direct_vs_matrix(oracle):
    rng = np.random.default_rng(23001)
    for _ in range(10):
        k, v = rng.standard_normal((32, 8)), rng.standard_normal((32, 8))
        k[5] = 0.0  # a zero-norm token: similarity 0 to everything
        for tau in (0.0, 0.1, 0.3, 0.6):
            assert oracle.redundancy_rate_direct(k, v, tau) == brute_redundancy(k, v, tau)


@pytest.mark.parametrize("n,seed", [(1, 0), (7, 1), (300, 2), (4096, 3)])
def test_sparsity_matches_reference(oracle, reflib, n, seed):
    rng = np.random.default_rng(seed)
    score = rng.exponential(1.0, n) ** 3
    score[rng.integers(0, n, n // 5)] = 0.0
    for zeta in (0.05, 0.5, 0.95, 1.0):
        assert oracle.sparsity_rate(score, zeta) == reflib.sparsity_rate(score, zeta)
    q = np.round(score * 4) / 4  # many exact ties
    if q.sum() > 0:
        assert oracle.sparsity_rate(q, 0.9) == reflib.sparsity_rate(q, 0.9)


@pytest.mark.parametrize("kind", [0, 1])
def test_redundancy_matches_reference(oracle, reflib, kind):
    q, k, v = reflib.gen_trace(kind, 4242 + kind, 256, 2, 16, 1, level=0.8)
    for h in range(2):
        for tau in (0.3, 0.6, 0.9):
            assert oracle.redundancy_rate_direct(k[h, :256], v[h, :256], tau) == \
                reflib.redundancy_rate_direct(k[h, :256], v[h, :256], tau)


def test_diagnostics_argument_checks(oracle, reflib):
    for lib in (oracle, reflib):
        with pytest.raises(InvalidArgument):
            lib.sparsity_rate(np.ones(4), 0.0)
        with pytest.raises(InvalidArgument):
            lib.sparsity_rate(np.ones(4), 1.5)
        with pytest.raises(DegenerateInput):
            lib.sparsity_rate(np.zeros(4), 0.5)
