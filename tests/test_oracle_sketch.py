"""Pins for the oracle sketch H~ D M (Algorithm 1)."""

import math

import numpy as np
import pytest

from oracle import srht


def test_single_nonzero_closed_form():
    # M = e_i: SM[t] = sigma_i (-1)^popc(k_t & i) / sqrt(r)  (the N-dependence cancels).
    n, r, seed = 100, 16, 4
    N = srht.padded_size(n)
    sig = srht.plan_signs(seed, 0, N)
    K = srht.plan_samples(seed, 0, N, r)
    for i in [0, 1, 37, 99]:
        e = np.zeros(n)
        e[i] = 1.0
        SM = srht.sketch(e, seed, r)[:, 0]
        expect = np.array([sig[i] * (-1.0) ** bin(int(k) & i).count("1") for k in K]) / math.sqrt(r)
        assert np.allclose(SM, expect, rtol=0, atol=1e-15)


def test_matches_bruteforce_entries():
    rng = np.random.default_rng(0)
    n, r, seed = 37, 9, 11
    col = rng.standard_normal(n)
    SM = srht.sketch(col, seed, r)[:, 0]
    for t in range(r):
        assert abs(SM[t] - srht.sketch_entry_bruteforce(col, seed, r, t)) <= 1e-12 * np.abs(col).sum()


def test_full_sampling_is_orthonormal():
    # r = N: S H_N D is orthonormal, so (SM)^T (SM) = M^T M.
    rng = np.random.default_rng(2)
    n = 50
    N = srht.padded_size(n)
    M = rng.standard_normal((n, 4))
    SM = srht.sketch(M, 5, N)
    assert np.allclose(SM.T @ SM, M.T @ M, rtol=0, atol=1e-11)


def test_expected_norm_preserved_monte_carlo():
    # E ||S H D x||^2 = ||x||^2 : each index kept w.p. r/N with scale^2 N/r.
    rng = np.random.default_rng(3)
    n, r = 64, 8
    x = rng.standard_normal(n)
    vals = np.array([np.sum(srht.sketch(x, s, r) ** 2) for s in range(600)])
    mean, sd = vals.mean(), vals.std(ddof=1) / math.sqrt(len(vals))
    assert abs(mean - x @ x) < 4 * sd


def test_shared_plan_for_b():
    # R7: b uses the same D and S as A.
    rng = np.random.default_rng(4)
    A = rng.random((30, 3))
    b = rng.random(30)
    SA, Sb = srht.sketch_problem(A, b, 9, 8)
    for j in range(3):
        assert np.array_equal(SA[:, j], srht.sketch(A[:, j], 9, 8)[:, 0])
    assert np.array_equal(Sb, srht.sketch(b, 9, 8)[:, 0])


def test_padding_rows_contribute_nothing():
    rng = np.random.default_rng(5)
    M = rng.standard_normal((5, 2))
    Mz = np.vstack([M, np.zeros((3, 2))])  # explicit padding to N = 8
    assert np.array_equal(srht.sketch(M, 1, 4), srht.sketch(Mz, 1, 4))


def test_linearity():
    rng = np.random.default_rng(6)
    x, y = rng.standard_normal(40), rng.standard_normal(40)
    lhs = srht.sketch(2.0 * x - 3.0 * y, 2, 16)
    rhs = 2.0 * srht.sketch(x, 2, 16) - 3.0 * srht.sketch(y, 2, 16)
    assert np.allclose(lhs, rhs, rtol=0, atol=1e-12)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_tiny_n(n):
    SM = srht.sketch(np.ones(n), 0, 2)
    assert SM.shape == (2, 1)


def test_rows_partial_matches_closed_form():
    # Row-shard partial against the closed form of the definition,
    # entry by entry with explicit loops: P[t, j] = sum_{i in rows} (-1)^popc(k_t & i) sigma_i M[i, j].
    n, r, seed, c = 23, 5, 3, 2
    N = srht.padded_size(n)
    rng = np.random.default_rng(11)
    M = rng.standard_normal((n, c))
    sigma = srht.plan_signs(seed, 0, N)
    K = srht.plan_samples(seed, 0, N, r)
    for row0, row1 in [(0, 8), (8, 23), (5, 6), (0, 23)]:
        got = srht.sketch_rows_partial(M[row0:row1], row0, n, seed, r)
        ref = np.zeros((r, c))
        for t in range(r):
            for i in range(row0, row1):
                sgn = (-1.0) ** bin(int(K[t]) & i).count("1") * sigma[i]
                ref[t] += sgn * M[i]
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_rows_partials_of_a_partition_sum_to_the_sketch():
    # linearity across a row partition, scaled by r^{-1/2} (the all-reduce of row sharding)
    n, r, seed = 300, 40, 7
    M = np.random.default_rng(5).standard_normal((n, 3))
    cuts = [0, 64, 128, 200, 300]
    tot = sum(srht.sketch_rows_partial(M[a:b], a, n, seed, r) for a, b in zip(cuts, cuts[1:]))
    np.testing.assert_allclose(tot / math.sqrt(r), srht.sketch(M, seed, r), rtol=1e-12, atol=1e-12)
