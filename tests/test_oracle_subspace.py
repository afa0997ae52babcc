"""Pins for Algorithm 2, SubspaceSampling."""

import math

import numpy as np

from oracle import philox, srht, subspace


def test_keeps_follow_the_definition():
    # row i kept iff u_i < floor(min(1, r p_i) 2^64), scaled by 1/sqrt(min(1, r p_i));
    # checked against the KAT-pinned pure-Python stream
    n, r, seed = 40, 6, 3
    rng = np.random.default_rng(0)
    p = rng.random(n)
    p[5] = 10.0  # r p_i >= 1: always kept, scale 1
    p /= p.sum()
    Phi = rng.standard_normal((n, 3))
    K, rows = subspace.subspace_sampling(Phi, r, p, seed)
    exp_K, exp_rows = [], []
    for i in range(n):
        q = min(1.0, r * p[i])
        u = philox.stream_word_py(seed, 1, i)
        if q >= 1.0 or u < math.floor(q * 2.0 ** 64):
            exp_K.append(i)
            exp_rows.append(Phi[i] / math.sqrt(q))
    assert K.tolist() == exp_K
    np.testing.assert_allclose(rows, np.array(exp_rows), rtol=0, atol=0)
    assert 5 in exp_K


def test_uniform_probabilities_reduce_to_the_bernoulli_srht():
    # p_i = 1/N on Phi = H_N D [M; 0] / sqrt(N): Algorithm 2 == Algorithm 1 with Bernoulli keeps
    n, r, seed = 100, 20, 9
    M = np.random.default_rng(1).standard_normal((n, 2))
    N = srht.padded_size(n)
    Mp = np.zeros((N, 2))
    Mp[:n] = M
    Phi = srht.hadamard(srht.plan_signs(seed, 0, N)[:, None] * Mp) / math.sqrt(N)
    K, rows = subspace.subspace_sampling(Phi, r, np.full(N, 1.0 / N), seed)
    assert K.tolist() == srht.plan_samples_bernoulli(seed, 0, N, r).tolist()
    np.testing.assert_allclose(rows, srht.sketch(M, seed, r, sampling="bernoulli"), rtol=1e-12, atol=1e-12)


def test_expected_rows_and_norm_estimate():
    # E[#rows] = sum_i min(1, r p_i) <= r, and E ||Phi~ y||^2 = ||Phi y||^2 (Monte Carlo)
    n, r = 64, 10
    rng = np.random.default_rng(2)
    p = rng.random(n) ** 3
    p /= p.sum()
    Phi = rng.standard_normal((n, 2))
    y = np.array([0.3, -1.0])
    counts, est = [], []
    for s in range(500):
        K, rows = subspace.subspace_sampling(Phi, r, p, s)
        counts.append(len(K))
        est.append(float(np.sum((rows @ y) ** 2)) if len(K) else 0.0)
    ev = float(np.sum(np.minimum(1.0, r * p)))
    assert ev <= r + 1e-12
    assert abs(np.mean(counts) - ev) <= 5 * math.sqrt(ev / 500) + 1e-9
    truth = float(np.sum((Phi @ y) ** 2))
    assert abs(np.mean(est) - truth) <= 4 * np.std(est) / math.sqrt(500)
