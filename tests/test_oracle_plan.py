"""Pins for the oracle plan: padding, D (step 4) and S / H~ (steps 2-3)."""

import heapq
import math

import numpy as np
import pytest

from oracle import philox, srht


@pytest.mark.parametrize("n,N", [(1, 2), (2, 2), (3, 4), (5, 8), (4096, 4096), (4097, 8192),
                                 (10000, 16384), (2 ** 26, 2 ** 26)])
def test_padded_size(n, N):
    assert srht.padded_size(n) == N


def test_signs_bit_mapping_from_definition():
    # R5: D_ii = -1 iff bit (i mod 64) of word i//64 of stream (seed, 2p) is 1,
    # checked against the pure-Python (KAT-pinned) Philox, not the numpy path.
    for seed, p, N in [(0, 0, 128), (7, 3, 256)]:
        sig = srht.plan_signs(seed, p, N)
        for i in range(N):
            w = philox.stream_word_py(seed, 2 * p, i // 64)
            assert sig[i] == (-1.0 if (w >> (i % 64)) & 1 else 1.0)


def test_signs_balanced():
    N = 1 << 20
    s = srht.plan_signs(0, 0, N)
    assert set(np.unique(s)) == {-1.0, 1.0}
    assert abs(s.mean()) < 5.0 / math.sqrt(N)


def test_samples_bruteforce_selection():
    # R1/R6: the r indices with smallest (u_i, i), sorted; brute force via heapq
    # on the pure-Python stream.
    for seed, p, N, r in [(0, 0, 64, 8), (5, 2, 128, 100), (1, 0, 32, 32), (9, 1, 16, 1)]:
        K = srht.plan_samples(seed, p, N, r)
        keys = [(philox.stream_word_py(seed, 2 * p + 1, i), i) for i in range(N)]
        expect = sorted(i for _, i in heapq.nsmallest(r, keys))
        assert K.tolist() == expect


def test_samples_structure():
    N, r = 1 << 16, 1000
    K = srht.plan_samples(3, 0, N, r)
    assert K.shape == (r,)
    assert np.all(np.diff(K) > 0)
    assert K[0] >= 0 and K[-1] < N
    with pytest.raises(ValueError):
        srht.plan_samples(0, 0, 16, 17)
    with pytest.raises(ValueError):
        srht.plan_samples(0, 0, 16, 0)


def test_inclusion_frequency_is_r_over_N():
    # Algorithm 1 step 2 keeps each row with probability r/n.
    N, r, seeds = 64, 16, 400
    counts = np.zeros(N)
    for s in range(seeds):
        counts[srht.plan_samples(s, 0, N, r)] += 1
    p = r / N
    freq = counts / seeds
    sd = math.sqrt(p * (1 - p) / seeds)
    assert np.all(np.abs(freq - p) < 5 * sd)
    assert abs(freq.mean() - p) < 1e-12  # exactly r per draw


def test_problems_have_independent_plans():
    a = srht.plan_samples(0, 0, 1024, 64)
    b = srht.plan_samples(0, 1, 1024, 64)
    assert not np.array_equal(a, b)


# ---- Bernoulli keeps (Algorithm 1 step 2 verbatim) ----

def test_bernoulli_threshold_exact():
    # T = floor(2^64 r / N) as an exact integer: for N = 2^L it is r * 2^(64 - L)
    for L, r in [(4, 1), (10, 37), (20, 8192), (26, 16384)]:
        N = 1 << L
        assert srht.bernoulli_threshold(N, r) == r * (1 << (64 - L))
    assert srht.bernoulli_threshold(8, 8) == 1 << 64  # r = N keeps everything


def test_bernoulli_keeps_are_the_threshold_set():
    # brute force from the raw stream words: kept iff u_i < T, ascending
    for seed, N, r in [(1, 64, 9), (2, 256, 100), (3, 16, 16)]:
        u = [philox.stream_word_py(seed, 1, i) for i in range(N)]  # KAT-pinned pure-Python Philox
        T = (r << 64) // N
        expect = [i for i in range(N) if u[i] < T]
        assert list(srht.plan_samples_bernoulli(seed, 0, N, r)) == expect


def test_bernoulli_inclusion_frequency_and_count():
    # each row kept w.p. r/N: per-index frequency and mean count over seeds (5 sigma)
    N, r, seeds = 256, 32, 400
    hits = np.zeros(N)
    counts = []
    for s in range(seeds):
        K = srht.plan_samples_bernoulli(s, 0, N, r)
        hits[K] += 1
        counts.append(len(K))
    pr = r / N
    sd = math.sqrt(pr * (1 - pr) / seeds)
    assert np.all(np.abs(hits / seeds - pr) <= 5 * sd + 1e-12)
    sd_mean = math.sqrt(N * pr * (1 - pr) / seeds)
    assert abs(np.mean(counts) - r) <= 5 * sd_mean


def test_bernoulli_sketch_is_unbiased_in_norm():
    # E ||S H D x||^2 = ||x||^2 with the sqrt(N/r) scale of P:298 (Monte Carlo, 4 sigma)
    n, r = 64, 16
    x = np.random.default_rng(0).standard_normal(n)
    vals = [float(np.sum(srht.sketch(x, s, r, sampling="bernoulli") ** 2)) for s in range(600)]
    m, sd = np.mean(vals), np.std(vals) / math.sqrt(len(vals))
    assert abs(m - float(x @ x)) <= 4 * sd
