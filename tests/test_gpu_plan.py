"""GPU plan vs oracle: D and the kept rows must be bit-exact (north_star)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srht():
    import paper_0812_4547_b200 as m
    return m


@pytest.mark.parametrize("n,r,seed", [(1, 1, 0), (2, 2, 3), (5, 3, 1), (1000, 100, 7), (4096, 256, 0),
                                      (10000, 350, 2), (8192, 1024, 0), (1 << 17, 4096, 0), (1 << 20, 8192, 0),
                                      (40000, 40000, 5)])
def test_plan_bit_exact(srht, n, r, seed):
    from oracle import srht as osr
    N = osr.padded_size(n)
    plan = srht.Plan(n, 3, r, seed)
    assert plan.N == N
    assert np.array_equal(plan.indices(0).astype(np.int64), osr.plan_samples(seed, 0, N, r))
    assert np.array_equal(plan.sign_words(0), osr.sign_words(seed, 0, N))


def test_plan_bit_exact_config5(srht):
    from oracle import srht as osr
    n, r = 1 << 26, 16384
    plan = srht.Plan(n, 127, r, 0)
    assert np.array_equal(plan.indices(0).astype(np.int64), osr.plan_samples(0, 0, n, r))
    assert np.array_equal(plan.sign_words(0), osr.sign_words(0, 0, n))


def test_batched_plans_bit_exact(srht):
    from oracle import srht as osr
    batch, n, r = 3000, 8192, 1024
    plan = srht.Plan(n, 100, r, 0, batch=batch)
    for p in list(range(0, batch, 97)) + [batch - 1]:
        assert np.array_equal(plan.indices(p).astype(np.int64), osr.plan_samples(0, p, n, r)), p
        assert np.array_equal(plan.sign_words(p), osr.sign_words(0, p, n)), p


def test_invalid_arguments(srht):
    from paper_0812_4547_b200._lib import SRHT_EINVAL
    for args in [(0, 1, 1), (4, 1, 5), (4, 1, 0), (-3, 1, 1)]:
        with pytest.raises(srht.SrhtError) as ei:
            srht.Plan(*args)
        assert ei.value.status == SRHT_EINVAL


# ---- Bernoulli keeps (Algorithm 1 step 2 verbatim) ----

@pytest.mark.parametrize("n,r,seed", [(4096, 256, 0), (100000, 3000, 5), (1 << 20, 8192, 9), (1 << 14, 1 << 14, 2), (37, 5, 3)])
def test_bernoulli_plan_bit_exact(srht, n, r, seed):
    from oracle import srht as osr
    plan = srht.Plan(n, 3, r, seed, sampling="bernoulli")
    N = osr.padded_size(n)
    K = osr.plan_samples_bernoulli(seed, 0, N, r)
    assert plan.r == len(K) and plan.r_target == r
    assert np.array_equal(plan.indices().astype(np.int64), K)
    assert np.array_equal(plan.sign_words(), osr.sign_words(seed, 0, N))
