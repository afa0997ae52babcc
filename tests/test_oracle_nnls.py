"""Pins for the oracle NNLS (Definition 1, Lawson-Hanson) and Algorithm 1 end to end."""

import numpy as np
import pytest
import scipy.optimize

from oracle import nnls, srht
from tests.conftest import golden_path


def _examples():
    out = []
    with open(golden_path("nnls_examples.txt")) as f:
        for line in f:
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            name, A, b, x, r2 = [t.strip() for t in s.split("|")]
            A = np.array([[float(v) for v in row.split()] for row in A.split(";")])
            out.append((name, A, np.array([float(v) for v in b.split()]),
                        np.array([float(v) for v in x.split()]), float(r2)))
    return out


@pytest.mark.parametrize("ex", _examples(), ids=lambda e: e[0])
def test_golden_examples(ex):
    _, A, b, x_opt, r2 = ex
    x, _ = nnls.lawson_hanson(A, b)
    assert np.allclose(x, x_opt, rtol=0, atol=1e-12)
    assert abs(nnls.residual_norm(A, x, b) ** 2 - r2) < 1e-12


@pytest.mark.parametrize("seed", range(40))
def test_lawson_hanson_vs_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n, d = int(rng.integers(6, 30)), int(rng.integers(1, 7))
    A = rng.standard_normal((n, d))
    b = rng.standard_normal(n)
    x, _ = nnls.lawson_hanson(A, b)
    xb = nnls.nnls_bruteforce(A, b)
    f, fb = np.sum((A @ x - b) ** 2), np.sum((A @ xb - b) ** 2)
    assert np.all(x >= 0)
    assert abs(f - fb) <= 1e-10 * max(1.0, fb)
    assert np.allclose(x, xb, atol=1e-8)


@pytest.mark.parametrize("seed", range(10))
def test_lawson_hanson_vs_scipy(seed):
    rng = np.random.default_rng(100 + seed)
    A = rng.random((200, 40))
    b = rng.random(200) * 5 - 1
    x, _ = nnls.lawson_hanson(A, b)
    xs, rs = scipy.optimize.nnls(A, b)
    assert abs(nnls.residual_norm(A, x, b) - rs) <= 1e-10 * max(1.0, rs)
    assert nnls.kkt_violation(A, b, x) < 1e-9


def test_consistent_b_recovers_x():
    rng = np.random.default_rng(7)
    A = rng.random((100, 8))
    xs = rng.random(8)
    xs[[1, 4]] = 0.0
    x, _ = nnls.lawson_hanson(A, A @ xs)
    assert np.allclose(x, xs, atol=1e-10)


def test_scaling_covariance():
    rng = np.random.default_rng(8)
    A, b = rng.standard_normal((40, 5)), rng.standard_normal(40)
    x1, _ = nnls.lawson_hanson(A, b)
    x2, _ = nnls.lawson_hanson(3.0 * A, 3.0 * b)
    assert np.allclose(x1, x2, atol=1e-10)


def test_kkt_detects_perturbation():
    rng = np.random.default_rng(9)
    A, b = rng.standard_normal((30, 4)), rng.standard_normal(30)
    x, _ = nnls.lawson_hanson(A, b)
    assert nnls.kkt_violation(A, b, x) < 1e-10
    bad = x.copy()
    bad[0] += 0.1
    assert nnls.kkt_violation(A, b, bad) > 1e-4


def test_full_sample_relative_error_is_one():
    # r = N: the sketch is an orthonormal map, the sketched problem has the same
    # objective, so x~ = x_opt and Fig. 1's relative error is 1.
    rng = np.random.default_rng(10)
    n, d = 60, 4
    A = rng.random((n, d))
    b = A @ np.array([0.5, 0.0, 0.3, 0.0]) + 0.1 * rng.standard_normal(n)
    x_opt, _ = nnls.lawson_hanson(A, b)
    xt = nnls.randomized_nnls(A, b, srht.padded_size(n), seed=3)
    assert abs(nnls.relative_error(A, b, xt, x_opt) - 1.0) < 1e-12


def test_relative_error_at_least_one():
    rng = np.random.default_rng(11)
    A = rng.random((128, 5))
    b = rng.random(128)
    x_opt = nnls.nnls_bruteforce(A, b)
    for seed in range(20):
        xt = nnls.randomized_nnls(A, b, 16, seed)
        assert nnls.relative_error(A, b, xt, x_opt) >= 1.0 - 1e-12


def test_theorem1_success_fraction_grows_with_r():
    # Reading R15: c_o is unspecified, so the bound itself is not
    # computable; check the fraction of seeds with relerr^2 <= 1 + eps is
    # non-decreasing in r (one inversion tolerated) and >= 0.5 at r >= N/2.
    rng = np.random.default_rng(12)
    n, d, eps = 64, 3, 0.5
    A = rng.random((n, d))
    b = A @ np.array([0.7, 0.0, 0.4]) + 0.3 * rng.standard_normal(n)
    x_opt = nnls.nnls_bruteforce(A, b)
    fr = []
    for r in [4, 8, 16, 32, 64]:
        ok = 0
        for seed in range(120):
            SA, Sb = srht.sketch_problem(A, b, seed, r)
            xt = nnls.nnls_bruteforce(SA, Sb)
            ok += nnls.relative_error(A, b, xt, x_opt) ** 2 <= 1 + eps
        fr.append(ok / 120)
    inversions = sum(1 for a, c in zip(fr, fr[1:]) if c < a)
    assert inversions <= 1, fr
    assert fr[3] >= 0.5 and fr[4] == 1.0, fr
