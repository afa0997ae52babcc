"""Pins for the oracle Hadamard-Walsh transform (Section 2)."""

import numpy as np
import pytest
import scipy.linalg

from oracle import srht
from tests.conftest import golden_path


def _golden_mats():
    mats, cur, name = {}, None, None
    with open(golden_path("hadamard_paper.txt")) as f:
        for line in f:
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            if s[0] == "H":
                name = s
                mats[name] = cur = []
            else:
                cur.append([int(t) for t in s.split()])
    return {k: np.array(v, dtype=np.float64) for k, v in mats.items()}


def test_paper_H2_H4():
    g = _golden_mats()
    assert np.array_equal(srht.hadamard_recursive(np.eye(2)), g["H2"])
    assert np.array_equal(srht.hadamard(np.eye(4)), g["H4"])
    # H is symmetric so H @ I_N = H whichever side the identity sits.


@pytest.mark.parametrize("N", [2, 4, 8, 16, 64, 256, 1024])
def test_matches_scipy_sylvester(N):
    # scipy.linalg.hadamard builds the Sylvester (natural order) matrix (R3).
    assert np.array_equal(srht.hadamard(np.eye(N)), scipy.linalg.hadamard(N).astype(np.float64))


@pytest.mark.parametrize("N", [2, 8, 32, 64])
def test_closed_form_popcount(N):
    H = srht.hadamard(np.eye(N))
    for k in range(N):
        for i in range(N):
            assert H[k, i] == (-1.0) ** bin(k & i).count("1")


def test_unrolled_equals_literal_recursion_bitwise():
    rng = np.random.default_rng(1)
    for N in [1, 2, 4, 32, 128, 512]:
        x = rng.standard_normal((N, 3))
        assert np.array_equal(srht.hadamard(x), srht.hadamard_recursive(x))


@pytest.mark.parametrize("N", [2, 16, 512, 4096])
def test_HH_is_NI_and_norm_preserving(N):
    H = srht.hadamard(np.eye(N))
    assert np.array_equal(H @ H, N * np.eye(N))
    x = np.random.default_rng(N).standard_normal(N)
    y = srht.hadamard(x) / np.sqrt(N)
    assert abs(np.linalg.norm(y) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    # involution of the normalized transform
    assert np.allclose(srht.hadamard(y) / np.sqrt(N), x, atol=1e-12, rtol=0)


def test_spec_examples():
    # normalized FWHT of (1, 0) is (1/sqrt2, 1/sqrt2)
    y = srht.hadamard(np.array([1.0, 0.0])) / np.sqrt(2.0)
    assert np.allclose(y, [2 ** -0.5, 2 ** -0.5], rtol=0, atol=1e-15)


def test_rejects_non_power_of_two():
    with pytest.raises(ValueError):
        srht.hadamard(np.ones(6))
