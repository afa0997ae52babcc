"""Pins for the oracle Gram / QP form (Section 3.4)."""

import numpy as np

from oracle import gram


def test_gram_entries_are_dot_products():
    rng = np.random.default_rng(1)
    SM = rng.standard_normal((7, 4))
    G = gram.gram(SM)
    for i in range(4):
        for j in range(4):
            acc = 0.0
            for k in range(7):
                acc += SM[k, i] * SM[k, j]
            assert abs(G[i, j] - acc) <= 1e-13 * (1 + abs(acc))


def test_qp_objective_is_the_residual():
    # x^T Q~ x - 2 q~^T x + Sb^T Sb = ||SA x - Sb||^2 for any x (the QP form of P:570-578)
    rng = np.random.default_rng(2)
    SA, Sb = rng.standard_normal((30, 5)), rng.standard_normal(30)
    G = gram.gram(np.column_stack([SA, Sb]))
    for _ in range(5):
        x = rng.random(5)
        assert abs(gram.qp_objective(G, x) - np.sum((SA @ x - Sb) ** 2)) <= 1e-10 * np.sum(Sb ** 2)


def test_gram_symmetric_psd_and_split():
    rng = np.random.default_rng(3)
    SM = rng.standard_normal((50, 6))
    G = gram.gram(SM)
    assert np.array_equal(G, G.T)
    assert np.min(np.linalg.eigvalsh(G)) >= -1e-10
    Q, q, bb = gram.split(G)
    assert Q.shape == (5, 5) and q.shape == (5,)
    assert abs(bb - np.sum(SM[:, -1] ** 2)) <= 1e-12 * bb
