"""Gram form of the sketched NNLS problem, float64 (TEST INFRASTRUCTURE ONLY).

Section 3.4: min_{x >= 0} ||A x - b||^2 is the quadratic program
min x^T Q x - 2 q^T x (+ b^T b) with Q = A^T A and q = A^T b; for the sketched
problem Q~ = (H~DA)^T H~DA and q~ = (H~DA)^T (H~Db) (reading R17: the paper's
(H~DA)^T b has mismatched dimensions; the sketched b is meant).  With the sketch
SM = [SA | Sb] in one matrix, G = SM^T SM = [[Q~, q~], [q~^T, Sb^T Sb]].
"""

import numpy as np


def gram(SM):
    """G = SM^T SM (float64), the definition (a library matrix product)."""
    SM = np.asarray(SM, dtype=np.float64)
    return SM.T @ SM


def split(G):
    """(Q~, q~, Sb^T Sb) from G = gram([SA | Sb])."""
    G = np.asarray(G, dtype=np.float64)
    return G[:-1, :-1], G[:-1, -1], G[-1, -1]


def qp_objective(G, x):
    """x^T Q~ x - 2 q~^T x + Sb^T Sb, which equals ||SA x - Sb||^2."""
    Q, q, bb = split(G)
    x = np.asarray(x, dtype=np.float64)
    return float(x @ Q @ x - 2.0 * q @ x + bb)
