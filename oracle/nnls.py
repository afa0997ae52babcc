"""NNLS solvers and metrics, float64 (TEST INFRASTRUCTURE ONLY).

* Definition 1: x_opt = argmin_{x >= 0} ||A x - b||_2^2.
* Lawson-Hanson active set (the paper's ``lsqnonneg``), with the
  tie-breaks and tolerances of reading R13.
* Brute-force support enumeration: the NNLS optimum is the least-squares
  solution on its own support, so the best feasible LS solution over all 2^d
  supports is the optimum (used to pin Lawson-Hanson, d <= 10).
* Fig. 1 relative error: ||A x~ - b|| / ||A x_opt - b|| (reading R12).
* Algorithm 1 end to end with the oracle sketch.
"""

import itertools

import numpy as np

from .srht import sketch_problem


def _ls(A, b):
    return np.linalg.lstsq(A, b, rcond=None)[0]


def lawson_hanson(A, b, tol=None, max_iter=None):
    """Lawson & Hanson (1974) NNLS active-set algorithm; returns (x, outer_iters).

    P = passive set, Z = active set (x_j = 0).  Outer loop: w = A^T (b - A x);
    stop when max_{j in Z} w_j <= tol; else move argmax_{j in Z} w_j (smallest
    index on ties) into P.  Inner loop: z = LS solution on P; if some z_j <= 0,
    step back x <- x + alpha (z - x) with alpha = min x_j / (x_j - z_j) over those
    j (smallest index on ties) and move every j in P with x_j <= 0 back to Z.
    """
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    n, d = A.shape
    if tol is None:
        tol = 1e-10 * max(np.max(np.abs(A.T @ b)), np.finfo(float).tiny)
    if max_iter is None:
        max_iter = 30 * max(d, 1)
    x = np.zeros(d)
    passive = np.zeros(d, dtype=bool)
    skipped = np.zeros(d, dtype=bool)   # entered with a non-positive LS value
    it = 0
    while True:
        w = A.T @ (b - A @ x)
        cand = (~passive) & (~skipped)
        if not cand.any() or np.max(np.where(cand, w, -np.inf)) <= tol:
            break
        it += 1
        if it > max_iter:
            raise RuntimeError("Lawson-Hanson: max_iter exceeded")
        wc = np.where(cand, w, -np.inf)
        t = int(np.flatnonzero(wc == wc.max())[0])
        passive[t] = True
        inner_guard = 0
        while True:
            inner_guard += 1
            if inner_guard > 10 * d + 10:
                raise RuntimeError("Lawson-Hanson: inner loop did not terminate")
            idx = np.flatnonzero(passive)
            z = np.zeros(d)
            z[idx] = _ls(A[:, idx], b)
            if np.all(z[idx] > 0):
                x = z
                skipped[:] = False
                break
            if inner_guard == 1 and z[t] <= 0:
                # Degenerate entry (w_t > tol only by rounding): t cannot move
                # off zero; leave x unchanged and do not offer t again until
                # x changes.
                passive[t] = False
                skipped[t] = True
                break
            neg = idx[z[idx] <= 0]
            ratios = x[neg] / (x[neg] - z[neg])
            alpha = ratios.min()
            x = x + alpha * (z - x)
            drop = passive & (x <= 0)
            # the ratio-minimizing index (smallest on ties) always leaves
            drop[int(neg[np.flatnonzero(ratios == alpha)[0]])] = True
            x[drop] = 0.0
            passive &= ~drop
            if not passive.any():
                break
    x[x < 1e-14] = 0.0
    return x, it


def nnls_bruteforce(A, b):
    """Exact NNLS by enumerating all 2^d supports (d <= 10)."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    d = A.shape[1]
    if d > 12:
        raise ValueError("brute force limited to d <= 12")
    best_x = np.zeros(d)
    best = float(b @ b)
    for k in range(1, d + 1):
        for S in itertools.combinations(range(d), k):
            S = list(S)
            xs = _ls(A[:, S], b)
            if np.all(xs >= 0):
                x = np.zeros(d)
                x[S] = xs
                f = float(np.sum((A @ x - b) ** 2))
                if f < best:
                    best, best_x = f, x
    return best_x


def kkt_violation(A, b, x):
    """Max violation of the NNLS KKT system for g = 2 A^T (A x - b).

    Optimality of the convex QP: x >= 0, g >= 0, x_j g_j = 0.
    Returned relative to ||2 A^T b||_inf.
    """
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    g = 2.0 * A.T @ (A @ x - b)
    scale = max(np.max(np.abs(2.0 * A.T @ b)), np.finfo(float).tiny)
    prim = max(0.0, -float(np.min(x)))
    dual = max(0.0, -float(np.min(g)))
    comp = float(np.max(np.abs(x * g))) / max(1.0, float(np.max(np.abs(x))))
    return max(prim, dual / scale, comp / scale)


def residual_norm(A, x, b):
    """R(x) = ||A x - b||_2, evaluated on the given (original) data."""
    A = np.asarray(A, dtype=np.float64)
    return float(np.linalg.norm(A @ np.asarray(x, dtype=np.float64) - np.asarray(b, dtype=np.float64).reshape(-1)))


def relative_error(A, b, x_tilde, x_opt):
    """Fig. 1 'Relative Error' := ||A x~ - b|| / ||A x_opt - b||."""
    return residual_norm(A, x_tilde, b) / residual_norm(A, x_opt, b)


def solve_sketched(SA, Sb):
    """Algorithm 1 step 5: Lawson-Hanson on the sketched problem."""
    return lawson_hanson(SA, Sb)[0]


def randomized_nnls(A, b, r, seed, p=0):
    """Algorithm 1 end to end with the oracle sketch; returns x~_opt."""
    SA, Sb = sketch_problem(A, b, seed, r, p=p)
    return solve_sketched(SA, Sb)
