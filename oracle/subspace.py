"""Algorithm 2, SubspaceSampling, float64 (TEST INFRASTRUCTURE ONLY).

Input Phi (n x d), integer r, probabilities p_i >= 0 summing to 1.  S is diagonal with
S_ii = 1/sqrt(min(1, r p_i)) with probability min(1, r p_i) and 0 otherwise; the output
is the non-zero rows of S Phi (E[#rows] <= r).

Reading (R18): the coin of row i is word i of the Philox stream (seed, 1)
(reading R4), u_i < floor(min(1, r p_i) 2^64) keeps the row (probability min(1, r p_i)
up to 2^-64; always when min(1, r p_i) = 1).  With p_i = 1/N and Phi = H_N D [M; 0] /
sqrt(N) this is exactly the Bernoulli SRHT sketch (srht.sketch(..., sampling="bernoulli")).
"""

import math

import numpy as np

from .philox import stream_words


def keep_thresholds(r, p):
    """T_i = floor(min(1, r p_i) 2^64) as Python ints (None = always kept)."""
    out = []
    for pi in np.asarray(p, dtype=np.float64):
        q = min(1.0, float(r) * float(pi))
        out.append(None if q >= 1.0 else int(math.floor(q * 2.0 ** 64)))
    return out


def subspace_sampling(Phi, r, p, seed):
    """(K, Phi~): kept row indices (ascending) and the non-zero rows of S Phi."""
    Phi = np.asarray(Phi, dtype=np.float64)
    if Phi.ndim == 1:
        Phi = Phi[:, None]
    n = Phi.shape[0]
    u = stream_words(seed, 1, n)
    K, rows = [], []
    for i, T in enumerate(keep_thresholds(r, p)):
        if T is None or int(u[i]) < T:
            q = min(1.0, float(r) * float(p[i]))
            K.append(i)
            rows.append(Phi[i] / math.sqrt(q))
    return np.array(K, dtype=np.int64), (np.array(rows) if rows else np.zeros((0, Phi.shape[1])))
