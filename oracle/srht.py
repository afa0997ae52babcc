"""SRHT sketch H~ D [A | b], float64, straight from PAPER.md (TEST INFRASTRUCTURE ONLY).

Notation follows the paper.  n rows, d columns of A, b the target; N = padded n.

* Hadamard-Walsh matrix (Section 2): H_n = [[H_{n/2}, H_{n/2}],
  [H_{n/2}, -H_{n/2}]] with H_2 = [[+1, +1], [+1, -1]]; the normalized matrix is
  H_n / sqrt(n); A and b are padded with all-zero rows to a power of two.
* Algorithm 1: S_ii = sqrt(n/r) with probability r/n (step 2),
  H~ = the non-zero rows of S H_n (step 3), D_ii = +-1 with probability 1/2
  (step 4), and step 5 solves the NNLS problem on (H~ D A, H~ D b).
* Proof of Theorem 1: Phi = [H_n D A, -H_n D b] -- the SAME D and S
  act on every column of A and on b (reading R7).

Readings: R1 exactly r distinct rows (uniform r-subset), R2 the
padded N is the n of sqrt(n/r), R3 natural (Sylvester) order, R4 Philox streams,
R5 sign-bit mapping, R6 sample keys and tie-break.
"""

import math

import numpy as np

from .philox import stream_words


def padded_size(n):
    """N = smallest power of two >= n, and >= 2 (reading R9)."""
    n = int(n)
    if n < 1:
        raise ValueError("n must be >= 1")
    N = 2
    while N < n:
        N *= 2
    return N


# ----------------------------------------------------------------------------
# Randomness of Algorithm 1 (steps 2 and 4).
# ----------------------------------------------------------------------------

def sign_words(seed, p, N):
    """The 64-bit words carrying D for problem p: stream (seed, 2p + 0) (R4, R5)."""
    return stream_words(seed, 2 * p + 0, (N + 63) // 64)


def plan_signs(seed, p, N):
    """Diagonal of D (Algorithm 1 step 4) as +-1 floats, length N.

    Reading R5: D_ii = -1 iff bit (i mod 64) of word floor(i / 64) is 1.
    """
    words = sign_words(seed, p, N)
    i = np.arange(N, dtype=np.uint64)
    bits = (words[i // np.uint64(64)] >> (i % np.uint64(64))) & np.uint64(1)
    return 1.0 - 2.0 * bits.astype(np.float64)


def plan_samples(seed, p, N, r):
    """Kept rows of S H_n (Algorithm 1 steps 2-3), sorted ascending.

    Reading R1/R6: exactly r rows -- the r indices i with the smallest
    (u_i, i), u_i = word i of stream (seed, 2p + 1).  This is the Bernoulli(r/N)
    selection of step 2 conditioned on keeping exactly r rows.
    """
    if not (1 <= r <= N):
        raise ValueError("need 1 <= r <= N")
    u = stream_words(seed, 2 * p + 1, N)
    order = np.argsort(u, kind="stable")  # stable: equal keys keep index order
    return np.sort(order[:r]).astype(np.int64)


def bernoulli_threshold(N, r):
    """Keep threshold for Algorithm 1 step 2 read verbatim:
    row i is kept iff u_i < T with T = floor(2^64 r / N), i.e. with probability r/N for a
    uniform 64-bit u_i (exactly r/N when N is a power of two)."""
    return (int(r) << 64) // int(N)


def plan_samples_bernoulli(seed, p, N, r):
    """Kept rows under independent Bernoulli(r/N) keeps (Algorithm 1 step 2 as written):
    {i < N : u_i < T}, ascending; the count is random with mean r (reading R1, variant)."""
    if not (1 <= r <= N):
        raise ValueError("need 1 <= r <= N")
    u = stream_words(seed, 2 * p + 1, N)
    T = bernoulli_threshold(N, r)
    if T >= 1 << 64:
        return np.arange(N, dtype=np.int64)
    return np.flatnonzero(u < np.uint64(T)).astype(np.int64)


# ----------------------------------------------------------------------------
# Hadamard-Walsh transform (Section 2).
# ----------------------------------------------------------------------------

def hadamard_recursive(x):
    """Unnormalized H_n x by the literal recursion of P:154-165 (small n only).

    H_n [x_top; x_bot] = [H_{n/2}(x_top + x_bot); H_{n/2}(x_top - x_bot)].
    """
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    if n == 1:
        return x.copy()
    if n % 2:
        raise ValueError("length must be a power of two")
    h = n // 2
    top, bot = x[:h], x[h:]
    return np.concatenate([hadamard_recursive(top + bot), hadamard_recursive(top - bot)], axis=0)


def hadamard(x):
    """Unnormalized H_n x along axis 0: the same recursion, unrolled level by level.

    Level with block size m: every block [x_top; x_bot] becomes
    [x_top + x_bot ; x_top - x_bot]; the two halves are then transformed as
    blocks of size m/2.  Each output entry receives exactly the additions of
    ``hadamard_recursive`` in the same order (tested), without Python recursion.
    """
    x = np.array(x, dtype=np.float64, copy=True)
    n = x.shape[0]
    if n & (n - 1):
        raise ValueError("length must be a power of two")
    tail = x.shape[1:]
    m = n
    while m > 1:
        y = x.reshape((n // m, m) + tail)
        top, bot = y[:, : m // 2], y[:, m // 2:]
        x = np.concatenate([top + bot, top - bot], axis=1).reshape((n,) + tail)
        m //= 2
    return x


# ----------------------------------------------------------------------------
# The sketch (Algorithm 1 step 5 inputs).
# ----------------------------------------------------------------------------

def sketch(M, seed, r, p=0, n=None, sampling="exact"):
    """H~ D M for M = [A | b] (n x c), float64 result of shape (r, c).

    Steps, in the paper's order: pad M with zero rows to N; D M
    (step 4); normalized H_N; keep rows K of S H_N with scale
    sqrt(N/r) (steps 2-3, reading R2).  sampling="bernoulli" keeps each row with
    probability r/N (plan_samples_bernoulli; the result then has that random
    number of rows, each still scaled by sqrt(N/r)).
    """
    M = np.asarray(M, dtype=np.float64)
    if M.ndim == 1:
        M = M[:, None]
    n = M.shape[0] if n is None else int(n)
    N = padded_size(n)
    sigma = plan_signs(seed, p, N)
    K = plan_samples_bernoulli(seed, p, N, r) if sampling == "bernoulli" else plan_samples(seed, p, N, r)
    Mpad = np.zeros((N, M.shape[1]), dtype=np.float64)
    Mpad[: M.shape[0]] = M
    DM = sigma[:, None] * Mpad
    HDM = hadamard(DM) / math.sqrt(N)          # normalized H_N
    return math.sqrt(N / r) * HDM[K]            # non-zero rows of S H_N, times D M


def sketch_rows_partial(M_rows, row0, n, seed, r, p=0):
    """Unscaled partial sums over rows [row0, row0 + len(M_rows)) of an n-row [A | b]:

        P[t, j] = sum_{i in rows} (-1)^{popc(k_t & i)} sigma_i M[i, j]  (float64, (r, c)).

    Written as the definition restricted to those rows: sqrt(r) times the sketch of the
    n-row matrix that equals M_rows on them and is zero elsewhere (H~ D is linear,
    P:311-312), so the sketch is r^{-1/2} times the sum over a row partition.
    """
    M_rows = np.asarray(M_rows, dtype=np.float64)
    if M_rows.ndim == 1:
        M_rows = M_rows[:, None]
    full = np.zeros((int(n), M_rows.shape[1]), dtype=np.float64)
    full[int(row0):int(row0) + M_rows.shape[0]] = M_rows
    return math.sqrt(r) * sketch(full, seed, r, p=p)


def sketch_problem(A, b, seed, r, p=0):
    """(H~ D A, H~ D b) with one shared plan (reading R7)."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    SM = sketch(np.column_stack([A, b]), seed, r, p=p)
    return SM[:, :-1], SM[:, -1]


def sketch_entry_bruteforce(col, seed, r, t, p=0):
    """One sketched entry from the closed form of the definition (tiny n only).

    SM[t] = sqrt(N/r) * N^{-1/2} * sum_i (-1)^{popc(k_t & i)} sigma_i col_i,
    where H_N[k, i] = (-1)^{popc(k & i)} in natural order (reading R3).
    """
    col = np.asarray(col, dtype=np.float64)
    n = col.shape[0]
    N = padded_size(n)
    sigma = plan_signs(seed, p, N)
    k = int(plan_samples(seed, p, N, r)[t])
    acc = 0.0
    for i in range(n):
        acc += (-1.0) ** bin(k & i).count("1") * sigma[i] * col[i]
    return math.sqrt(N / r) / math.sqrt(N) * acc
