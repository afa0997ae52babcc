"""Seeded synthetic workloads of BASELINE.json (inputs only; no SRHT arithmetic).

The only module both sides of a parity test may share.  Dense Uniform[0,1)
columns come from a counter-based generator implemented twice -- on the host
here (numpy's Philox4x64 library routine) and on the device in
``srht_gen_uniform`` -- with the same definition:

    A[i, j] = (word i of Philox stream (seed, 2^32 + stream0 + j) >> 40) * 2^-24

so any column can be regenerated on the host bit-for-bit (exact FP32 values).
Everything else (x_true, noise, sparse positions, log-normal values) is drawn
on the host with ``numpy.random.Generator(Philox(key=...))`` and copied to the
device, so both sides see identical inputs.  Where b = A x_true + noise needs a
large A that lives only on the device, it is computed there in FP64 with torch
(a library call, untimed) and copied back; it is an input, not a result.

Config recipes (BASELINE.json configs 1-5):
  1 tiny dense   n=4096,  d=16,  r=256,   U[0,1) A, x_true half zeros, b = A x + N(0, 0.01^2)
  2 batched CSC  3000 problems, n=8192, d=100 (+b as column 101), 2% density
                 (exactly 164 distinct uniform rows per column), exp(N(0,1)) values,
                 every column (b included) L2-normalised, r=1024
  3 sparse tall  n=2^17, d=300, CSC 1% (1311 rows/col), exp(N(0,1)) values,
                 x_true 80% zeros else U[0,1), dense b = A x + |N(0, 0.1^2)|, r=4096
  4 dense large  n=2^20, d=512, U[0,1) A, x_true half zeros, b = A x + N(0, 0.01^2), r=8192
  5 multi-GPU    n=2^26, d=127, U[0,1) A + b like cfg 4 (128 columns, 34.4 GB), r=16384
TechTC300 (the paper's dataset) is not available; config 2 stands in
for its shape class (many independent tall sparse nonnegative problems).
"""

import math

import numpy as np

CONFIGS = {
    1: dict(name="tiny_dense", n=4096, d=16, r=256, kind="dense", density=None, batch=1),
    2: dict(name="batched_csc", n=8192, d=100, r=1024, kind="csc_batched", density=0.02, batch=3000),
    3: dict(name="sparse_tall", n=1 << 17, d=300, r=4096, kind="csc", density=0.01, batch=1),
    4: dict(name="dense_large", n=1 << 20, d=512, r=8192, kind="dense", density=None, batch=1),
    5: dict(name="multi_gpu_scale", n=1 << 26, d=127, r=16384, kind="dense", density=None, batch=1),
}

SEED = 0
_MASK64 = (1 << 64) - 1


def _rng(seed, tag):
    """Host generator for everything that is not a dense uniform column."""
    return np.random.Generator(np.random.Philox(key=np.array([seed & _MASK64, (3 << 32) + tag], dtype=np.uint64)))


def host_uniform_column(seed, stream, rows):
    """Exact FP32 Uniform[0,1) column, bit-identical to srht_gen_uniform."""
    g = np.random.Philox(key=np.array([seed & _MASK64, (1 << 32) + stream], dtype=np.uint64))
    w = g.random_raw(int(rows)).astype(np.uint64)
    return ((w >> np.uint64(40)).astype(np.float64) * 2.0 ** -24).astype(np.float32)


def host_uniform_matrix(seed, stream0, rows, cols):
    out = np.empty((rows, cols), dtype=np.float32, order="F")
    for j in range(cols):
        out[:, j] = host_uniform_column(seed, stream0 + j, rows)
    return out


def x_true_half_zeros(seed, d, tag=1):
    """x_true with a random floor(d/2)-subset of zeros and U[0,1) elsewhere."""
    g = _rng(seed, tag)
    x = g.random(d)
    x[g.permutation(d)[: d // 2]] = 0.0
    return x


def x_true_fraction_zeros(seed, d, frac, tag=1):
    g = _rng(seed, tag)
    x = g.random(d)
    x[g.permutation(d)[: int(round(frac * d))]] = 0.0
    return x


# ---------------------------------------------------------------------------
# Dense configs (1, 4, 5 and scaled variants)
# ---------------------------------------------------------------------------

def dense_host(n, d, seed=SEED, noise=0.01):
    """Host-only dense problem: (M = [A | b] float32 Fortran, x_true)."""
    A = host_uniform_matrix(seed, 0, n, d)
    x = x_true_half_zeros(seed, d)
    e = _rng(seed, 2).standard_normal(n) * noise
    b = (A.astype(np.float64) @ x + e).astype(np.float32)
    M = np.empty((n, d + 1), dtype=np.float32, order="F")
    M[:, :d] = A
    M[:, d] = b
    return M, x


def dense_device(n, d, seed=SEED, noise=0.01, device="cuda", gen_uniform=None, col_chunk=8):
    """Device dense problem: M = [A | b] (n x (d+1), column-major FP32, on device).

    A is generated on the device (srht_gen_uniform via `gen_uniform`); b is
    computed on the device in FP64 with torch and rounded to FP32.  Returns
    (M, x_true) with M a torch tensor.
    """
    import torch
    if gen_uniform is None:
        from paper_0812_4547_b200 import gen_uniform as _g
        gen_uniform = _g
    M = torch.empty((d + 1, n), dtype=torch.float32, device=device).t()
    gen_uniform(seed, 0, M[:, :d])
    x = x_true_half_zeros(seed, d)
    e = _rng(seed, 2).standard_normal(n) * noise
    b64 = torch.from_numpy(e).to(device)
    xt = torch.from_numpy(x).to(device)
    for j0 in range(0, d, col_chunk):
        j1 = min(d, j0 + col_chunk)
        b64 += M[:, j0:j1].double() @ xt[j0:j1]
    M[:, d] = b64.float()
    torch.cuda.synchronize()
    return M, x


# ---------------------------------------------------------------------------
# Sparse configs (2, 3)
# ---------------------------------------------------------------------------

def distinct_rows(g, n, ncols, k):
    """For each of ncols columns, k distinct uniform rows of [0, n) (sorted).

    Sequential draws without replacement: draw extra candidates, keep first
    occurrences in draw order, take the first k.
    """
    extra = max(16, int(4 * math.sqrt(k) + k * k / max(n, 1) * 2))
    m = k + extra
    out = np.empty((ncols, k), dtype=np.int32)
    todo = np.arange(ncols)
    while todo.size:
        cand = g.integers(0, n, size=(todo.size, m), dtype=np.int64)
        order = np.argsort(cand, axis=1, kind="stable")
        srt = np.take_along_axis(cand, order, axis=1)
        first_sorted = np.ones_like(srt, dtype=bool)
        first_sorted[:, 1:] = srt[:, 1:] != srt[:, :-1]
        first = np.empty_like(first_sorted)
        np.put_along_axis(first, order, first_sorted, axis=1)
        rank = np.cumsum(first, axis=1)
        ok = rank[:, -1] >= k
        sel = first & (rank <= k)
        rows_ok = todo[ok]
        if rows_ok.size:
            picked = cand[ok][sel[ok]].reshape(-1, k)
            out[rows_ok] = np.sort(picked, axis=1).astype(np.int32)
        todo = todo[~ok]
        m *= 2
    return out


def csc_lognormal(seed, n, ncols, per_col, tag=10, normalize=False):
    """CSC with exactly per_col distinct uniform rows per column and exp(N(0,1)) values."""
    g = _rng(seed, tag)
    rows = distinct_rows(g, n, ncols, per_col)
    vals = np.exp(g.standard_normal((ncols, per_col)))
    if normalize:
        vals /= np.sqrt(np.sum(vals * vals, axis=1, keepdims=True))
    colptr = np.arange(ncols + 1, dtype=np.int64) * per_col
    return colptr, rows.reshape(-1), vals.astype(np.float32).reshape(-1)


def csc_to_dense(colptr, rowidx, vals, n, ncols):
    out = np.zeros((n, ncols), dtype=np.float64, order="F")
    for j in range(ncols):
        a, b = colptr[j], colptr[j + 1]
        np.add.at(out[:, j], rowidx[a:b].astype(np.int64), vals[a:b].astype(np.float64))
    return out


def config2_host(seed=SEED, batch=None, n=None, d=None, density=None):
    """Batched CSC problems: all batch*(d+1) columns in one CSC (b is column d of each)."""
    c = CONFIGS[2]
    batch = c["batch"] if batch is None else batch
    n = c["n"] if n is None else n
    d = c["d"] if d is None else d
    density = c["density"] if density is None else density
    per = int(round(density * n))
    colptr, rowidx, vals = csc_lognormal(seed, n, batch * (d + 1), per, tag=20, normalize=True)
    return dict(n=n, d=d, batch=batch, r=c["r"], colptr=colptr, rowidx=rowidx, vals=vals, per_col=per)


def config3_host(seed=SEED, n=None, d=None, density=None):
    """Sparse tall CSC A with a dense b = A x_true + |N(0, 0.1^2)|."""
    c = CONFIGS[3]
    n = c["n"] if n is None else n
    d = c["d"] if d is None else d
    density = c["density"] if density is None else density
    per = int(round(density * n))
    colptr, rowidx, vals = csc_lognormal(seed, n, d, per, tag=30)
    x = x_true_fraction_zeros(seed, d, 0.8, tag=31)
    b = np.abs(_rng(seed, 32).standard_normal(n) * 0.1)
    for j in range(d):
        a, e = colptr[j], colptr[j + 1]
        np.add.at(b, rowidx[a:e].astype(np.int64), vals[a:e].astype(np.float64) * x[j])
    return dict(n=n, d=d, r=c["r"], colptr=colptr, rowidx=rowidx, vals=vals, b=b.astype(np.float32), x_true=x,
                per_col=per)


def input_bytes_dense(n, cols):
    return 4 * n * cols


def input_bytes_csc(nnz, cols, dense_b_rows=0):
    return 8 * nnz + 8 * (cols + 1) + 4 * dense_b_rows
