"""GPU sketch vs oracle, element by element (through the C ABI)."""

import math

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    import paper_0812_4547_b200 as m
    torch.cuda.init()
    return m


def to_dev(M):
    import torch
    t = torch.from_numpy(np.asfortranarray(M, dtype=np.float32))
    return t.t().contiguous().t().cuda() if t.dim() == 2 else t.cuda()


def tol(M, n):
    """north_star: |gpu - oracle| <= 1e-5 * sqrt(n) * max|col| (R11: n original, per column)."""
    return 1e-5 * math.sqrt(n) * np.max(np.abs(M), axis=0)


def check_close(got, ref, M):
    got = np.asarray(got, dtype=np.float64)
    bound = tol(M, M.shape[0])
    err = np.abs(got - ref)
    assert np.all(err <= bound[None, :] + 1e-30), (err.max(), (err / np.maximum(bound, 1e-30)).max())
    return (err / np.maximum(bound, 1e-30)).max()


# Tile kernel each case must run (srht_debug_last_kernel): 1 k_sketch_tiles (v1), 2 k_sketch_ws (v2,
# dense columns not 16-byte aligned), 3 k_sketch_tma (v3, aligned dense, N >= 2^14, r <= 16384),
# 5 k_sketch_col (whole-column kernel, N = 2^13 with enough columns for one slab per column).
V1, V2, V3, COL = 1, 2, 3, 5


def last_kernel(lib):
    return lib.library().srht_debug_last_kernel()


@pytest.mark.parametrize("n,c,r,seed,kern", [
    (4096, 17, 256, 0, V1),         # config 1 shape
    (1000, 3, 100, 1, V1),          # ragged tail, r not a power of two
    (5, 2, 3, 2, V1),               # tiny n (N = 8 < tile)
    (1, 1, 1, 3, V1),               # n = 1
    (10000, 4, 352, 4, V3),         # paper Section 4.2 shape class (n = 10,000 -> N = 16384)
    (33333, 5, 1500, 5, V2),        # several tiles + ragged; ld = n is not a multiple of 4
    (1 << 17, 3, 4096, 6, V3),      # multi sub-block, single slab
    (300000, 2, 2000, 7, V3),       # several slabs (partials + reduce)
    (3 << 19, 2, 8192, 8, V3),      # several slabs
    (1 << 21, 2, 16384, 9, V3),     # B = 2^14, two slabs
    (70000, 2, 20000, 10, V1),      # r > 16384: v1 with several sample groups
    ((1 << 20) + 3 * 16384 + 7, 3, 8192, 11, V2),   # ragged last tile, tail slab of 4 sub-blocks
    ((1 << 20) + 5 * 16384 + 1, 2, 16384, 12, V2),  # tail slab of 6 sub-blocks (inactive Gray steps)
    ((1 << 20) + 5 * 16384 + 4, 2, 16384, 18, V3),  # the same tail through v3 (aligned)
    (1 << 14, 3, 300, 13, V3),      # a single tile
    ((1 << 14) + 1, 2, 16384, 14, V2),  # r = 16384 > n, two tiles, second holds one row
    ((1 << 14) + 4, 2, 16384, 19, V3),  # the same through v3: second tile holds 4 rows
    (5000, 3, 700, 15, V1),         # N = 2^13, few columns: short slabs, v1
    (8192, 2, 8192, 16, COL),       # N = 2^13, r = N: a single tile per column -> whole-column kernel
    (8192, 1200, 1024, 17, COL),    # N = 2^13, many columns: whole-column kernel
    (1 << 20, 2, 14000, 20, V3),    # v3 with rpt/8 = 8 shared-gather slots (56 load slots: odd chunk count)
    ((1 << 18) + 12344, 3, 12000, 21, V3),  # the same slot count with a ragged tail tile (ld % 4 == 0)
])
def test_dense_random_parity(lib, n, c, r, seed, kern):
    from oracle import srht as osr
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, c)).astype(np.float32)
    plan = lib.Plan(n, c - 1, r, seed)
    SM = plan.sketch_columns(to_dev(M)).cpu().numpy()
    assert last_kernel(lib) == kern
    ref = osr.sketch(M.astype(np.float64), seed, r)
    check_close(SM, ref, M)


def test_random_shapes_fuzz(lib):
    # 24 seeded random shapes across every dense path (v1 tiles, whole-column N = 2^13, v2 for
    # unaligned ld, v3) and CSC, each checked entry by entry against the oracle
    from oracle import srht as osr
    rng = np.random.default_rng(2024)
    for case in range(24):
        n = int(rng.integers(1, 400000)) if case % 3 else int(rng.integers(4097, 8193))
        N = 1 << max(1, (n - 1).bit_length())
        c = int(rng.integers(1, 5))
        r = int(rng.integers(1, min(N, 20000) + 1))
        seed = int(rng.integers(0, 2**31))
        M = rng.standard_normal((n, c)).astype(np.float32)
        plan = lib.Plan(n, c - 1, r, seed)
        if case % 4 == 1:  # CSC with ~1% density
            mask = rng.random((n, c)) < 0.01
            M = np.where(mask, M, 0).astype(np.float32)
            colptr = np.concatenate([[0], np.cumsum(mask.sum(axis=0))]).astype(np.int64)
            rowidx = np.concatenate([np.nonzero(mask[:, j])[0] for j in range(c)]).astype(np.int32)
            vals = np.concatenate([M[mask[:, j], j] for j in range(c)]).astype(np.float32)
            SM = plan.sketch_columns(_csc_dev(colptr, rowidx, vals, (n, c))).cpu().numpy()
        else:
            SM = plan.sketch_columns(to_dev(M)).cpu().numpy()
        ref = osr.sketch(M.astype(np.float64), seed, r)
        check_close(SM, ref, M)


@pytest.mark.parametrize("n,r", [(4096, 256), (1 << 16, 1024), (1 << 18, 4096), (1 << 20, 16384), (50000, 1024)])
def test_integer_inputs_bit_exact(lib, n, r):
    # Integer inputs with n * max|a| < 2^24 make every partial sum exact in FP32
    # under any summation order, and r = 4^j makes r^{-1/2} a power of two, so
    # the GPU result must equal the oracle's exactly.
    from oracle import srht as osr
    rng = np.random.default_rng(n)
    amax = max(1, (1 << 23) // n)
    M = rng.integers(-amax, amax + 1, size=(n, 3)).astype(np.float32)
    plan = lib.Plan(n, 2, r, 11)
    SM = plan.sketch_columns(to_dev(M)).cpu().numpy().astype(np.float64)
    ref = osr.sketch(M.astype(np.float64), 11, r)
    assert np.array_equal(SM, ref)


@pytest.mark.parametrize("n,r", [(8192, 1024), (5000, 256), (8192, 1000)])
def test_column_kernel_integer_bit_exact(lib, n, r):
    # Whole-column kernel (N = 2^13): with r <= 1024 the last three row bits are evaluated only at
    # the kept rows (plan gather order); integer inputs keep every sum exact, so the batched sketch
    # must equal the oracle's bit for bit (r = 1000 is not a power of 4: compare with the same
    # FP32 scale applied).
    from oracle import srht as osr
    batch, c = 12, 100  # >= 1184 columns: one slab per column (the column kernel's condition)
    rng = np.random.default_rng(n + r)
    amax = max(1, (1 << 23) // n)
    M = rng.integers(-amax, amax + 1, size=(n, batch * c)).astype(np.float32)
    M[rng.random(M.shape) < 0.95] = 0.0  # sparse CSC input (the batched CSC path runs the column kernel)
    colptr = np.concatenate([[0], np.cumsum((M != 0).sum(axis=0))]).astype(np.int64)
    rows = np.concatenate([np.flatnonzero(M[:, j]) for j in range(M.shape[1])]).astype(np.int32)
    vals = np.concatenate([M[M[:, j] != 0, j] for j in range(M.shape[1])]).astype(np.float32)
    plan = lib.Plan(n, c - 1, r, 17, batch=batch)
    out = plan.sketch_batched(_csc_dev(colptr, rows, vals, (n, batch * c))).cpu().numpy().astype(np.float64)
    assert lib.library().srht_debug_last_kernel() == 5
    scale = float(np.float32(1.0 / np.sqrt(r)))
    for p in range(batch):
        ref = osr.sketch(M[:, p * c:(p + 1) * c].astype(np.float64), 17, r, p=p)  # r^{-1/2} sum
        unscaled = ref * np.sqrt(r)  # exact integers
        assert np.allclose(unscaled, np.round(unscaled), atol=1e-6)
        want = (np.round(unscaled).astype(np.float32) * np.float32(scale)).astype(np.float64)
        assert np.array_equal(out[p].T, want)


def test_single_nonzero_closed_form(lib):
    from oracle import srht as osr
    n, r, seed = 20000, 1024, 3
    N = osr.padded_size(n)
    rows = [0, 1, 31, 4095, 12345, n - 1]
    M = np.zeros((n, len(rows)), dtype=np.float32)
    for j, i in enumerate(rows):
        M[i, j] = 1.0
    plan = lib.Plan(n, 0, r, seed)
    SM = plan.sketch_columns(to_dev(M)).cpu().numpy()
    sig = osr.plan_signs(seed, 0, N)
    K = osr.plan_samples(seed, 0, N, r)
    for j, i in enumerate(rows):
        expect = np.array([sig[i] * (-1.0) ** bin(int(k) & i).count("1") for k in K]) / 32.0
        assert np.array_equal(SM[:, j].astype(np.float64), expect)


def test_sketch_A_b_matches_columns(lib):
    import torch
    n, d, r = 30000, 6, 512
    M, _ = workloads.dense_host(n, d, seed=4)
    plan = lib.Plan(n, d, r, 4)
    Md = to_dev(M)
    SA, Sb = plan.sketch(Md[:, :d], Md[:, d])
    SM = plan.sketch_columns(Md)
    torch.cuda.synchronize()
    assert torch.equal(SA, SM[:, :d]) and torch.equal(Sb, SM[:, d])


def test_column_shards_bit_identical(lib):
    import torch
    n, c, r = 1 << 19, 13, 4096
    M = np.random.default_rng(0).random((n, c), dtype=np.float32)
    plan = lib.Plan(n, c - 1, r, 1)
    Md = to_dev(M)
    full = plan.sketch_columns(Md)
    parts = [plan.sketch_columns(Md[:, a:b]) for a, b in [(0, 5), (5, 6), (6, 13)]]
    assert torch.equal(full, torch.cat(parts, dim=1))


def test_tma_kernel_repeatable(lib):
    # kernel v3 (TMA ring, split quarter loads, mbarrier elections, slot-order partials):
    # repeated launches on the same input agree bit for bit, and a tail tile is included
    import torch
    n, c, r = (1 << 20) + 12345, 6, 8192
    M = torch.empty((c, (n + 3) & ~3), dtype=torch.float32, device="cuda").t()[:n]  # 16-byte aligned columns
    lib.gen_uniform(9, 0, M)
    plan = lib.Plan(n, c - 1, r, 3)
    ws = plan.workspace(c)
    ref = plan.sketch_columns(M, workspace=ws).clone()
    assert lib.library().srht_debug_last_kernel() == 3
    for _ in range(4):
        assert torch.equal(plan.sketch_columns(M, workspace=ws), ref)


def test_ld_greater_than_n_and_unaligned(lib):
    import torch
    from oracle import srht as osr
    n, c, r = 5003, 3, 200
    rng = np.random.default_rng(2)
    big = torch.from_numpy(rng.standard_normal((5011, c + 1)).astype(np.float32)).t().contiguous().t().cuda()
    view = big[3:3 + n, 1:]  # ld = 5011, base pointer not 16-byte aligned
    plan = lib.Plan(n, c - 1, r, 2)
    SM = plan.sketch_columns(view).cpu().numpy()
    Mh = view.cpu().numpy()
    check_close(SM, osr.sketch(Mh.astype(np.float64), 2, r), Mh)


def _csc_dev(colptr, rowidx, vals, shape):
    import torch
    return lib_csc(torch.from_numpy(np.asarray(colptr, dtype=np.int64)).cuda(),
                   torch.from_numpy(np.asarray(rowidx, dtype=np.int32)).cuda(),
                   torch.from_numpy(np.asarray(vals, dtype=np.float32)).cuda(), shape)


def check_fp64_mode(got, ref, M):
    """FP64-accumulation mode: each output is the FP64 sum rounded once to FP32, so it is
    within one FP32 spacing of the exact sketch (plus an FP64-level absolute term for
    entries that cancel to ~0)."""
    got = np.asarray(got, dtype=np.float64)
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    floor = 1e-12 * math.sqrt(M.shape[0]) * np.max(np.abs(M), axis=0)
    err = np.abs(got - ref)
    assert np.all(err <= ulp + floor[None, :] + 1e-300), float((err / (ulp + floor[None, :] + 1e-300)).max())


F64, TMA64 = 4, 6  # k_sketch_f64 (CSC, batched, small or unaligned inputs), k_sketch_tma64 (aligned dense)


@pytest.mark.parametrize("n,c,r,seed,kern", [
    (4096, 17, 256, 0, TMA64),        # config 1 shape: a single 2^12 tile
    (1000, 3, 100, 1, F64),           # N < 2^12: the plain FP64 kernel
    (1, 1, 1, 3, F64),                # n = 1
    (33333, 3, 1500, 5, F64),         # ld = n not a multiple of 4 (no TMA)
    (300000, 2, 2000, 7, TMA64),      # several slabs: FP64 partials + FP64 reduce
    (5000, 3, 700, 15, TMA64),        # ragged tail tile (904 rows) staged by the producers
    ((1 << 20) + 4100, 2, 8192, 11, TMA64),  # tail tile of 4 rows, last slab short
    (3 << 19, 3, 8192, 8, TMA64),     # r = 8192: one sample group of 32 accumulators per thread
    (1 << 21, 2, 16384, 9, TMA64),    # two sample groups
    (70000, 2, 20000, 10, TMA64),     # three sample groups, r not a multiple of the group size
    (40000, 2, 30000, 12, TMA64),     # four sample groups
    (1 << 16, 2, 37, 13, TMA64),      # 4 accumulators per thread, most slots empty
    (70000, 2, 40000, 14, F64),       # r > 32768: the plain FP64 kernel
])
def test_fp64_mode_dense_parity(lib, n, c, r, seed, kern):
    from oracle import srht as osr
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, c)).astype(np.float32)
    plan = lib.Plan(n, c - 1, r, seed, accum="fp64")
    SM = plan.sketch_columns(to_dev(M), workspace=plan.workspace(c)).cpu().numpy()
    assert last_kernel(lib) == kern
    ref = osr.sketch(M.astype(np.float64), seed, r)
    check_fp64_mode(SM, ref, M)


@pytest.mark.parametrize("n,r", [(1 << 20, 4096), (3 << 18, 16384), (50000, 1024), (4096, 64)])
def test_fp64_mode_integer_inputs_correctly_rounded(lib, n, r):
    # Integers up to 2^24 are exact in FP32 and their sums (< 2^53) exact in FP64 under any
    # order; r = 4^j makes the scale a power of two.  So the FP64 mode must return the exact
    # sketch rounded once to FP32 -- the oracle's value rounded to FP32, bit for bit.
    from oracle import srht as osr
    rng = np.random.default_rng(n + r)
    M = rng.integers(-(1 << 24), (1 << 24) + 1, size=(n, 3)).astype(np.float32)
    plan = lib.Plan(n, 2, r, 17, accum="fp64")
    SM = plan.sketch_columns(to_dev(M), workspace=plan.workspace(3)).cpu().numpy()
    assert last_kernel(lib) == TMA64
    ref = osr.sketch(M.astype(np.float64), 17, r).astype(np.float32)
    assert np.array_equal(SM, ref)


def test_fp64_mode_repeatable_and_shard_invariant(lib):
    # deterministic (fixed slab order) and independent of how the columns are split
    import torch
    n, c, r = (1 << 20) + 4100, 6, 8192
    M = to_dev(np.random.default_rng(5).random((n, c), dtype=np.float32))
    plan = lib.Plan(n, c - 1, r, 3, accum="fp64")
    ws = plan.workspace(c)
    a = plan.sketch_columns(M, workspace=ws).clone()
    b = plan.sketch_columns(M, workspace=ws)
    assert torch.equal(a, b)
    parts = torch.cat([plan.sketch_columns(M[:, :2], workspace=ws), plan.sketch_columns(M[:, 2:], workspace=ws)], 1)
    assert torch.equal(a, parts)


def test_fp64_mode_row_shards_dense(lib):
    import torch
    from oracle import srht as osr
    n, c, r, seed = (3 << 19) + 780, 3, 16384, 31
    M = np.random.default_rng(seed).standard_normal((n, c)).astype(np.float32)
    Md = to_dev(M)
    plan = lib.Plan(n, c - 1, r, seed, accum="fp64")
    g = plan.row_shard_rows()
    tot = np.zeros((r, c))
    for a, b in _row_cuts(n, g, 3):
        P = plan.sketch_rows_partial(Md[a:b], a, workspace=plan.workspace(c)).cpu().numpy()
        assert last_kernel(lib) == TMA64
        ref = osr.sketch_rows_partial(M[a:b].astype(np.float64), a, n, seed, r)
        assert np.all(np.abs(P - ref) <= 1e-9 * np.maximum(np.abs(ref), 1.0))
        tot += P
    fin = plan.rows_finish(torch.from_numpy(np.asfortranarray(tot)).cuda()).cpu().numpy()
    check_fp64_mode(fin, osr.sketch(M.astype(np.float64), seed, r), M)


def test_fp64_mode_csc_and_batched(lib):
    from oracle import srht as osr
    n, ncols, per, r = 300000, 3, 3000, 2048
    colptr, rowidx, vals = workloads.csc_lognormal(1, n, ncols, per)
    dense = workloads.csc_to_dense(colptr, rowidx, vals, n, ncols)
    plan = lib.Plan(n, ncols - 1, r, 5, accum="fp64")
    SM = plan.sketch_columns(_csc_dev(colptr, rowidx, vals, (n, ncols)), workspace=plan.workspace(ncols)).cpu().numpy()
    check_fp64_mode(SM, osr.sketch(dense, 5, r), dense.astype(np.float32))
    batch, n, c, r = 5, 3000, 4, 256
    M = np.random.default_rng(3).random((n, batch * c), dtype=np.float32)
    plan = lib.Plan(n, c - 1, r, 13, batch=batch, accum="fp64")
    out = plan.sketch_batched(to_dev(M)).cpu().numpy()
    for p in range(batch):
        check_fp64_mode(out[p].T, osr.sketch(M[:, p * c:(p + 1) * c].astype(np.float64), 13, r, p=p),
                        M[:, p * c:(p + 1) * c])


def lib_csc(*a):
    import paper_0812_4547_b200 as m
    return m.CSC(*a)


@pytest.mark.parametrize("n,ncols,per,r", [(8192, 12, 164, 1024), (1 << 17, 5, 1311, 4096), (3000, 4, 40, 64),
                                           (300000, 3, 3000, 2048)])
def test_csc_parity(lib, n, ncols, per, r):
    from oracle import srht as osr
    colptr, rowidx, vals = workloads.csc_lognormal(1, n, ncols, per)
    dense = workloads.csc_to_dense(colptr, rowidx, vals, n, ncols)
    plan = lib.Plan(n, ncols - 1, r, 5)
    SM = plan.sketch_columns(_csc_dev(colptr, rowidx, vals, (n, ncols))).cpu().numpy()
    check_close(SM, osr.sketch(dense, 5, r), dense.astype(np.float32))


def test_csc_empty_and_duplicate_columns(lib):
    from oracle import srht as osr
    n, r = 5000, 300
    # col0: empty; col1: duplicates of row 7 (summed) and rows at the tile edges; col2: one entry at n-1
    colptr = np.array([0, 0, 6, 7], dtype=np.int64)
    rowidx = np.array([7, 7, 1023, 1024, 2047, 4999, 4999], dtype=np.int32)
    vals = np.array([1.5, 2.5, -1.0, 3.0, 0.25, 4.0, -2.0], dtype=np.float32)
    dense = workloads.csc_to_dense(colptr, rowidx, vals, n, 3)
    plan = lib.Plan(n, 2, r, 9)
    SM = plan.sketch_columns(_csc_dev(colptr, rowidx, vals, (n, 3))).cpu().numpy()
    assert np.all(SM[:, 0] == 0)
    check_close(SM, osr.sketch(dense, 9, r), dense.astype(np.float32) + 1e-30)


def test_mixed_csc_A_dense_b(lib):
    import torch
    from oracle import srht as osr
    w = workloads.config3_host(n=1 << 15, d=20)
    n, d, r = w["n"], w["d"], 2048
    plan = lib.Plan(n, d, r, 0)
    A = _csc_dev(w["colptr"], w["rowidx"], w["vals"], (n, d))
    SA, Sb = plan.sketch(A, torch.from_numpy(w["b"]).cuda())
    dense = workloads.csc_to_dense(w["colptr"], w["rowidx"], w["vals"], n, d)
    M = np.column_stack([dense, w["b"].astype(np.float64)])
    ref = osr.sketch(M, 0, r)
    got = np.column_stack([SA.cpu().numpy(), Sb.cpu().numpy()])
    check_close(got, ref, M.astype(np.float32))


def test_batched_dense_parity(lib):
    from oracle import srht as osr
    batch, n, c, r = 7, 3000, 4, 256
    rng = np.random.default_rng(3)
    M = rng.random((n, batch * c), dtype=np.float32)
    plan = lib.Plan(n, c - 1, r, 13, batch=batch)
    out = plan.sketch_batched(to_dev(M)).cpu().numpy()  # (batch, c, r)
    for p in range(batch):
        ref = osr.sketch(M[:, p * c:(p + 1) * c].astype(np.float64), 13, r, p=p)
        check_close(out[p].T, ref, M[:, p * c:(p + 1) * c])


def test_batched_csc_parity_small(lib):
    from oracle import srht as osr
    w = workloads.config2_host(batch=20, n=8192, d=10)
    n, c, r = w["n"], w["d"] + 1, w["r"]
    plan = lib.Plan(n, w["d"], r, 0, batch=w["batch"])
    out = plan.sketch_batched(_csc_dev(w["colptr"], w["rowidx"], w["vals"], (n, w["batch"] * c))).cpu().numpy()
    dense = workloads.csc_to_dense(w["colptr"], w["rowidx"], w["vals"], n, w["batch"] * c)
    for p in range(w["batch"]):
        blk = dense[:, p * c:(p + 1) * c]
        check_close(out[p].T, osr.sketch(blk, 0, r, p=p), blk.astype(np.float32))


def test_host_buffer_call_matches_device(lib):
    import torch
    n, c, r = 1 << 20, 9, 8192
    M = torch.rand((c, n), dtype=torch.float32).t()
    plan = lib.Plan(n, c - 1, r, 0)
    dev = plan.sketch_columns(M.t().contiguous().t().cuda()).cpu()
    host = plan.sketch_columns_host(M.t().contiguous().pin_memory().t())
    assert torch.equal(dev, host)


def test_invalid_sketch_arguments(lib):
    import torch
    plan = lib.Plan(100, 1, 10, 0)
    with pytest.raises(lib.SrhtError):
        plan.sketch_columns(torch.zeros((99, 2), device="cuda").t().contiguous().t())


@pytest.mark.parametrize("n,r", [(1 << 20, 8192), (1 << 26, 16384), (1 << 18, 5000), (1 << 15, 16384)])
def test_ws_slot_layout(lib, n, r):
    # Kernel-v2 consumer slots: every sample exactly once, metadata consistent
    # with the plan, and each warp-row of 32 gathers at most 2-way bank-conflicted.
    import ctypes
    from paper_0812_4547_b200 import _lib
    plan = lib.Plan(n, 1, r, 3)
    L = _lib.load()
    rpt = ctypes.c_int()
    assert L.srht_debug_copy_ws_layout(plan._h, None, None, ctypes.byref(rpt)) == 0
    meta = np.empty(rpt.value * 256, dtype=np.uint32)
    perm = np.empty(rpt.value * 256, dtype=np.int32)
    assert L.srht_debug_copy_ws_layout(plan._h, meta.ctypes.data, perm.ctypes.data, ctypes.byref(rpt)) == 0
    valid = perm >= 0
    assert np.array_equal(np.sort(perm[valid]), np.arange(r))
    K = plan.indices().astype(np.int64)
    lo = K[perm[valid]] & ((1 << 14) - 1)
    phys = (lo & 511) + (((lo >> 9) & 7) << 2) + (lo >> 9) * 544
    assert np.array_equal(meta[valid] & 0x1FFFF, (phys * 4).astype(np.uint32))
    banks = np.where(valid, ((meta & 0x1FFFF) // 4 % 32).astype(np.int64), -1).reshape(-1, 32)
    worst = max(np.bincount(row[row >= 0], minlength=32).max() if (row >= 0).any() else 0 for row in banks)
    assert worst <= 2, worst


@pytest.mark.parametrize("n,r,want_pairs", [(1 << 26, 16384, 16), (1 << 20, 8192, 4), (1 << 20, 16384, 16),
                                             (1 << 16, 1024, 0), (1 << 18, 5000, 0)])
def test_v3_shared_gather_layout(lib, n, r, want_pairs):
    # Kernel-v3 consumer layout with shared gathers: every sample is an accumulator exactly once;
    # load slot l < pairs feeds accumulators (2l, 2l+1), which must be two samples with one k_lo;
    # the others feed accumulator pairs + l; offsets match the mid layout of k_lo; every warp-row
    # of 32 loads is at most 2-way bank-conflicted.
    import ctypes
    from paper_0812_4547_b200 import _lib
    plan = lib.Plan(n, 1, r, 3)
    L = _lib.load()
    rpt, pairs = ctypes.c_int(), ctypes.c_int()
    assert L.srht_debug_copy_v3_layout(plan._h, None, None, ctypes.byref(rpt), ctypes.byref(pairs)) == 0
    R, P = rpt.value, pairs.value
    assert P == want_pairs
    nl = R - P
    meta = np.empty(256 * nl, dtype=np.uint32)
    ttab = np.empty(256 * (R // 2), dtype=np.uint32)
    assert L.srht_debug_copy_v3_layout(plan._h, meta.ctypes.data, ttab.ctypes.data, ctypes.byref(rpt),
                                       ctypes.byref(pairs)) == 0
    meta = meta.reshape(256, nl)
    tt = ttab.reshape(256, R // 2)
    acc_t = np.stack([tt & 0xFFFF, tt >> 16], axis=2).reshape(256, R).astype(np.int64)  # [c][q]
    valid = acc_t != 0xFFFF
    assert np.array_equal(np.sort(acc_t[valid]), np.arange(r))
    K = plan.indices().astype(np.int64)
    lo = K & ((1 << 14) - 1)

    def mid(x):  # kernel v3 z layout
        return ((x >> 1) & 127) + 130 * ((x & 1) | ((x >> 8) << 1))

    for c in range(256):
        for l in range(nl):
            qs = (2 * l, 2 * l + 1) if l < P else (P + l,)
            ts = [acc_t[c, q] for q in qs if acc_t[c, q] != 0xFFFF]
            if not ts:
                continue
            assert len({int(lo[t]) for t in ts}) == 1, (c, l)
            assert meta[c, l] == 4 * mid(int(lo[ts[0]])), (c, l)
    used = np.zeros((256, nl), dtype=bool)
    for l in range(nl):
        qs = (2 * l, 2 * l + 1) if l < P else (P + l,)
        used[:, l] = np.any(valid[:, list(qs)], axis=1)
    words = np.where(used, (meta // 4).astype(np.int64), -1).T.reshape(nl, 8, 32).reshape(-1, 32)
    # a warp-wide gather costs one wavefront per distinct word in its most used bank (same-word lanes
    # are one broadcast); the plan's bank dealing stays within 2% + 4 of one per instruction
    cost = [np.bincount(np.unique(row[row >= 0]) % 32, minlength=32).max() for row in words if (row >= 0).any()]
    assert sum(cost) <= 1.02 * len(words) + 4, (sum(cost), len(words))


# ---- row shards: unscaled FP64 partials per shard, summed by the caller ----

def _row_cuts(n, g, k):
    """k shards of whole granules (the last takes the tail)."""
    gran = -(-n // g)
    cuts = [min(n, (gran * i // k) * g) for i in range(k)] + [n]
    return [(a, b) for a, b in zip(cuts, cuts[1:]) if b > a]


@pytest.mark.parametrize("n,c,r,seed,ld_pad,kern", [
    ((3 << 20) + 780, 3, 8192, 21, 0, V3),   # kernel v3 (ld = n, a multiple of 4), ragged last shard
    ((3 << 20) + 777, 3, 8192, 24, 0, V2),   # ld = n not a multiple of 4: kernel v2
    ((1 << 21) + 5, 2, 16384, 22, 1, V2),    # ld = n + 1: kernel v2
    (50000, 3, 20000, 23, 0, V1),            # r > 16384: kernel v1 (partials forced)
])
def test_row_shard_partials_dense(lib, n, c, r, seed, ld_pad, kern):
    import torch
    from oracle import srht as osr
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, c)).astype(np.float32)
    buf = torch.zeros((c, n + ld_pad), dtype=torch.float32)
    buf[:, :n] = torch.from_numpy(M.T)
    Md = buf.cuda().t()[:n]  # column-major, ld = n + ld_pad
    plan = lib.Plan(n, c - 1, r, seed)
    g = plan.row_shard_rows()
    full = plan.sketch_columns(Md, workspace=plan.workspace(c)).cpu().numpy().astype(np.float64)
    tot = np.zeros((r, c))
    for a, b in _row_cuts(n, g, 3):
        P = plan.sketch_rows_partial(Md[a:b], a, workspace=plan.workspace(c)).cpu().numpy()
        assert last_kernel(lib) == kern
        ref = osr.sketch_rows_partial(M[a:b].astype(np.float64), a, n, seed, r)
        bound = 1e-5 * math.sqrt(n) * np.max(np.abs(M), axis=0) * math.sqrt(r)
        assert np.all(np.abs(P - ref) <= bound[None, :])
        tot += P
    scaled = (tot / math.sqrt(r)).astype(np.float32).astype(np.float64)
    # the library's finish (srht_rows_finish) is the same FP64 scale and one rounding
    import torch
    fin = plan.rows_finish(torch.from_numpy(np.asfortranarray(tot)).cuda()).cpu().numpy().astype(np.float64)
    assert np.array_equal(fin, scaled)
    # same slab partials as the full sketch; only the FP64 association order differs
    ulp = np.spacing(np.abs(full).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(scaled - full) <= ulp)
    check_close(scaled, osr.sketch(M.astype(np.float64), seed, r), M)


def test_row_shard_csc_global_indices_and_fp64(lib):
    from oracle import srht as osr
    n, ncols, per, r = 300000, 3, 3000, 2048
    colptr, rowidx, vals = workloads.csc_lognormal(4, n, ncols, per)
    dense = workloads.csc_to_dense(colptr, rowidx, vals, n, ncols)
    for accum in ("fp32", "fp64"):
        plan = lib.Plan(n, ncols - 1, r, 6, accum=accum)
        g = plan.row_shard_rows()
        tot = np.zeros((r, ncols))
        for a, b in _row_cuts(n, g, 2):
            cp, ri, va = [0], [], []
            for j in range(ncols):  # the shard's entries, global row indices
                sel = slice(colptr[j], colptr[j + 1])
                keep = (rowidx[sel] >= a) & (rowidx[sel] < b)
                ri.extend(rowidx[sel][keep]); va.extend(vals[sel][keep]); cp.append(len(ri))
            P = plan.sketch_rows_partial(_csc_dev(cp, ri, va, (b - a, ncols)), a,
                                         workspace=plan.workspace(ncols)).cpu().numpy()
            ref = osr.sketch_rows_partial(dense[a:b], a, n, 6, r)
            bound = 1e-5 * math.sqrt(n) * np.max(np.abs(dense), axis=0) * math.sqrt(r)
            assert np.all(np.abs(P - ref) <= bound[None, :])
            if accum == "fp64":
                assert np.all(np.abs(P - ref) <= 1e-9 * np.maximum(np.abs(ref), 1.0))
            tot += P
        check_close(tot / math.sqrt(r), osr.sketch(dense, 6, r), dense.astype(np.float32))


def test_row_shard_invalid_arguments(lib):
    import torch
    n, r = (1 << 21), 1024
    plan = lib.Plan(n, 1, r, 0)
    g = plan.row_shard_rows()
    M = torch.zeros((2, n), device="cuda").t()
    with pytest.raises(lib.SrhtError):
        plan.sketch_rows_partial(M[g // 2:g], g // 2)        # row0 not a multiple of G
    with pytest.raises(lib.SrhtError):
        plan.sketch_rows_partial(M[0:g + 3], 0)             # ends inside a granule, not at n
    P = plan.sketch_rows_partial(M[g:], g)                  # ends at n: fine
    assert P.dtype == torch.float64 and P.shape == (r, 2)


# ---- Gram matrices of sketches (the QP form of P:570-590) ----

def test_gram_matches_oracle(lib):
    import torch
    from oracle import gram as og
    rng = np.random.default_rng(31)
    for r, c, pad in [(1000, 37, 0), (8192, 65, 0), (31, 1, 0), (16384, 128, 0), (8192, 513, 0), (777, 70, 3),
                      (4097, 200, 1), (64, 64, 0), (5, 3, 2)]:
        SM = rng.standard_normal((r, c)).astype(np.float32)
        dev = torch.zeros((c, r + pad), dtype=torch.float32)
        dev[:, :r] = torch.from_numpy(SM.T)
        G = lib.gram(dev.cuda().t()[:r]).cpu().numpy()  # ld = r + pad (unaligned when pad % 4)
        ref = og.gram(SM.astype(np.float64))
        absdot = np.abs(SM.astype(np.float64)).T @ np.abs(SM.astype(np.float64))
        assert np.all(np.abs(G - ref) <= 1e-12 * absdot + 1e-300)
        assert np.array_equal(G, G.T)


def test_gram_of_batched_sketches(lib):
    import torch
    from oracle import gram as og
    batch, n, c, r = 9, 3000, 5, 256
    M = np.random.default_rng(32).random((n, batch * c), dtype=np.float32)
    plan = lib.Plan(n, c - 1, r, 17, batch=batch)
    SMb = plan.sketch_batched(to_dev(M))          # (batch, c, r)
    G = lib.gram(SMb).cpu().numpy()
    SMh = SMb.cpu().numpy().astype(np.float64)
    for p in range(batch):
        ref = og.gram(SMh[p].T)
        absdot = np.abs(SMh[p]) @ np.abs(SMh[p]).T
        assert np.all(np.abs(G[p] - ref) <= 1e-12 * absdot + 1e-300)


# ---- NNLS on the Gram form: Algorithm 1 step 5 on the GPU ----

def _nnls_problem(rng, r, d, zeros):
    SA = rng.standard_normal((r, d)).astype(np.float32)
    xs = rng.random(d)
    xs[rng.choice(d, zeros, replace=False)] = 0.0
    Sb = (SA.astype(np.float64) @ xs + 0.1 * rng.standard_normal(r)).astype(np.float32)
    return SA, Sb


@pytest.mark.parametrize("batch,c,r", [(320, 37, 100), (300, 101, 256), (296, 112, 33), (300, 128, 40), (400, 1, 50)])
def test_gram_many_small_problems(lib, batch, c, r):
    # batch >= 296 and c <= 128: the one-CTA-per-problem upper-triangle kernel
    import torch
    rng = np.random.default_rng(c)
    SMh = rng.standard_normal((batch, c, r)).astype(np.float32)   # (batch, c, r) as sketch_batched returns
    G = lib.gram(torch.from_numpy(SMh).cuda()).cpu().numpy()
    S64 = SMh.astype(np.float64)
    for p in (0, 1, batch // 2, batch - 1):
        ref = S64[p] @ S64[p].T
        absdot = np.abs(S64[p]) @ np.abs(S64[p]).T
        assert np.all(np.abs(G[p] - ref) <= 1e-12 * absdot + 1e-300)
        assert np.array_equal(G[p], G[p].T)


@pytest.mark.parametrize("method", ["lh", "bpp"])
@pytest.mark.parametrize("r,d,zeros", [(64, 8, 4), (512, 50, 20), (2048, 100, 50), (4096, 200, 100), (2048, 300, 150),
                                       (8192, 512, 256), (600, 33, 0), (300, 40, 40)])
def test_nnls_gram_matches_lawson_hanson(lib, r, d, zeros, method):
    # Lawson-Hanson with the oracle's rules and block principal pivoting must both return the
    # oracle's NNLS optimum (unique: full column rank), same support
    from oracle import nnls
    if method == "lh" and d > 300:
        pytest.skip("the d = 512 Lawson-Hanson case runs in the config-4 pipeline test")
    rng = np.random.default_rng(d)
    SA, Sb = _nnls_problem(rng, r, d, zeros)
    G = lib.gram(to_dev(np.column_stack([SA, Sb])))
    x, it = lib.nnls_gram(G, method=method)
    x = x.cpu().numpy()
    assert int(it) > 0
    A64, b64 = SA.astype(np.float64), Sb.astype(np.float64)
    xr = nnls.lawson_hanson(A64, b64)[0]
    f = lambda v: float(np.sum((A64 @ v - b64) ** 2))
    assert abs(f(x) - f(xr)) <= 1e-10 * f(xr)
    assert np.all(x >= 0)
    assert np.array_equal(x > 0, xr > 0)  # same support
    assert np.max(np.abs(x - xr)) <= 1e-8 * max(1.0, np.max(np.abs(xr)))
    assert nnls.kkt_violation(A64, b64, x) <= 1e-9
    if d <= 10:
        xb = nnls.nnls_bruteforce(A64, b64)
        assert abs(f(x) - f(xb)) <= 1e-10 * f(xb)


def test_nnls_gram_large_d_deterministic(lib):
    # d > 156 (factor in the workspace, CTA-wide blocked solves, deletions with Givens):
    # repeated runs must agree bit for bit (a race in the shared updates would not)
    import torch
    rng = np.random.default_rng(7)
    SA, Sb = _nnls_problem(rng, 1024, 240, 120)
    G = lib.gram(to_dev(np.column_stack([SA, Sb])))
    for method in ("lh", "bpp"):  # bpp: the single-problem cluster solver (d >= 128)
        x0, it0 = lib.nnls_gram(G, method=method)
        for _ in range(3):
            x1, it1 = lib.nnls_gram(G, method=method)
            assert int(it1) == int(it0)
            assert torch.equal(x1, x0)


def test_randomized_nnls_end_to_end_on_gpu(lib):
    # Algorithm 1 on the GPU: sketch (config-1 shape) -> Gram -> Lawson-Hanson, against the
    # oracle pipeline (oracle sketch, oracle LH) through R(x~) on the original data.
    from oracle import nnls, srht as osr
    n, d, r, seed = 4096, 16, 256, 0
    M, _ = workloads.dense_host(n, d, seed=seed)
    plan = lib.Plan(n, d, r, seed)
    SM = plan.sketch_columns(to_dev(M))
    x, it = lib.nnls_gram(lib.gram(SM))
    x = x.cpu().numpy()
    A, b = M[:, :d].astype(np.float64), M[:, d].astype(np.float64)
    ref = osr.sketch(M.astype(np.float64), seed, r)
    xo = nnls.solve_sketched(ref[:, :d], ref[:, d])
    Rg, Ro = nnls.residual_norm(A, x, b), nnls.residual_norm(A, xo, b)
    assert abs(Rg - Ro) / Ro <= 1e-6


def test_nnls_bpp_ill_conditioned_uniform(lib):
    # config-4 shape class: nonnegative Uniform[0,1) columns share a large mean direction
    # (cond(Q) ~ 3 d), d = 512 as in config 4; block principal pivoting against the oracle's LH
    from oracle import nnls
    rng = np.random.default_rng(44)
    r, d = 8192, 512
    SA = rng.random((r, d), dtype=np.float32)
    xs = rng.random(d)
    xs[rng.choice(d, d // 2, replace=False)] = 0.0
    Sb = (SA.astype(np.float64) @ xs + 0.01 * rng.standard_normal(r)).astype(np.float32)
    G = lib.gram(to_dev(np.column_stack([SA, Sb])))
    x, it = lib.nnls_gram(G, method="bpp")
    x = x.cpu().numpy()
    assert int(it) > 0
    A64, b64 = SA.astype(np.float64), Sb.astype(np.float64)
    xr = nnls.lawson_hanson(A64, b64)[0]
    f = lambda v: float(np.sum((A64 @ v - b64) ** 2))
    assert abs(f(x) - f(xr)) <= 1e-10 * f(xr)
    assert np.array_equal(x > 0, xr > 0)
    assert nnls.kkt_violation(A64, b64, x) <= 1e-9


@pytest.mark.parametrize("method", ["lh", "bpp"])
def test_batched_gram_nnls_config2_shape(lib, method):
    # config-2 shape class: many independent sparse problems, sketch -> Gram -> NNLS batched
    from oracle import nnls
    w = workloads.config2_host(workloads.SEED, batch=40)
    n, d, batch, r = w["n"], w["d"], w["batch"], w["r"]
    c = d + 1
    plan = lib.Plan(n, d, r, workloads.SEED, batch=batch)
    SMb = plan.sketch_batched(_csc_dev(w["colptr"], w["rowidx"], w["vals"], (n, batch * c)))
    x, it = lib.nnls_gram(lib.gram(SMb), method=method)
    x, it, SMh = x.cpu().numpy(), it.cpu().numpy(), SMb.cpu().numpy().astype(np.float64)
    assert np.all(it > 0)
    for p in range(0, batch, 7):
        SA, Sb = SMh[p, :d].T, SMh[p, d]
        xr = nnls.lawson_hanson(SA, Sb)[0]
        f = lambda v: float(np.sum((SA @ v - Sb) ** 2))
        assert abs(f(x[p]) - f(xr)) <= 1e-10 * f(xr)


# ---- Bernoulli keeps: sketches with the random kept count ----

@pytest.mark.parametrize("n,c,r,seed", [(4096, 5, 256, 0), (1 << 20, 3, 8192, 4), (300000, 2, 2000, 7), (6000, 3, 800, 3)])
def test_bernoulli_sketch_parity(lib, n, c, r, seed):
    from oracle import srht as osr
    M = np.random.default_rng(seed).standard_normal((n, c)).astype(np.float32)
    plan = lib.Plan(n, c - 1, r, seed, sampling="bernoulli")
    SM = plan.sketch_columns(to_dev(M), workspace=plan.workspace(c)).cpu().numpy()
    ref = osr.sketch(M.astype(np.float64), seed, r, sampling="bernoulli")
    assert SM.shape == ref.shape == (plan.r, c)
    check_close(SM, ref, M)


# ---- Algorithm 2, SubspaceSampling ----

def test_subspace_sampling_matches_oracle(lib):
    import torch
    from oracle import subspace
    rng = np.random.default_rng(41)
    for n, d, r in [(5000, 4, 300), (100000, 2, 2000), (77, 3, 100)]:
        Phi = rng.standard_normal((n, d)).astype(np.float32)
        p = rng.random(n) ** 2
        p[0] = 1e3  # r p_0 >= 1: kept with scale 1
        p /= p.sum()
        K, rows = lib.subspace_sampling(to_dev(Phi), r, torch.from_numpy(p).cuda(), seed=n)
        Ko, ro = subspace.subspace_sampling(Phi.astype(np.float64), r, p, n)
        assert np.array_equal(K.cpu().numpy().astype(np.int64), Ko)   # bit-exact keep decisions
        np.testing.assert_allclose(rows.cpu().numpy(), ro, rtol=1e-6, atol=0)  # one FP32 rounding


def test_subspace_uniform_equals_bernoulli_srht(lib):
    # p_i = 1/N on Phi = H_N D [M; 0] / sqrt(N) (formed by the oracle) keeps the Bernoulli plan's rows
    import torch
    from oracle import srht as osr
    n, r, seed = 3000, 200, 5
    M = np.random.default_rng(2).standard_normal((n, 2))
    N = osr.padded_size(n)
    Mp = np.zeros((N, 2))
    Mp[:n] = M
    Phi = (osr.hadamard(osr.plan_signs(seed, 0, N)[:, None] * Mp) / np.sqrt(N)).astype(np.float32)
    K, rows = lib.subspace_sampling(to_dev(Phi), r, torch.full((N,), 1.0 / N, dtype=torch.float64).cuda(), seed=seed)
    plan = lib.Plan(n, 1, r, seed, sampling="bernoulli")
    assert np.array_equal(K.cpu().numpy(), plan.indices())


def test_binding_rejects_bad_outputs(lib):
    # the C ABI writes r x c entries: wrong shape/dtype/device outputs must fail before the call
    import torch
    n, c, r = 20000, 3, 512
    plan = lib.Plan(n, c - 1, r, 0)
    M = torch.zeros((c, n), device="cuda").t()
    bad = [torch.empty((c, r - 1), device="cuda").t(),                 # too few rows
           torch.empty((c + 1, r), device="cuda").t(),                 # too many columns
           torch.empty((c, r), device="cuda", dtype=torch.float64).t(),
           torch.empty((c, r)).t(),                                     # host tensor
           torch.empty((r, c), device="cuda")]                          # row-major
    for out in bad:
        with pytest.raises(ValueError):
            plan.sketch_columns(M, out=out)
    with pytest.raises(ValueError):
        plan.sketch(M[:, :2], M[:, 2], Sb=torch.empty(r - 1, device="cuda"))
    with pytest.raises(ValueError):
        plan.sketch_rows_partial(M, 0, out=torch.empty((c, r), device="cuda").t())  # float32, not float64
    with pytest.raises(ValueError):
        plan.rows_finish(torch.zeros((r, c), device="cuda"))                      # float32 partials
    bplan = lib.Plan(n, c - 1, r, 0, batch=2)
    with pytest.raises(ValueError):
        bplan.sketch_batched(torch.zeros((2 * c, n), device="cuda").t(), out=torch.empty((2, c, r - 1), device="cuda"))


def test_rows_finish_invalid_arguments(lib):
    import ctypes
    plan = lib.Plan(1 << 16, 1, 256, 0)
    L = lib.library()
    assert L.srht_rows_finish(plan._h, None, 256, 1, None, 256, None) == 1       # null pointers
    assert L.srht_rows_finish(plan._h, ctypes.c_void_p(16), 255, 1, ctypes.c_void_p(16), 256, None) == 1
    assert L.srht_rows_finish(plan._h, None, 256, 0, None, 256, None) == 0       # nothing to do
