"""Host logic of the plan (no GPU): the consumer slot dealing of kernel v3 (shared gathers) and the
gather order of the whole-column kernel, run on the oracle's kept rows through host-only hooks of
libsrht.so.  These layouts decide only which thread/slot handles a sample (the arithmetic is the same
for any valid layout), so the checks are the layout invariants the kernels rely on."""

import ctypes

import numpy as np
import pytest

from oracle import srht as osr


@pytest.fixture(scope="module")
def lib():
    from paper_0812_4547_b200 import build
    return ctypes.CDLL(build.build())


def v3_mid(x):
    """Kernel v3's z layout: word offset of in-tile row x."""
    return ((x >> 1) & 127) + 130 * ((x & 1) | ((x >> 8) << 1))


@pytest.mark.parametrize("N,r,seed,want_pairs", [(1 << 26, 16384, 0, 16), (1 << 20, 8192, 0, 4),
                                                 (1 << 20, 16384, 5, 16), (1 << 18, 4096, 1, 0),
                                                 (1 << 16, 1024, 2, 0), (1 << 20, 5000, 3, 0),
                                                 (1 << 20, 14000, 3, 8)])
def test_v3_shared_gather_dealing(lib, N, r, seed, want_pairs):
    K = osr.plan_samples(seed, 0, N, r).astype(np.int32)
    rpt = 8 if r <= 2048 else 16 if r <= 4096 else 32 if r <= 8192 else 64
    pairs = ctypes.c_int()
    acc_t = np.empty(rpt * 256, dtype=np.int32)
    meta = np.empty(256 * rpt, dtype=np.uint32)
    assert lib.srht_debug_deal_v3(K.ctypes.data, ctypes.c_int64(r), rpt, ctypes.byref(pairs),
                                  acc_t.ctypes.data, meta.ctypes.data) == 0
    P = pairs.value
    assert P == want_pairs
    nl = rpt - P
    acc = acc_t.reshape(rpt, 256)      # [q][c]
    meta = meta[:256 * nl].reshape(256, nl)  # [c][l]
    valid = acc >= 0
    assert np.array_equal(np.sort(acc[valid]), np.arange(r))  # every sample exactly once
    lo = (K & ((1 << 14) - 1)).astype(np.int64)
    banks = np.full((nl, 256), -1, dtype=np.int64)
    for l in range(nl):
        qs = (2 * l, 2 * l + 1) if l < P else (P + l,)
        ts = acc[list(qs)]
        used = (ts >= 0).any(axis=0)
        if l < P:  # a pair slot: its two samples share k_lo
            both = (ts >= 0).all(axis=0)
            assert np.array_equal(lo[ts[0, both]], lo[ts[1, both]])
        t0 = np.where(ts[0] >= 0, ts[0], ts[-1])
        assert np.array_equal(meta[used, l], 4 * v3_mid(lo[t0[used]]))  # byte offset of z[k_lo]
        banks[l, used] = v3_mid(lo[t0[used]])
    rows = banks.reshape(nl, 8, 32).reshape(-1, 32)  # warp-wide loads: (slot, warp) x 32 lanes
    # a warp-wide LDS costs one wavefront per distinct word in its most used bank (lanes reading the
    # same word are served by one broadcast)
    cost = [np.bincount(np.unique(row[row >= 0]) % 32, minlength=32).max() for row in rows if (row >= 0).any()]
    assert max(cost) <= 8, max(cost)  # the excess of an overfull bank may meet in one row
    # bank dealing: within 2% + 4 of the one-wavefront-per-instruction floor (round-robin dealing by
    # bank gave 511 for config 5's plan and 346 for config 4's)
    assert sum(cost) <= 1.02 * len(rows) + 4, (sum(cost), len(rows))
    # empty lanes read a word their row already reads (no extra wavefront)
    for l in range(nl):
        for w in range(8):
            lanes = slice(32 * w, 32 * w + 32)
            qs = (2 * l, 2 * l + 1) if l < P else (P + l,)
            empty = (acc[list(qs)][:, lanes] < 0).all(axis=0)
            if empty.any() and (~empty).any():
                assert set(meta[lanes, l][empty]) <= set(meta[lanes, l][~empty])
    # shared gathers cut the loads per thread to rpt - P
    assert nl * 256 >= r - 256 * P


@pytest.mark.parametrize("p", [0, 7, 2999])
def test_column_kernel_gather_order(lib, p):
    # config 2's problems: N = 2^13, r = 1024
    N, r, seed = 1 << 13, 1024, 0
    K = osr.plan_samples(seed, p, N, r).astype(np.int32)
    out = np.empty(5 * 256, dtype=np.uint32)
    assert lib.srht_debug_deal_col(K.ctypes.data, ctypes.c_int64(r), out.ctypes.data) == 0
    used = out != 0xFFFFFFFF
    t = (out[used] >> 16).astype(np.int64)
    k = (out[used] & 0xFFFF).astype(np.int64)
    assert np.array_equal(np.sort(t), np.arange(r))  # every kept row exactly once
    assert np.array_equal(k, K[t])                     # with its own row index
    steps = np.where(used, out & 0xFFFF, 0xFFFFFFFF).reshape(40, 32)
    gather = store = 0
    for row in steps:
        ks = row[row != 0xFFFFFFFF].astype(np.int64)
        if not len(ks):
            continue
        lo = ks & 1023
        gather += 8 * np.bincount((lo + (lo >> 5)) & 31, minlength=32).max()
    for row in np.where(used, out >> 16, 0xFFFFFFFF).reshape(40, 32):
        ts = row[row != 0xFFFFFFFF].astype(np.int64)
        if len(ts):
            store += np.bincount(ts & 31, minlength=32).max()
    # the one-per-bank bound is 8 x 40 = 320 gather and 40 store wavefronts; a sorted, undealt
    # order costs ~2x that
    assert gather <= 8 * 48 and store <= 64, (gather, store)
