"""Multi-rank column sharding on CPU (gloo, world_size 2) with the oracle as the per-rank sketch.

Checks the sharding / all-gather glue of paper_0812_4547_b200.dist without GPUs:
the gathered result must equal the single-process oracle sketch exactly, for
even and uneven shards, and mismatched plans must be detected.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0812_4547_b200.dist import column_range, sketch_sharded


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OraclePlan:
    """Stands in for srht.Plan on CPU: same contract, oracle arithmetic."""

    def __init__(self, n, r, seed):
        from oracle import srht as osr
        self.n, self.r, self.seed, self.N = n, r, seed, osr.padded_size(n)

    def sketch(self, M):
        from oracle import srht as osr
        return torch.from_numpy(osr.sketch(M.numpy().astype(np.float64), self.seed, self.r).astype(np.float32))

    # introspection used by dist.plan_digest / check_same_plan
    def indices(self):
        from oracle import srht as osr
        return osr.plan_samples(self.seed, 0, self.N, self.r).astype(np.int32)

    def sign_words(self):
        from oracle import srht as osr
        return osr.sign_words(self.seed, 0, self.N)


def _worker(rank, world, port, n, c, r, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)
        M = rng.standard_normal((n, c)).astype(np.float32)
        c0, c1 = column_range(c, world, rank)
        plan = OraclePlan(n, r, seed)
        shard = torch.from_numpy(np.asfortranarray(M[:, c0:c1]))
        full = sketch_sharded(plan, shard, c, sketch_fn=plan.sketch)
        q.put((rank, full.contiguous().numpy()))
    finally:
        dist.destroy_process_group()


def _run_world(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(k, world, port) + args + (q,)) for k in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _oracle_ref(n, c, r, seed, gen=123):
    from oracle import srht as osr
    M = np.random.default_rng(gen).standard_normal((n, c)).astype(np.float32)
    return osr.sketch(M.astype(np.float64), seed, r).astype(np.float32)


@pytest.mark.parametrize("c,world", [(6, 2), (5, 2), (1, 2), (513, 2), (513, 3), (7, 3)])
def test_gloo_ranks_match_single_process(c, world):
    n, r, seed = 300, 40, 7
    res = _run_world(_worker, world, n, c, r, seed)
    ref = _oracle_ref(n, c, r, seed)
    for k in range(world):
        assert res[k].shape == (r, c)
        assert np.array_equal(res[k], ref)


def _out_worker(rank, world, port, n, c, r, seed, q):
    """The bench's path: out= given (direct gather into it when c % world == 0), then a second
    call with out=None must not alias the first call's result (the cached gather buffer)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0812_4547_b200.dist import check_same_plan
        plan = OraclePlan(n, r, seed)
        check_same_plan(plan)  # same seed on every rank: passes
        c0, c1 = column_range(c, world, rank)
        out = torch.full((c, r), float("nan"), dtype=torch.float32).t()  # column-major (r, c)
        res = []
        for gen in (123, 456):
            M = np.random.default_rng(gen).standard_normal((n, c)).astype(np.float32)
            shard = torch.from_numpy(np.asfortranarray(M[:, c0:c1]))
            got = sketch_sharded(plan, shard, c, out=out, sketch_fn=plan.sketch)
            assert got is out
            res.append(out.clone())
        a = sketch_sharded(plan, torch.from_numpy(np.asfortranarray(
            np.random.default_rng(123).standard_normal((n, c)).astype(np.float32)[:, c0:c1])), c,
            sketch_fn=plan.sketch)
        a_copy = a.clone()
        sketch_sharded(plan, torch.from_numpy(np.asfortranarray(
            np.random.default_rng(456).standard_normal((n, c)).astype(np.float32)[:, c0:c1])), c,
            sketch_fn=plan.sketch)
        q.put((rank, (res[0].contiguous().numpy(), res[1].contiguous().numpy(),
                      bool(torch.equal(a, a_copy)), a.contiguous().numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("c,world", [(6, 2), (9, 3), (5, 2)])
def test_gloo_out_direct_gather_and_no_aliasing(c, world):
    n, r, seed = 200, 32, 3
    res = _run_world(_out_worker, world, n, c, r, seed)
    ref1 = _oracle_ref(n, c, r, seed, 123)
    ref2 = _oracle_ref(n, c, r, seed, 456)
    for k in range(world):
        first, second, unchanged, a = res[k]
        assert np.array_equal(first, ref1) and np.array_equal(second, ref2)
        assert unchanged, "a later sketch_sharded call overwrote an earlier result"
        assert np.array_equal(a, ref1)


def _plan_check_worker(rank, world, port, seeds, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0812_4547_b200.dist import check_same_plan
        plan = OraclePlan(1000, 64, seeds[rank])
        try:
            check_same_plan(plan)
            q.put((rank, "ok"))
        except RuntimeError as e:
            q.put((rank, "mismatch: %s" % e))
    finally:
        dist.destroy_process_group()


def test_check_same_plan_accepts_equal_and_rejects_different_plans():
    assert all(v == "ok" for v in _run_world(_plan_check_worker, 2, (5, 5)).values())
    bad = _run_world(_plan_check_worker, 3, (5, 5, 6))
    assert all(v.startswith("mismatch") for v in bad.values())


def test_column_range_partition():
    for c in [1, 5, 128, 513]:
        for world in [1, 2, 3, 4, 8]:
            ranges = [column_range(c, world, k) for k in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == c
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


# ---- row sharding: partial sums per row shard, one all-reduce ----

class OracleRowPlan:
    """Stands in for srht.Plan for row shards on CPU: oracle partials, same contract."""

    def __init__(self, n, r, seed):
        self.n, self.r, self.seed = n, r, seed

    def partial(self, M_rows, row0):
        from oracle import srht as osr
        P = osr.sketch_rows_partial(M_rows.numpy().astype(np.float64), row0, self.n, self.seed, self.r)
        return torch.from_numpy(np.asfortranarray(P))

    def rows_finish(self, part, out=None):
        return (part * (1.0 / float(self.r) ** 0.5)).float()


def _row_worker(rank, world, port, n, c, r, seed, gran, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0812_4547_b200.dist import row_range, sketch_row_sharded
        rng = np.random.default_rng(321)
        M = rng.standard_normal((n, c)).astype(np.float32)
        r0, r1 = row_range(n, world, rank, gran)
        plan = OracleRowPlan(n, r, seed)
        full = sketch_row_sharded(plan, torch.from_numpy(M[r0:r1]), r0, partial_fn=plan.partial)
        q.put((rank, full.contiguous().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,gran", [(300, 64), (256, 128), (100, 64)])
def test_gloo_row_shards_match_single_process(n, gran):
    c, r, seed, world = 3, 40, 9, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_worker, args=(k, world, port, n, c, r, seed, gran, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import srht as osr
    M = np.random.default_rng(321).standard_normal((n, c)).astype(np.float32)
    ref = osr.sketch(M.astype(np.float64), seed, r)
    for k in range(world):
        np.testing.assert_allclose(res[k].astype(np.float64), ref, rtol=1e-6, atol=1e-6)
        assert np.array_equal(res[k], res[0])  # every rank holds the same result


def test_row_range_partition():
    from paper_0812_4547_b200.dist import row_range
    for n, gran in [(1 << 20, 1 << 14), (300, 64), (100, 64), ((1 << 20) + 5, 1 << 18)]:
        for world in [1, 2, 3, 8]:
            rr = [row_range(n, world, k, gran) for k in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == n
            for (a0, a1), (b0, b1) in zip(rr, rr[1:]):
                assert a1 == b0
            for a, b in rr:
                assert (a % gran == 0 and (b % gran == 0 or b == n)) or a == b == n  # empty tail ranks
