"""Fused gather over peer memory (srht_sketch_columns_peers, dist.sketch_sharded_p2p) on one B200.

Every rank's output buffer is mapped into every rank with CUDA IPC handles; each rank's sketch
stores its columns straight into all of them (kernel v3's slab reduction, or one copy kernel on the
other paths).  Here two processes share GPU 0 (a gloo group for the handle exchange and a host
barrier after a device synchronize: no kernel waits on another), and the gathered result must be
bit-identical to the single-process sketch -- the slab geometry depends only on (n, r).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(n, c, kind):
    rng = np.random.default_rng(99)
    M = rng.standard_normal((n, c)).astype(np.float32)
    if kind == "csc":
        M[rng.random((n, c)) > 0.02] = 0.0
    return M


def _to_dev(M, kind):
    import torch
    import paper_0812_4547_b200 as srht
    if kind == "dense":
        return torch.from_numpy(np.asfortranarray(M)).t().contiguous().t().cuda()
    c = M.shape[1]
    mask = M != 0
    colptr = np.concatenate([[0], np.cumsum(mask.sum(axis=0))]).astype(np.int64)
    rowidx = np.concatenate([np.nonzero(mask[:, j])[0] for j in range(c)]).astype(np.int32)
    vals = np.concatenate([M[mask[:, j], j] for j in range(c)]).astype(np.float32)
    return srht.CSC(torch.from_numpy(colptr).cuda(), torch.from_numpy(rowidx).cuda(),
                    torch.from_numpy(vals).cuda(), M.shape)


def _worker(rank, world, port, n, c, r, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_0812_4547_b200 as srht
        from paper_0812_4547_b200 import dist as sdist
        plan = srht.Plan(n, c - 1, r, 5)
        M = _data(n, c, kind)
        c0, c1 = sdist.column_range(c, world, rank)
        peers = sdist.PeerOutputs(plan, c)
        out = None
        for _ in range(2):  # twice: the buffers are reused
            out = sdist.sketch_sharded_p2p(plan, _to_dev(M[:, c0:c1], kind), c, peers, host_barrier=True)
        got = out.cpu().numpy().copy()
        kern = srht.library().srht_debug_last_kernel()
        dist.barrier()
        peers.close()
        q.put((rank, got, kern))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,c,r,kind,fused", [
    ((1 << 20) + 4096, 6, 8192, "dense", True),   # kernel v3: the reduction stores into every peer
    (50000, 5, 700, "csc", False),                # kernel v1 + the copy kernel
])
def test_two_processes_fused_gather_matches_single_process(n, c, r, kind, fused):
    import torch
    import torch.multiprocessing as mp
    import paper_0812_4547_b200 as srht
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(k, world, port, n, c, r, kind, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        k, got, kern = q.get(timeout=300)
        res[k] = (got, kern)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    plan = srht.Plan(n, c - 1, r, 5)
    ref = plan.sketch_columns(_to_dev(_data(n, c, kind), kind)).cpu().numpy()
    for k in range(world):
        got, kern = res[k]
        assert (kern == 3) == fused
        assert np.array_equal(got, ref)
    torch.cuda.synchronize()


def test_single_rank_peers_and_invalid_arguments():
    import ctypes
    import torch
    import torch.distributed as dist
    import paper_0812_4547_b200 as srht
    from paper_0812_4547_b200 import dist as sdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        n, c, r = 1 << 18, 3, 4096
        M = _data(n, c, "dense")
        plan = srht.Plan(n, c - 1, r, 5)
        peers = sdist.PeerOutputs(plan, c)
        out = sdist.sketch_sharded_p2p(plan, _to_dev(M, "dense"), c, peers, host_barrier=True)
        ref = plan.sketch_columns(_to_dev(M, "dense"))
        assert torch.equal(out, ref)
        L = srht.library()
        arr = (ctypes.c_void_p * 1)(peers.ptrs[0])
        assert L.srht_sketch_columns_peers(plan._h, None, 0, arr, 1, r, None, 0, None) == 1
        peers.close()
    finally:
        dist.destroy_process_group()
