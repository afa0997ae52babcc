"""Column- and row-sharded SRHT across ranks (one process per GPU, torch.distributed).

Columns of M = [A | b] are independent given the plan, and every rank derives
the same D and kept rows from the same seed (R4-R6), so rank k sketches
a contiguous column range with no communication and one all-gather assembles
the r x c result (one plan for every column).  The gathered
buffer is column-major r x c as soon as shards are equal-sized; uneven shards
are padded to ceil(c / world) columns for ``all_gather_into_tensor`` and
compacted afterwards.  With the NCCL backend the gather runs over NVLink /
NVSwitch; the tile and slab geometry depend only on (n, r), so the result is
bit-identical to a single-GPU sketch.

Row sharding (for data that arrives partitioned by rows): rank k
holds rows [row0_k, row1_k) of every column, computes the unscaled FP64 partial sums
of its rows (srht_sketch_rows_partial), and one all-reduce (SUM, FP64) adds them; by
linearity of H~ D r^{-1/2} times the total is the sketch.
"""

import hashlib

import torch
import torch.distributed as dist


def column_range(c, world, rank):
    """Contiguous shard [c0, c1) of c columns for `rank` (first c % world ranks get one more)."""
    base, rem = divmod(int(c), int(world))
    c0 = rank * base + min(rank, rem)
    return c0, c0 + base + (1 if rank < rem else 0)


def plan_digest(plan):
    """64-bit digest of a plan (N, r, seed, kept rows, sign words) for cross-rank checks."""
    h = hashlib.blake2b(digest_size=8)
    h.update(("%d,%d,%d" % (plan.N, plan.r, plan.seed)).encode())
    h.update(plan.indices().tobytes())
    h.update(plan.sign_words().tobytes())
    return int.from_bytes(h.digest(), "little") & ((1 << 63) - 1)


def check_same_plan(plan, group=None, device=None):
    """Raise if the ranks in `group` do not hold the same plan."""
    d = torch.tensor([plan_digest(plan)], dtype=torch.int64, device=device)
    world = dist.get_world_size(group)
    out = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, d, group=group)
    if not bool(torch.all(out == out[0])):
        raise RuntimeError("ranks hold different SRHT plans: %s" % out.tolist())


def sketch_sharded(plan, M_shard, total_cols, group=None, out=None, sketch_fn=None, workspace=None):
    """Sketch this rank's column shard and all-gather the full r x total_cols result.

    plan:       srht Plan (same seed on every rank)
    M_shard:    this rank's columns [c0, c1) of M (column_range), column-major
    total_cols: c, the number of columns over all ranks
    sketch_fn:  optional replacement for ``plan.sketch_columns`` with the same
                contract (used by the CPU/gloo tests to plug in the oracle)
    Returns a column-major (r, total_cols) tensor on M_shard's device.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r = plan.r
    c0, c1 = column_range(total_cols, world, rank)
    cl = c1 - c0
    if M_shard.shape[1] != cl:
        raise ValueError("rank %d expects %d columns, got %d" % (rank, cl, M_shard.shape[1]))
    cmax = -(-int(total_cols) // world)
    dev = M_shard.device
    # Buffers are cached on the plan so repeated calls launch nothing but the
    # sketch kernels and the collective.  Padding rows of `local` (uneven
    # shards) are never read back.
    key = (world, cmax, str(dev))
    cache = getattr(plan, "_dist_bufs", None)
    if cache is None or cache[0] != key:
        local_buf = torch.empty((cmax, r), dtype=torch.float32, device=dev)  # [col][t] == column-major r x cmax
        gath_buf = torch.empty((world * cmax, r), dtype=torch.float32, device=dev)
        try:
            plan._dist_bufs = (key, local_buf, gath_buf)
        except AttributeError:
            pass
    else:
        _, local_buf, gath_buf = cache
    local = local_buf
    if cl:
        if sketch_fn is None:
            plan.sketch_columns(M_shard, out=local[:cl].t(), workspace=workspace)
        else:
            local[:cl] = sketch_fn(M_shard).t()
    direct = (out is not None and total_cols % world == 0 and out.stride(0) == 1
              and out.stride(1) == r and out.device == dev)
    gathered = out.t() if direct else gath_buf
    dist.all_gather_into_tensor(gathered, local, group=group)
    if direct:
        return out
    if total_cols % world == 0:
        # gath_buf is cached on the plan and reused by the next call: hand out a copy
        full = gathered if out is not None else gathered.clone()
    else:
        idx = []
        for k in range(world):
            a, b = column_range(total_cols, world, k)
            idx.extend(range(k * cmax, k * cmax + (b - a)))
        full = gathered.index_select(0, torch.tensor(idx, device=dev))
    if out is not None:
        out.copy_(full.t())
        return out
    return full.t()


class _DevArray:
    """Zero-copy torch view of a library-allocated device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr, shape, strides):
        self.__cuda_array_interface__ = {"shape": shape, "strides": strides, "typestr": "<f4",
                                         "data": (int(ptr), False), "version": 3}


class PeerOutputs:
    """Every rank's r x c output buffer, mapped into every rank (CUDA IPC), for the fused gather.

    Rank k allocates its own buffer with the library (srht_ipc_alloc), the 64-byte handles are
    all-gathered over `group`, and each rank maps the others' buffers (srht_ipc_open; peer access
    over NVLink between GPUs).  `out` is this rank's buffer as a column-major (r, c) float32 tensor.
    """

    def __init__(self, plan, total_cols, group=None):
        import ctypes
        lib = plan._lib
        self._lib = lib
        self.r, self.c = plan.r, int(total_cols)
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        nbytes = 4 * self.r * self.c
        own = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        from . import _lib as L
        L.check(lib.srht_ipc_alloc(nbytes, ctypes.byref(own), handle), "srht_ipc_alloc")
        self._own = own.value
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.ptrs = [0] * self.world
        self._opened = []
        for k in range(self.world):
            if k == self.rank:
                self.ptrs[k] = self._own
                continue
            p = ctypes.c_void_p()
            buf = (ctypes.c_char * 64).from_buffer_copy(handles[k])
            L.check(lib.srht_ipc_open(buf, ctypes.byref(p)), "srht_ipc_open")
            self.ptrs[k] = p.value
            self._opened.append(p.value)
        self.out = torch.as_tensor(_DevArray(self._own, (self.r, self.c), (4, 4 * self.r)),
                                   device=torch.device("cuda", torch.cuda.current_device()))

    def peer_order(self):
        """Device pointers with this rank's own buffer first (the library's convention)."""
        return [self.ptrs[self.rank]] + [p for k, p in enumerate(self.ptrs) if k != self.rank]

    def close(self):
        for p in self._opened:
            self._lib.srht_ipc_close(p)
        self._opened = []
        if self._own:
            self.out = None
            self._lib.srht_ipc_free(self._own)
            self._own = 0


def sketch_sharded_p2p(plan, M_shard, total_cols, peers, group=None, workspace=None, host_barrier=False):
    """Column-shard sketch with the gather fused into the sketch (no NCCL all-gather): this rank's
    columns are stored straight into every rank's output buffer (PeerOutputs) by the library's
    reduction kernel over peer memory; one barrier then orders the ranks.  Returns this rank's full
    (r, total_cols) output (a view of peers.out: the next call overwrites it).

    host_barrier: synchronize the device and use a host barrier (gloo groups); otherwise the NCCL
    barrier is stream-ordered after the stores.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    c0, c1 = column_range(total_cols, world, rank)
    if M_shard.shape[1] != c1 - c0:
        raise ValueError("rank %d expects %d columns, got %d" % (rank, c1 - c0, M_shard.shape[1]))
    if c1 > c0:
        plan.sketch_columns_peers(M_shard, c0, peers.peer_order(), plan.r, workspace=workspace)
    if host_barrier:
        torch.cuda.synchronize()
    dist.barrier(group=group)
    return peers.out


def row_range(n, world, rank, granularity):
    """Row shard [r0, r1) of n rows for `rank`: whole multiples of `granularity`, the last
    rank also takes the tail (balanced over granules)."""
    granules = -(-int(n) // int(granularity))
    base, rem = divmod(granules, int(world))
    g0 = rank * base + min(rank, rem)
    g1 = g0 + base + (1 if rank < rem else 0)
    return min(g0 * granularity, n), min(g1 * granularity, n)


def sketch_row_sharded(plan, M_rows, row0, group=None, partial_fn=None, workspace=None, finish_fn=None, out=None):
    """Sketch of a row-partitioned [A | b]: this rank's rows [row0, row0 + M_rows.rows).

    plan:       srht Plan (same seed on every rank)
    M_rows:     this rank's rows of every column (row_range with plan.row_shard_rows())
    partial_fn: optional replacement for ``plan.sketch_rows_partial`` with the same contract
                (the CPU/gloo tests plug in the oracle)
    finish_fn:  optional replacement for ``plan.rows_finish`` (r^{-1/2} scale + FP32 rounding,
                done by the library's srht_rows_finish on the GPU path)
    Returns the float32 (r, c) sketch (column-major) on every rank.
    """
    if M_rows.shape[0] == 0:  # a rank past the last granule contributes zeros
        part = torch.zeros((M_rows.shape[1], plan.r), dtype=torch.float64, device=M_rows.device).t()
    elif partial_fn is None:
        part = plan.sketch_rows_partial(M_rows, row0, workspace=workspace)
    else:
        part = partial_fn(M_rows, row0)
    if not part.t().is_contiguous():
        part = part.t().contiguous().t()  # column-major (r, c)
    flat = part.t()  # (c, r) view of the column-major buffer, contiguous
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    if finish_fn is not None:
        return finish_fn(part)
    return plan.rows_finish(part, out=out)
