"""B200-native SRHT sketch of [A | b] -- the hot path of RandomizedNNLS (arXiv 0812.4547).

Thin Python binding over the C ABI in ``include/srht.h`` (``libsrht.so``, built
in-tree for sm_100a).  Every step of the sketch runs in the library's CUDA
kernels; this module only marshals torch tensors into pointers, sizes and the
current CUDA stream.  There is no CPU fallback: importing works without a GPU
(so the ABI can be inspected), but every call needs a CUDA device.

    plan = Plan(n, d, r, seed)            # Algorithm 1 steps 2 and 4 (device)
    SA, Sb = plan.sketch(A, b)            # H~ D A and H~ D b (step 5 inputs)

Dense inputs are column-major FP32 CUDA tensors of shape (n, c) (stride(0) == 1);
sparse inputs are ``CSC`` triples or ``torch.sparse_csc`` tensors.  Outputs are
column-major (r, c) FP32 tensors.
"""

import ctypes
from collections import namedtuple

import numpy as np

from . import _lib
from ._lib import SRHT_CSC, SRHT_DENSE, SrhtMatrix, SrhtError, check

__all__ = ["Plan", "CSC", "SrhtError", "colmajor", "gen_uniform", "gram", "nnls_gram", "padded_size", "library",
           "subspace_sampling"]

CSC = namedtuple("CSC", ["colptr", "rowidx", "vals", "shape"])
CSC.__doc__ = "Compressed sparse columns: int64 colptr[c+1], int32 rowidx[nnz] (sorted per column), float32 vals."


def library():
    """The loaded ctypes library (raises ImportError if it was not built)."""
    return _lib.load()


def padded_size(n):
    N = 2
    while N < n:
        N *= 2
    return N


def _torch():
    import torch
    return torch


def colmajor(x):
    """Column-major copy/view of a 2-D tensor (no copy if already column-major)."""
    if x.dim() == 1:
        return x.reshape(-1, 1)
    if x.stride(0) == 1 and (x.shape[1] <= 1 or x.stride(1) >= x.shape[0]):
        return x
    return x.t().contiguous().t()


def _check_out(out, shape, dtype, device):
    """Raise ValueError unless `out` is a column-major `dtype` tensor of `shape` on `device`."""
    torch = _torch()
    if not isinstance(out, torch.Tensor) or out.dtype != dtype or out.device != torch.device(device):
        raise ValueError("output must be a %s tensor on %s" % (dtype, device))
    if tuple(out.shape) != tuple(shape):
        raise ValueError("output has shape %s, expected %s" % (tuple(out.shape), tuple(shape)))
    rows = shape[0]
    if len(shape) == 1:
        if out.numel() > 1 and out.stride(0) != 1:
            raise ValueError("vector output must be contiguous")
        return
    if rows > 1 and out.stride(0) != 1:
        raise ValueError("output must be column-major (stride(0) == 1)")
    if shape[1] > 1 and out.stride(1) < rows:
        raise ValueError("output columns overlap (stride(1) < rows)")


def _stream_ptr(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _as_csc(M):
    torch = _torch()
    if isinstance(M, CSC):
        return M
    if isinstance(M, torch.Tensor) and M.layout == torch.sparse_csc:
        return CSC(M.ccol_indices().to(torch.int64), M.row_indices().to(torch.int32),
                   M.values().to(torch.float32), tuple(M.shape))
    return None


def _describe(M, keep):
    """srht_matrix for a device tensor / CSC; `keep` collects tensors to keep alive."""
    torch = _torch()
    csc = _as_csc(M)
    if csc is not None:
        colptr = csc.colptr.to(torch.int64).contiguous()
        rowidx = csc.rowidx.to(torch.int32).contiguous()
        vals = csc.vals.to(torch.float32).contiguous()
        keep += [colptr, rowidx, vals]
        rows, cols = int(csc.shape[0]), int(csc.shape[1])
        for t in (colptr, rowidx, vals):
            if not t.is_cuda:
                raise ValueError("CSC arrays must be CUDA tensors")
        return SrhtMatrix(SRHT_CSC, rows, cols, vals.data_ptr(), max(rows, 1), colptr.data_ptr(),
                          rowidx.data_ptr(), int(vals.numel()))
    if not isinstance(M, torch.Tensor) or not M.is_cuda:
        raise ValueError("dense input must be a CUDA tensor")
    if M.dtype != torch.float32:
        raise ValueError("dense input must be float32")
    M = colmajor(M)
    keep.append(M)
    rows, cols = int(M.shape[0]), int(M.shape[1])
    ld = int(M.stride(1)) if cols > 1 else max(rows, 1)
    return SrhtMatrix(SRHT_DENSE, rows, cols, M.data_ptr(), max(ld, rows, 1), None, None, 0)


class Plan:
    """Plan of Algorithm 1's random matrices D and S for `batch` problems of shape n x d.

    Created on the current CUDA device (synchronous).  `seed` selects the
    Philox streams (R4); problem p uses streams (seed, 2p), (seed, 2p+1).
    """

    def __init__(self, n, d, r, seed=0, batch=1, accum="fp32", sampling="exact"):
        if accum not in ("fp32", "fp64"):
            raise ValueError("accum must be 'fp32' or 'fp64'")
        if sampling not in ("exact", "bernoulli"):
            raise ValueError("sampling must be 'exact' or 'bernoulli'")
        self._lib = _lib.load()
        self._h = ctypes.c_void_p()
        flags = (_lib.SRHT_PLAN_ACCUM_FP64 if accum == "fp64" else 0) | \
                (_lib.SRHT_PLAN_BERNOULLI if sampling == "bernoulli" else 0)
        self.sampling = sampling
        self.r_target = int(r)
        check(self._lib.srht_plan_create_ex(int(n), int(d), int(r), ctypes.c_uint64(int(seed) & (2**64 - 1)),
                                            int(batch), flags, ctypes.byref(self._h)), "srht_plan_create_ex")
        self.accum = accum
        N, rr, bb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(self._lib.srht_plan_info(self._h, ctypes.byref(N), ctypes.byref(rr), ctypes.byref(bb)), "srht_plan_info")
        self.n, self.d, self.r, self.N, self.batch, self.seed = int(n), int(d), int(rr.value), int(N.value), int(bb.value), int(seed)
        torch = _torch()
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._ws = None

    # -- lifetime --
    def close(self):
        if self._h:
            self._lib.srht_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- introspection --
    def indices(self, problem=0):
        out = np.empty(self.r, dtype=np.int32)
        check(self._lib.srht_plan_copy_indices(self._h, int(problem), out.ctypes.data), "srht_plan_copy_indices")
        return out

    def sign_words(self, problem=0):
        out = np.empty((self.N + 63) // 64, dtype=np.uint64)
        check(self._lib.srht_plan_copy_signs(self._h, int(problem), out.ctypes.data), "srht_plan_copy_signs")
        return out

    def workspace_bytes(self, ncols):
        return int(self._lib.srht_workspace_bytes(self._h, int(ncols)))

    def workspace(self, ncols):
        nb = self.workspace_bytes(ncols)
        if nb == 0:
            return None
        torch = _torch()
        if self._ws is None or self._ws.numel() < nb:
            self._ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
        return self._ws

    def _ws_args(self, ncols, workspace):
        nb = self.workspace_bytes(ncols)
        if nb == 0:
            return None, 0
        ws = workspace if workspace is not None else self.workspace(ncols)
        return ws.data_ptr(), int(ws.numel())

    def _out(self, rows, cols, out, dtype=None):
        """A column-major (rows, cols) output on the plan's device: new, or the caller's after
        checking dtype, device, shape and strides (the C ABI writes rows x cols entries)."""
        torch = _torch()
        dtype = torch.float32 if dtype is None else dtype
        if out is None:
            return torch.empty((cols, rows), dtype=dtype, device=self.device).t()
        _check_out(out, (rows, cols), dtype, self.device)
        return out

    # -- the sketch --
    def sketch(self, A, b=None, SA=None, Sb=None, workspace=None):
        """(H~ D A, H~ D b) with one shared plan (Algorithm 1 step 5)."""
        keep = []
        dA = _describe(A, keep)
        SA = self._out(self.r, dA.cols, SA)
        db, sb_ptr = None, None
        if b is not None:
            if _as_csc(b) is None and b.dim() == 1:
                b = b.reshape(-1, 1)
            db = _describe(b, keep)
            torch = _torch()
            if Sb is None:
                Sb = torch.empty(self.r, dtype=torch.float32, device=self.device)
            else:
                _check_out(Sb, (self.r,), torch.float32, self.device)
            sb_ptr = Sb.data_ptr()
        ncols = dA.cols + (1 if b is not None else 0)
        ws, wsb = self._ws_args(ncols, workspace)
        ldsa = int(SA.stride(1)) if SA.shape[1] > 1 else self.r
        check(self._lib.srht_sketch(self._h, ctypes.byref(dA), ctypes.byref(db) if db is not None else None,
                                    SA.data_ptr(), ldsa, sb_ptr, ws, wsb, _stream_ptr(self.device)), "srht_sketch")
        return SA, Sb

    def sketch_columns(self, M, out=None, workspace=None):
        """H~ D M for every column of M (the column-shard primitive)."""
        keep = []
        dM = _describe(M, keep)
        SM = self._out(self.r, dM.cols, out)
        ws, wsb = self._ws_args(dM.cols, workspace)
        ld = int(SM.stride(1)) if SM.shape[1] > 1 else self.r
        check(self._lib.srht_sketch_columns(self._h, ctypes.byref(dM), SM.data_ptr(), ld, ws, wsb,
                                            _stream_ptr(self.device)), "srht_sketch_columns")
        return SM

    def sketch_columns_peers(self, M, col0, peer_ptrs, ld, workspace=None):
        """Sketch of M's columns stored at columns [col0, col0 + cols) of every buffer in
        `peer_ptrs` (device addresses, this rank's own output first; ld >= r): the column-shard
        sketch with the gather fused in (srht_sketch_columns_peers)."""
        keep = []
        dM = _describe(M, keep)
        ws, wsb = self._ws_args(dM.cols, workspace)
        arr = (ctypes.c_void_p * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
        check(self._lib.srht_sketch_columns_peers(self._h, ctypes.byref(dM), int(col0), arr, len(peer_ptrs), int(ld),
                                                  ws, wsb, _stream_ptr(self.device)), "srht_sketch_columns_peers")

    def row_shard_rows(self):
        """Row granularity of row shards (srht_row_shard_rows)."""
        return int(self._lib.srht_row_shard_rows(self._h))

    def sketch_rows_partial(self, M, row0, out=None, workspace=None):
        """Unscaled FP64 partial sums of rows [row0, row0 + M.rows) of [A | b] (a row shard).

        M holds the shard's rows (dense: the local rows; CSC: global row indices).  Returns a
        column-major float64 (r, c) tensor; r^{-1/2} times the sum over a row partition is the
        sketch (srht_sketch_rows_partial).
        """
        torch = _torch()
        keep = []
        dM = _describe(M, keep)
        out = self._out(self.r, dM.cols, out, dtype=torch.float64)
        ws, wsb = self._ws_args(dM.cols, workspace)
        ld = int(out.stride(1)) if dM.cols > 1 else self.r
        check(self._lib.srht_sketch_rows_partial(self._h, ctypes.byref(dM), int(row0), out.data_ptr(), ld, ws, wsb,
                                                 _stream_ptr(self.device)), "srht_sketch_rows_partial")
        return out

    def rows_finish(self, part, out=None):
        """Float32 sketch r^{-1/2} * part from the summed FP64 partials of a row partition
        (srht_rows_finish: one FP64 scale and one rounding per entry, in the library)."""
        torch = _torch()
        if part.dim() != 2 or part.shape[0] != self.r:
            raise ValueError("part must be (r, c)")
        _check_out(part, tuple(part.shape), torch.float64, self.device)
        cols = int(part.shape[1])
        out = self._out(self.r, cols, out)
        ldp = int(part.stride(1)) if cols > 1 else self.r
        ld = int(out.stride(1)) if cols > 1 else self.r
        check(self._lib.srht_rows_finish(self._h, part.data_ptr(), ldp, cols, out.data_ptr(), ld,
                                         _stream_ptr(self.device)), "srht_rows_finish")
        return out

    def sketch_batched(self, M, out=None, workspace=None):
        """Batched problems: M has batch*c columns; returns (batch, c, r) (row t fastest)."""
        torch = _torch()
        keep = []
        dM = _describe(M, keep)
        c = dM.cols // self.batch
        if out is None:
            out = torch.empty((self.batch, c, self.r), dtype=torch.float32, device=self.device)
        elif (not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or out.device != self.device
              or tuple(out.shape) != (self.batch, c, self.r) or not out.is_contiguous()):
            raise ValueError("out must be a contiguous float32 (batch, c, r) tensor on %s" % self.device)
        ws, wsb = self._ws_args(dM.cols, workspace)
        check(self._lib.srht_sketch_batched(self._h, ctypes.byref(dM), out.data_ptr(), ws, wsb,
                                            _stream_ptr(self.device)), "srht_sketch_batched")
        return out

    def sketch_columns_host(self, M, out=None):
        """End-to-end call on HOST buffers (copies, sketch and read-back inside).

        M: column-major float32 CPU tensor (n, c) (pinned for full PCIe speed) or a
        CSC of CPU tensors.  Returns a column-major float32 CPU tensor (r, c).
        """
        torch = _torch()
        csc = _as_csc(M)
        if csc is not None:
            colptr = csc.colptr.to(torch.int64).contiguous()
            rowidx = csc.rowidx.to(torch.int32).contiguous()
            vals = csc.vals.to(torch.float32).contiguous()
            desc = SrhtMatrix(SRHT_CSC, int(csc.shape[0]), int(csc.shape[1]), vals.data_ptr(), max(int(csc.shape[0]), 1),
                              colptr.data_ptr(), rowidx.data_ptr(), int(vals.numel()))
            cols = int(csc.shape[1])
        else:
            M = colmajor(M)
            if M.is_cuda or M.dtype != torch.float32:
                raise ValueError("host input must be a float32 CPU tensor")
            cols = int(M.shape[1])
            ld = int(M.stride(1)) if cols > 1 else max(int(M.shape[0]), 1)
            desc = SrhtMatrix(SRHT_DENSE, int(M.shape[0]), cols, M.data_ptr(), ld, None, None, 0)
        if out is None:
            out = torch.empty((cols, self.r), dtype=torch.float32).t()
        ld_out = int(out.stride(1)) if cols > 1 else self.r
        check(self._lib.srht_sketch_columns_host(self._h, ctypes.byref(desc), out.data_ptr(), ld_out),
              "srht_sketch_columns_host")
        return out


def gen_uniform(seed, stream0, out):
    """Fill a column-major float32 CUDA tensor with the workload generator's exact
    Uniform[0,1) values (column j <- Philox stream (seed, 2^32 + stream0 + j))."""
    lib = _lib.load()
    out2 = out.reshape(-1, 1) if out.dim() == 1 else out
    if out2.stride(0) != 1:
        raise ValueError("gen_uniform needs a column-major tensor")
    rows, cols = int(out2.shape[0]), int(out2.shape[1])
    ld = int(out2.stride(1)) if cols > 1 else max(rows, 1)
    check(lib.srht_gen_uniform(ctypes.c_uint64(seed), ctypes.c_uint64(stream0), rows, cols, out2.data_ptr(), ld,
                               _stream_ptr(out.device)), "srht_gen_uniform")
    return out


def gram(SM):
    """FP64 Gram matrices G = SM^T SM of sketches (srht_gram; the QP form of Section 3.4).

    SM: column-major float32 CUDA tensor (r, c), or a (batch, c, r) tensor as returned by
    Plan.sketch_batched.  Returns (c, c) or (batch, c, c) float64 (symmetric).
    """
    torch = _torch()
    lib = _lib.load()
    if not SM.is_cuda or SM.dtype != torch.float32:
        raise ValueError("SM must be a float32 CUDA tensor")
    if SM.dim() == 3:  # (batch, c, r): block p is column-major r x c with ld = r
        batch, c, r = (int(x) for x in SM.shape)
        SM = SM.contiguous()
        ld, stride = r, r * c
    else:
        SM = colmajor(SM)
        batch, r, c = 1, int(SM.shape[0]), int(SM.shape[1])
        ld = int(SM.stride(1)) if c > 1 else max(r, 1)
        stride = ld * c
    G = torch.empty((batch, c, c), dtype=torch.float64, device=SM.device)
    wsb = int(lib.srht_gram_workspace_bytes(r, c, batch))
    ws = _gram_scratch(SM.device, wsb)
    check(lib.srht_gram_ex(r, c, batch, SM.data_ptr(), ld, stride, G.data_ptr(), c, c * c,
                           ws.data_ptr() if ws is not None else None, wsb, _stream_ptr(SM.device)), "srht_gram_ex")
    return G if SM.dim() == 3 else G[0]


_GRAM_WS = {}


def _gram_scratch(device, nbytes):
    """256-byte aligned scratch for srht_gram_ex, cached per device.  Calls on different streams
    of one device must not overlap (torch's current stream orders them)."""
    if nbytes == 0:
        return None
    torch = _torch()
    key = str(device)
    buf = _GRAM_WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _GRAM_WS[key] = buf
    return buf


def nnls_gram(G, method="auto"):
    """NNLS on the Gram form: x = argmin_{x>=0} x^T Q x - 2 q^T x (Algorithm 1 step 5).

    G: float64 CUDA tensor (c, c) or (batch, c, c) from :func:`gram` of [SA | Sb] (c = d + 1).
    method: "lh" Lawson-Hanson with the oracle's pivot rules (srht_nnls_gram), "bpp" block
    principal pivoting (srht_nnls_gram_bpp; same optimum, few refactorizations, d <= 580),
    "auto" = bpp for d > 156 (factor outside shared memory), else lh.
    Returns (x, iters): x float64 (d,) or (batch, d); iters int32 (iterations, or a negative
    failure code per problem, see the header).
    """
    torch = _torch()
    lib = _lib.load()
    if not G.is_cuda or G.dtype != torch.float64:
        raise ValueError("G must be a float64 CUDA tensor")
    single = G.dim() == 2
    Gb = (G.unsqueeze(0) if single else G).contiguous()
    batch, c = int(Gb.shape[0]), int(Gb.shape[1])
    d = c - 1
    x = torch.empty((batch, d), dtype=torch.float64, device=G.device)
    iters = torch.empty((batch,), dtype=torch.int32, device=G.device)
    if method == "auto":
        method = "bpp" if d > 156 else "lh"
    if method not in ("lh", "bpp"):
        raise ValueError("method must be 'lh', 'bpp' or 'auto'")
    fn = lib.srht_nnls_gram_bpp if method == "bpp" else lib.srht_nnls_gram
    wsb = int(lib.srht_nnls_bpp_workspace_bytes(d, batch) if method == "bpp" else lib.srht_nnls_workspace_bytes(d, batch))
    ws = torch.empty((max(wsb, 8) // 8,), dtype=torch.float64, device=G.device)
    check(fn(d, batch, Gb.data_ptr(), c, c * c, x.data_ptr(), d, iters.data_ptr(),
             ws.data_ptr(), wsb, _stream_ptr(G.device)), fn.__name__)
    return (x[0], iters[0]) if single else (x, iters)


def subspace_sampling(Phi, r, p, seed=0):
    """Algorithm 2, SubspaceSampling (srht_subspace_sample): (K, Phi~) with K the kept row
    indices (int32, ascending) and Phi~ the kept rows of Phi scaled by 1/sqrt(min(1, r p_i)).

    Phi: float32 CUDA tensor (n, d) (column-major used as is, else copied); p: float64 CUDA
    tensor (n,) of probabilities.
    """
    torch = _torch()
    lib = _lib.load()
    Phi = colmajor(Phi)
    n, d = int(Phi.shape[0]), int(Phi.shape[1])
    p = p.to(torch.float64).contiguous()
    st = _stream_ptr(Phi.device)
    kept = ctypes.c_int64()
    check(lib.srht_subspace_sample_count(n, int(r), ctypes.c_uint64(int(seed) & (2**64 - 1)), p.data_ptr(),
                                         ctypes.byref(kept), st), "srht_subspace_sample_count")
    k = int(kept.value)
    K = torch.empty((max(k, 1),), dtype=torch.int32, device=Phi.device)
    out = torch.empty((d, max(k, 1)), dtype=torch.float32, device=Phi.device).t()
    ld = int(Phi.stride(1)) if d > 1 else max(n, 1)
    check(lib.srht_subspace_sample(n, d, int(r), ctypes.c_uint64(int(seed) & (2**64 - 1)), p.data_ptr(),
                                   Phi.data_ptr(), ld, K.data_ptr(), out.data_ptr(), max(k, 1), k, st),
          "srht_subspace_sample")
    return K[:k], out[:k]
