"""ctypes declarations of include/srht.h (argument marshalling only)."""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("SRHT_LIB", "libsrht.so"))

SRHT_DENSE = 0
SRHT_CSC = 1

SRHT_PLAN_ACCUM_FP64 = 1
SRHT_PLAN_BERNOULLI = 2

SRHT_OK = 0
SRHT_EINVAL = 1
SRHT_ENOMEM = 2
SRHT_ECUDA = 3
SRHT_EUNSUPPORTED = 4


class SrhtMatrix(ctypes.Structure):
    _fields_ = [
        ("fmt", ctypes.c_int32),
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("vals", ctypes.c_void_p),
        ("ld", ctypes.c_int64),
        ("colptr", ctypes.c_void_p),
        ("rowidx", ctypes.c_void_p),
        ("nnz", ctypes.c_int64),
    ]


# (name, restype, argtypes) for every symbol the header declares.
_P = ctypes.c_void_p
_PP = ctypes.POINTER(ctypes.c_void_p)
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_MP = ctypes.POINTER(SrhtMatrix)
SIGNATURES = [
    ("srht_plan_create", ctypes.c_int, [_I64, _I64, _I64, _U64, _PP]),
    ("srht_plan_create_batched", ctypes.c_int, [_I64, _I64, _I64, _U64, _I64, _PP]),
    ("srht_plan_create_ex", ctypes.c_int, [_I64, _I64, _I64, _U64, _I64, ctypes.c_uint32, _PP]),
    ("srht_plan_destroy", ctypes.c_int, [_P]),
    ("srht_plan_info", ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("srht_plan_copy_indices", ctypes.c_int, [_P, _I64, _P]),
    ("srht_plan_copy_signs", ctypes.c_int, [_P, _I64, _P]),
    ("srht_workspace_bytes", ctypes.c_size_t, [_P, _I64]),
    ("srht_sketch", ctypes.c_int, [_P, _MP, _MP, _P, _I64, _P, _P, ctypes.c_size_t, _P]),
    ("srht_sketch_columns", ctypes.c_int, [_P, _MP, _P, _I64, _P, ctypes.c_size_t, _P]),
    ("srht_sketch_columns_peers", ctypes.c_int, [_P, _MP, _I64, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, _I64,
                                                 _P, ctypes.c_size_t, _P]),
    ("srht_sketch_batched", ctypes.c_int, [_P, _MP, _P, _P, ctypes.c_size_t, _P]),
    ("srht_sketch_columns_host", ctypes.c_int, [_P, _MP, _P, _I64]),
    ("srht_row_shard_rows", ctypes.c_int64, [_P]),
    ("srht_gram", ctypes.c_int, [_I64, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P]),
    ("srht_gram_workspace_bytes", ctypes.c_size_t, [_I64, _I64, _I64]),
    ("srht_gram_ex", ctypes.c_int, [_I64, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P, ctypes.c_size_t, _P]),
    ("srht_nnls_workspace_bytes", ctypes.c_size_t, [_I64, _I64]),
    ("srht_subspace_sample_count", ctypes.c_int, [_I64, _I64, _U64, _P, ctypes.POINTER(_I64), _P]),
    ("srht_subspace_sample", ctypes.c_int, [_I64, _I64, _I64, _U64, _P, _P, _I64, _P, _P, _I64, _I64, _P]),
    ("srht_nnls_gram", ctypes.c_int, [_I64, _I64, _P, _I64, _I64, _P, _I64, _P, _P, ctypes.c_size_t, _P]),
    ("srht_nnls_bpp_workspace_bytes", ctypes.c_size_t, [_I64, _I64]),
    ("srht_nnls_gram_bpp", ctypes.c_int, [_I64, _I64, _P, _I64, _I64, _P, _I64, _P, _P, ctypes.c_size_t, _P]),
    ("srht_sketch_rows_partial", ctypes.c_int, [_P, _MP, _I64, _P, _I64, _P, ctypes.c_size_t, _P]),
    ("srht_rows_finish", ctypes.c_int, [_P, _P, _I64, _I64, _P, _I64, _P]),
    ("srht_ipc_alloc", ctypes.c_int, [ctypes.c_size_t, _PP, _P]),
    ("srht_ipc_open", ctypes.c_int, [_P, _PP]),
    ("srht_ipc_close", ctypes.c_int, [_P]),
    ("srht_ipc_free", ctypes.c_int, [_P]),
    ("srht_status_str", ctypes.c_char_p, [ctypes.c_int]),
    ("srht_gen_uniform", ctypes.c_int, [_U64, _U64, _I64, _I64, _P, _I64, _P]),
    ("srht_profile_start", ctypes.c_int, [ctypes.c_int]),
    ("srht_profile_stop", ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
]

_lib = None


def load():
    """Load libsrht.so; raise (loudly) if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            "libsrht.so not found at %s; build it with `python -m paper_0812_4547_b200.build` "
            "(there is no CPU fallback)" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class SrhtError(RuntimeError):
    def __init__(self, status, where):
        msg = load().srht_status_str(status).decode()
        super().__init__("%s failed: %s (status %d)" % (where, msg, status))
        self.status = status


def check(status, where):
    if status != SRHT_OK:
        raise SrhtError(status, where)
